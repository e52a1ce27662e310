"""bench.py — candidate plans evaluated/sec and time-to-best-plan, B200 vs the CPU reference.

Workload (BASELINE.json configs[4], the config the metric's 1/2/4/8-B200 sharding is
quoted on): cfg5 = omni-modal 8-module MM (7 encoders -> backbone, profiler.hpp:212-285)
on 128 modeled GPUs, quota granularity 1/32, GAHC (solver.hpp:157-289).

Both arms time the SAME work (like-for-like):
  * one STEP = the identical-work sample: the stage_eval calls (stage_eval.hpp:302-382) of
    the cfg5 GAHC solve that the reference finishes in seconds — the 29 EvalCache entries
    with k <= 4 modules, in call order, cold cache (tests/golden/cfg5_sample.json);
  * value = the REFERENCE's complete-allocation count for that sample (its verify_complete
    leaves, stage_eval.hpp:254, counted once by the instrumented reference and committed)
    / the arm's time, so value_ours / value_reference = t_reference / t_ours on identical
    work.  Our arm also checks every stage time against the reference's, bit for bit.
  * time_to_best_plan_s = the full cfg5 solve.  Ours: device-timed.  Reference: run under a
    wall-clock cap and reported as "> cap" when it does not finish.
  * e2e (ours) = the sample through the C ABI from HOST buffers: mosaic_gpu_create from host
    surface tables (option tables packed on the device) + the 29 stage_evals + results read
    back, host wall clock.
  * evaluator = K1 (mosaic_gpu_evaluate) on 2^20 random cfg5 allocations, with its roofline.
Multi-GPU (torchrun, one rank per GPU): the sample's masks are dealt to ranks (no
collective); the full solve shards each device search's frontier (mosaic_gpu_set_shard).

--impl reference runs the reference's own CPU planner (oracle/_ref, the unmodified headers
compiled by oracle/Makefile) on the same sample, one process per stage_eval on every host
core (the reference is single-threaded), plus the capped full solve.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = "cfg5"
METRIC = ("candidate plans evaluated/sec (reference-equivalent: the reference's complete "
          "allocations over an identical cfg5 GAHC stage_eval sample) and time-to-best-plan")
UNIT = "plans/s"
REF_DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver_instr")
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
with open(os.path.join(ROOT, "tests", "golden", "cfg5_sample.json")) as _f:
    SAMPLE = json.load(_f)
SAMPLE_LEAVES = SAMPLE["leaves"]
CONFIG = {"workload": "cfg5: omni-modal 8-module MM, 128 modeled GPUs, quota 1/32; step = "
                      "the 29 stage_evals (k<=4) of its GAHC solve, cold cache; "
                      "time_to_best_plan = the full GAHC solve",
          "modeled_gpus": 128, "quota_levels": 32, "modules": 8,
          "sample_masks": len(SAMPLE["masks"]), "sample_reference_leaves": SAMPLE_LEAVES}


def mask_bits(m: int) -> list[int]:
    return [i for i in range(64) if m >> i & 1]


def deal(masks: list[dict], rank: int, world: int) -> list[dict]:
    """Masks of this rank: dealt in decreasing reference cost (k-module stages dominate)."""
    order = sorted(range(len(masks)), key=lambda i: -masks[i]["cpu_s"])
    mine = sorted(order[rank::world])
    return [masks[i] for i in mine]


def peaks() -> tuple[float, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        for k in ("hbm_gbs", "hbm_GBs", "hbm"):
            if k in d:
                return float(d[k]), "measured"
    except Exception:
        pass
    return FALLBACK_HBM_GBS, "fallback"


class Clocks:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()  # the first sample lands before the timed region starts
            while not self.rows and time.time() - t0 < 3.0 and self.proc.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm = [float(r[0]) for r in self.rows if len(r) > 1 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 3 + i and r[3 + i].lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def flush_l2(torch, dev) -> None:
    # 256 MiB write > 126 MB L2, between timed steps (outside the timed region)
    buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    buf.fill_(1.0)
    torch.cuda.synchronize(dev)


def host_cpu() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_ref_sample(masks: list[dict], parallel: int) -> dict:
    """The reference planner on `masks`, one process per stage_eval, `parallel` at a time
    (largest first), pinned to one core each when parallel == 1."""
    if not os.path.exists(REF_DRIVER):
        raise FileNotFoundError(f"{REF_DRIVER} missing (build with make -C oracle ref)")
    todo = sorted(masks, key=lambda m: -m["cpu_s"])
    t0 = time.perf_counter()
    procs, leaves = [], 0
    while todo or procs:
        while todo and len(procs) < parallel:
            m = todo.pop(0)
            cmd = [REF_DRIVER, WORKLOAD, "stage", str(m["mask"])]
            if parallel == 1:
                cmd = ["taskset", "-c", "0"] + cmd
            procs.append((m, subprocess.Popen(cmd, stdout=subprocess.PIPE, text=True)))
        m, p = procs.pop(0)
        d = json.loads(p.communicate()[0])
        assert d["t"] == m["t"] or float.fromhex(d["t"]) == float.fromhex(m["t"])
        leaves += d["leaves"]
    wall = time.perf_counter() - t0
    return {"leaves": leaves, "wall_s": wall, "value": leaves / wall if wall > 0 else 0.0}


def ref_solve_capped(cap: float) -> dict:
    t0 = time.perf_counter()
    try:
        subprocess.run([REF_DRIVER.replace("_instr", ""), WORKLOAD, "solve"],
                       capture_output=True, text=True, timeout=cap)
        return {"time_to_best_plan_s": time.perf_counter() - t0, "finished": True}
    except subprocess.TimeoutExpired:
        return {"time_to_best_plan_s": f"> {cap:.0f}", "finished": False, "cap_s": cap}


def reference_arm(args) -> None:
    if int(os.environ.get("RANK", "0")) != 0:
        return
    ncores = os.cpu_count() or 1
    par = max(1, min(ncores, len(SAMPLE["masks"])))
    for _ in range(args.warmup):
        run_ref_sample(SAMPLE["masks"], par)
    walls, leaves = [], 0
    for _ in range(args.steps):
        r = run_ref_sample(SAMPLE["masks"], par)
        walls.append(r["wall_s"])
        leaves += r["leaves"]
    total = sum(walls)
    value = leaves / total if total else 0.0
    tt = ref_solve_capped(args.ref_cap)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * total / max(1, args.steps), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": CONFIG, "same_config": True,
        "time_to_best_plan_s": tt["time_to_best_plan_s"], "full_solve": tt,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": par, "kind": "reference",
                         "sample": f"the {len(SAMPLE['masks'])} cfg5 stage_evals of one step, "
                                   "one process per stage_eval on every host core "
                                   "(the reference is single-threaded)",
                         "cpu": host_cpu(), "host_cores": ncores},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


N_EVAL = 1 << 20  # allocations per evaluator step
# dram__bytes_read.sum + dram__bytes_write.sum of k_evaluate_fast on this workload, one
# `ncu --set full` capture (profiles/r2_ncu_k_evaluate_fast.md): 761.9 MB + 12.0 MB
EVAL_TRAFFIC_PER_LAUNCH = 773.8e6


def evaluator_leg(pl, torch, dev, steps: int, warmup: int, peak: float, peak_kind: str) -> dict:
    """K1 (mosaic_gpu_evaluate): stage_time of N_EVAL random cfg5 allocations per step.
    Device leg: inputs resident in HBM (>L2, and L2 flushed between steps), kernel time by
    CUDA events on the context stream.  e2e leg: the same call on pinned HOST arrays (H2D of
    the inputs + D2H of the stage times inside the timed region)."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from evalgen import random_allocations
    ent, gpus, off = random_allocations(pl, N_EVAL, seed=0)
    n = len(off) - 1
    tE, tG, tO = (torch.from_numpy(x).to(dev) for x in (ent, gpus, off))
    st = torch.empty(n, dtype=torch.float64, device=dev)
    torch.cuda.synchronize(dev)
    for _ in range(warmup):
        pl.evaluate(tE, tG, tO, st, None, device=True)
    pl.reset_counters()
    for _ in range(steps):
        flush_l2(torch, dev)
        pl.evaluate(tE, tG, tO, st, None, device=True)
    s = pl.evaluate_stats()
    s0 = s
    k_ms = s["kernel_ms"] / max(1, s["launches"])
    f_ms = s["fast_kernel_ms"] / max(1, s["launches"])
    alg = s["alg_bytes"] / max(1, s["launches"])
    achieved = alg / (k_ms / 1e3) / 1e9 if k_ms > 0 else 0.0
    hE, hG, hO = (torch.from_numpy(x).pin_memory() for x in (ent, gpus, off))
    hst = torch.empty(n, dtype=torch.float64).pin_memory()
    pl.evaluate(hE, hG, hO, hst, None)
    t0 = time.perf_counter()
    for _ in range(steps):
        pl.evaluate(hE, hG, hO, hst, None)
    e2e_s = (time.perf_counter() - t0) / max(1, steps)
    assert torch.equal(hst.to(dev), st), "host and device evaluator legs disagree"
    h2d = ent.nbytes + gpus.nbytes + off.nbytes
    return {"metric": "allocations scored/sec (K1 stage_time, mosaic_gpu_evaluate)",
            "value": n / (k_ms / 1e3) if k_ms > 0 else 0.0, "unit": "allocations/s",
            "allocations": n, "entries": int(len(ent)), "gpu_ids": int(len(gpus)),
            "kernel_ms": k_ms, "fast_kernel_ms": f_ms,
            "full_path_allocs": s0["full_path_allocs"],
            "kernels": "k_evaluate_fast (include_self, <= 32 entries, distinct modules) + "
                       "k_evaluate over the worklist of allocations it hands over",
            "e2e": {"value": n / e2e_s, "unit": "allocations/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": n * 8, "timing": "host wall clock, pinned host arrays"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if peak else None,
                         "traffic": EVAL_TRAFFIC_PER_LAUNCH,
                         "kernel": "k_evaluate_fast + k_evaluate (eval.cu), per call",
                         "peak_kind": peak_kind,
                         "algorithmic_bytes": "per allocation 16 B (offset + stage time) + "
                                              "32 B per entry + 4 B per GPU id"},
            "data": "synthetic: random module subsets of cfg5, candidate options, "
                    "windows of d consecutive GPUs; inputs > L2, L2 flushed between steps"}


TRAFFIC_CSV = "profiles/r2_dram_sample.csv"
# `ncu --set full` of the dominant launch (cfg5 7-encoder MIN proof, 363.2 ms):
# profiles/r2_ncu_ksearch_min_cfg5_k7.ncu-rep
NCU_MIN7 = {"smem_wavefronts_frac_of_peak": 0.441, "lsu_pipe_frac": 0.435,
            "issue_active_frac": 0.490, "fp64_pipe_frac": 0.081,
            "source": "profiles/r2_ncu_ksearch_min7.md"}


def dram_traffic_per_launch():
    """Average DRAM bytes (read + write) per k_search launch in the committed ncu list."""
    import csv
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), TRAFFIC_CSV)
    if not os.path.exists(path):
        return None
    rows = list(csv.reader(open(path)))
    hdr = next((r for r in rows if "Kernel Name" in r), None)
    if hdr is None:
        return None
    tot, ids = 0.0, set()
    for r in rows:
        if len(r) != len(hdr) or r is hdr:
            continue
        d = dict(zip(hdr, r))
        if not d["Kernel Name"].startswith("k_search"):
            continue
        if d["Metric Name"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(d["Metric Unit"], 1)
            tot += float(d["Metric Value"].replace(",", "")) * scale
            ids.add(d["ID"])
    return tot / len(ids) if ids else None


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N>1: weak = every rank runs its own copy of the sample (independent "
                         "planning requests, no collective); strong = the sample's stage_evals "
                         "dealt over the ranks")
    ap.add_argument("--no-evaluator", action="store_true", help="skip the K1 evaluator leg")
    ap.add_argument("--workload", default="cfg5",
                    help="cfg5 (default, the headline); cfg1..cfg4 time only the full solve "
                         "(value = device leaves/s; used by the sharding tests)")
    ap.add_argument("--ref-cap", type=float, default=60.0,
                    help="wall-clock cap (s) of the reference's full cfg5 solve")
    ap.add_argument("--dist-backend", default="nccl",
                    help="nccl (default); gloo lets several ranks share one GPU for testing")
    ap.add_argument("--same-device", action="store_true",
                    help="every rank uses cuda:0 (sharding test on a single GPU)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch under torchrun on this node (the driver's own launch
        # sets WORLD_SIZE and lands below)
        os.execvp(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                   "--nproc-per-node", str(args.gpus), "--master-addr",
                                   "127.0.0.1", "--master-port", str(29400 + os.getpid() % 500),
                                   os.path.abspath(__file__)] + sys.argv[1:])
    if args.impl == "reference":
        reference_arm(args)
        return

    import torch
    import torch.distributed as dist

    global WORKLOAD
    WORKLOAD = args.workload
    headline = WORKLOAD == "cfg5"
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = 0 if args.same_device else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)

    from paper_2605_18710_b200 import mosaic

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    comm_dev = dev if args.dist_backend == "nccl" else torch.device("cpu")

    def allgather_bytes(b: bytes) -> list[bytes]:
        t = torch.frombuffer(bytearray(b), dtype=torch.uint8).to(comm_dev)
        outs = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(outs, t)
        return [bytes(o.cpu().numpy().tobytes()) for o in outs]

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=comm_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    # weak (default): per-GPU work fixed — every rank runs the whole sample, as independent
    # planning requests would arrive at a multi-GPU planner; strong: the 29 stage_evals dealt
    weak = args.scaling == "weak" or world == 1
    if headline:
        mine = list(SAMPLE["masks"]) if weak else deal(SAMPLE["masks"], rank, world)
    else:
        mine = []
    copies = world if weak else 1  # samples processed per step over all ranks
    want = {m["mask"]: float.fromhex(m["t"]) for m in mine}

    def run_sample(pl) -> None:
        if not mine:
            return
        # one batched stage search (mosaic_gpu_search): the stage_evals advance together,
        # one launch per wave of their device searches
        ts = pl.search([mask_bits(m["mask"]) for m in mine], times_only=True)
        for m, t in zip(mine, ts):
            # identical work: every stage time equals the reference's, bit for bit
            assert t == want[m["mask"]], (m["mask"], t)

    # ---- device-resident: tables already in HBM, time the sample ----
    pl = mosaic.Planner.from_spec(WORKLOAD, device=local)
    for _ in range(args.warmup):
        run_sample(pl)
    barrier()
    pl.reset_counters()
    dev_ms = []
    clk = Clocks(local).__enter__()  # sampled through both timed legs (sample and full solve)
    for _ in range(args.steps):
        flush_l2(torch, dev)
        barrier()
        pl.mark(0)
        run_sample(pl)
        pl.mark(1)
        dev_ms.append(pl.marked_ms())
    barrier()
    ctr = pl.counters()
    t_max = max_over_ranks(sum(dev_ms))
    value = copies * SAMPLE_LEAVES * args.steps / (t_max / 1000.0) if t_max > 0 else 0.0

    # ---- time to the best plan: the full solve (frontier sharded over ranks) ----
    plane = None
    if world > 1:
        if args.dist_backend == "nccl":
            # the library's own data plane: one NCCL communicator from a unique id rank 0 makes
            idt = torch.zeros(128, dtype=torch.uint8, device=dev)
            if rank == 0:
                idt.copy_(torch.frombuffer(bytearray(mosaic.nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(idt, 0)
            try:
                pl.set_shard_nccl(rank, world, bytes(idt.cpu().numpy().tobytes()))
                ok = 1
            except mosaic.MosaicError as e:  # reported in the line, never silent
                print(f"[bench] in-library NCCL plane unavailable: {e}", file=sys.stderr)
                ok = 0
            flag = torch.tensor([ok], dtype=torch.int32, device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag[0]):
                plane = "in-library NCCL all-gather per batched launch"
            else:
                pl.set_shard(rank, world, allgather_bytes)
                plane = "caller all-gather over torch.distributed (in-library NCCL failed)"
        else:
            pl.set_shard(rank, world, allgather_bytes)
            plane = f"caller all-gather over {args.dist_backend} per batched launch"
    for _ in range(max(1, args.warmup)):
        res = pl.solve()
    solve_ms = []
    for _ in range(args.steps):
        flush_l2(torch, dev)
        barrier()
        pl.mark(0)
        res = pl.solve()
        pl.mark(1)
        solve_ms.append(pl.marked_ms())
    clk.__exit__(None, None, None)
    ttbp = max_over_ranks(statistics.median(solve_ms)) / 1000.0
    if not headline:
        # no reference-equivalent count for the other configs: device leaves per second
        value = res.trace.leaves / ttbp if ttbp > 0 else 0.0
        t_max = ttbp * 1000.0 * args.steps
    best_plan = res.plan.predicted_iteration_time
    searches_per_solve = res.trace.stage_eval_calls
    peer_links = pl.counters()["peer_links"]

    # ---- e2e through the C ABI with host buffers (create + sample + read back) ----
    for _ in range(args.warmup):  # untimed: first-use allocations of the process
        p2 = mosaic.Planner.from_spec(WORKLOAD, device=local)
        run_sample(p2)
        p2.close()
    e2e_s, h2d, d2h = 0.0, 0, 0
    for _ in range(args.steps):
        barrier()
        t0 = time.perf_counter()
        p2 = mosaic.Planner.from_spec(WORKLOAD, device=local)
        run_sample(p2)
        c2 = p2.counters()
        p2.close()
        barrier()
        e2e_s += time.perf_counter() - t0
        h2d, d2h = c2["h2d_bytes"], c2["d2h_bytes"]
    e2e_s = max_over_ranks(e2e_s)
    e2e_value = copies * SAMPLE_LEAVES * args.steps / e2e_s if e2e_s > 0 and headline else None

    peak, peak_kind = peaks()
    evaluator = None
    if not args.no_evaluator and headline:
        evaluator = evaluator_leg(pl, torch, dev, args.steps, args.warmup, peak, peak_kind)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel of the sample (k_search) ----
    ks_ms = ctr["ksearch_ms"]
    ks_n = max(1, ctr["ksearch_launches"])
    alg_bytes = ctr.get("alg_bytes", 0)
    avg_launch_s = ks_ms / ks_n / 1000.0
    achieved = (alg_bytes / ks_n) / avg_launch_s / 1e9 if avg_launch_s > 0 else 0.0
    # SURVEY.md §8(d)'s on-chip roofline: the same algorithmic bytes against the measured
    # shared-memory bandwidth, beside the shared-memory pipe utilisation ncu measured on the
    # dominant launch (the 7-encoder MIN proof, profiles/r2_ncu_ksearch_min7.md)
    try:
        smem_peak = mosaic.smem_peak_gbs(local)
    except mosaic.MosaicError:
        smem_peak = None
    roofline_smem = {"bound": "smem", "achieved": achieved, "peak": smem_peak, "unit": "GB/s",
                     "frac": achieved / smem_peak if smem_peak else None,
                     "peak_kind": "measured (mosaic_gpu_smem_peak: conflict-free 16-B shared "
                                  "loads on every SM, this run)",
                     "ncu_min_proof": NCU_MIN7}

    cpu = None
    if not args.no_cpu_baseline and world == 1 and headline and os.path.exists(REF_DRIVER):
        small = [m for m in SAMPLE["masks"] if m["k"] <= 3]
        try:
            r = run_ref_sample(small, 1)
            cpu = {"value": r["value"], "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": f"the {len(small)} k<=3 stage_evals of the step, {r['leaves']} "
                             f"reference leaves in {r['wall_s']:.2f}s on one core",
                   "cpu": host_cpu(), "host_cores": os.cpu_count()}
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / max(1, args.steps),
        "higher_is_better": True, "scaling": "weak" if weak else "strong", "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic", "config": dict(CONFIG if headline else {"workload": WORKLOAD},
                                            l2="flushed between steps (256 MiB write)",
                                            parallelism=(f"every one of {world} GPU(s) runs its own "
                                                         f"copy of the sample (no collective)"
                                                         if weak else
                                                         f"sample masks dealt over {world} GPU(s)")
                                                        + "; full solve frontier sharded"),
        "same_config": headline,
        "time_to_best_plan_s": ttbp, "best_plan_iteration_time": best_plan,
        "full_solve": {"stage_eval_calls": searches_per_solve, "median_ms": ttbp * 1000.0,
                       "data_plane": plane,
                       # ranks whose search control blocks this rank mapped (CUDA IPC) for
                       # in-search incumbent / earliest-hit sharing
                       "peer_links": peer_links if world > 1 else None},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "timing": "host wall clock, create+sample+readback"},
        "gpu_launches": ctr["own_launches"],
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if peak else None, "traffic": dram_traffic_per_launch(),
                     "traffic_source": TRAFFIC_CSV,
                     "kernel": "k_search (k_search_fast_min / _first builds for this model)",
                     "peak_kind": peak_kind,
                     "algorithmic_bytes": "24*k B per last-level option screen (k option rows "
                                          "x 3 fp64, SURVEY.md 8d)",
                     "note": "branch-bound tree search; HBM is not the binding resource "
                             "(DESIGN.md)"},
        "roofline_smem": roofline_smem,
        "cpu_baseline": cpu,
        "evaluator": evaluator,
        "clocks": clk.summary(),
        "counters": ctr,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
