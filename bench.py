"""bench.py — candidate plans evaluated/sec and time-to-best-plan, B200 vs CPU reference.

Workload (BASELINE.json configs[4], the config the metric's 1/2/4/8-B200 sharding is
quoted on): cfg5 = omni-modal 8-module MM (7 encoders -> backbone, profiler.hpp:212-285)
on 128 modeled GPUs, quota granularity 1/32, GAHC search (solver.hpp:157-289) to the
best plan.  One STEP = one full solve(): every stage_eval of every GAHC round, each a
tau-probe replay whose feasibility searches run on the GPU.

  value  = complete stage allocations scored on the device (leaves) / device time of the
           timed steps (CUDA events on the library's own stream), whole job over ranks.
  e2e    = the same metric through the C ABI with HOST buffers: mosaic_gpu_create from
           host surface tables (option tables copied H2D) + mosaic_gpu_solve + plan read
           back, per step, host wall clock.
  ms_per_step = time to the best plan (device-timed).

--impl reference runs the reference's own CPU planner (oracle/_ref, the unmodified
headers compiled by oracle/Makefile) on a bounded sample of the same workload: the
stage_eval calls GAHC issues in its first two rounds on cfg5 (all singletons and all
encoder pairs), which is where the reference spends its first ~seconds; the full cfg5
solve does not finish on the CPU (>90 min).
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
DESCR = {
    "cfg1": "cfg1: CLIP ViT-L/14 + text encoder, 8 modeled GPUs, exhaustive-size stage search",
    "cfg2": "cfg2: LLaVA ViT + projector + 7B LLM, 16 modeled GPUs, quota 1/8, GAHC",
    "cfg3": "cfg3: Qwen3-VL vision + text + deepstack + LLM, 32 modeled GPUs, GAHC",
    "cfg4": "cfg4: omni-6 (3 encoders -> LLM -> 2 decoders), 64 modeled GPUs, GAHC",
    "cfg5": "cfg5: omni-modal 8-module MM, 128 modeled GPUs, quota 1/32, GAHC to best plan",
}
METRIC = "candidate plans evaluated/sec (cfg5 GAHC solve to best plan)"
UNIT = "plans/s"
REF_DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver_instr")
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


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
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
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


def cpu_sample_masks() -> list[int]:
    """GAHC round 0 + round 1 stage_evals on cfg5: 8 singletons + 21 encoder pairs."""
    masks = [1 << m for m in range(8)]
    for a in range(7):
        for b in range(a + 1, 7):
            masks.append((1 << a) | (1 << b))
    return masks


def run_cpu_sample(parallel: int) -> dict:
    """Reference CPU planner on the bounded sample; leaves counted by the instrumented
    build (verify_complete, stage_eval.hpp:254)."""
    if not os.path.exists(REF_DRIVER):
        raise FileNotFoundError(f"{REF_DRIVER} missing (build with make -C oracle ref)")
    masks = cpu_sample_masks()
    t0 = time.perf_counter()
    procs = []
    results = []
    pending = list(masks)
    while pending or procs:
        while pending and len(procs) < parallel:
            m = pending.pop(0)
            cmd = [REF_DRIVER, WORKLOAD, "stage", str(m)]
            if parallel == 1 and shutil_which("taskset"):
                cmd = ["taskset", "-c", "0"] + cmd
            procs.append(subprocess.Popen(cmd, stdout=subprocess.PIPE, text=True))
        p = procs.pop(0)
        out, _ = p.communicate()
        results.append(json.loads(out))
    wall = time.perf_counter() - t0
    leaves = sum(r.get("leaves", 0) for r in results)
    return {"leaves": leaves, "wall_s": wall, "stage_evals": len(masks),
            "value": leaves / wall if wall > 0 else 0.0}


def shutil_which(x: str):
    from shutil import which
    return which(x)


def host_cpu() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def reference_arm(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    ncores = os.cpu_count() or 1
    par = max(1, min(ncores, len(cpu_sample_masks())))
    for _ in range(args.warmup):
        run_cpu_sample(par)
    vals, walls, leaves = [], [], 0
    for _ in range(args.steps):
        r = run_cpu_sample(par)
        vals.append(r["value"])
        walls.append(r["wall_s"])
        leaves += r["leaves"]
    total_wall = sum(walls)
    value = leaves / total_wall if total_wall else 0.0
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * total_wall / max(1, args.steps), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD + " (bounded sample: GAHC rounds 0-1 stage_evals, "
                   "8 singletons + 21 encoder pairs)", "modeled_gpus": 128,
                   "quota_levels": 32, "modules": 8},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": par, "kind": "reference",
                         "sample": "29 stage_eval calls of cfg5 GAHC rounds 0-1, one process "
                                   "per stage_eval (harness-parallel; the reference is "
                                   "single-threaded)", "cpu": host_cpu(),
                         "host_cores": ncores},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "time_to_best_plan_s": None,
        "note": "the reference does not finish the full cfg5 solve (>90 min, SURVEY.md §6)",
    }
    print(json.dumps(line), flush=True)


N_EVAL = 1 << 20  # allocations per evaluator step


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
    k_ms = s["kernel_ms"] / max(1, s["launches"])
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
            "kernel_ms": k_ms,
            "e2e": {"value": n / e2e_s, "unit": "allocations/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": n * 8, "timing": "host wall clock, pinned host arrays"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if peak else None, "traffic": None,
                         "kernel": "k_evaluate (eval.cu)", "peak_kind": peak_kind,
                         "algorithmic_bytes": "per allocation 16 B (offset + stage time) + "
                                              "32 B per entry + 4 B per GPU id"},
            "data": "synthetic: random module subsets of cfg5, candidate options, "
                    "windows of d consecutive GPUs; inputs > L2, L2 flushed between steps"}


TRAFFIC_CSV = "profiles/r1_dram_cfg5_solve.csv"


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
    ap.add_argument("--no-evaluator", action="store_true", help="skip the K1 evaluator leg")
    ap.add_argument("--workload", default="cfg5", help="cfg1..cfg5 (default cfg5)")
    ap.add_argument("--dist-backend", default="nccl",
                    help="nccl (default); gloo lets several ranks share one GPU for testing")
    ap.add_argument("--same-device", action="store_true",
                    help="every rank uses cuda:0 (sharding test on a single GPU)")
    args = ap.parse_args()
    if args.impl == "reference":
        reference_arm(args)
        return

    import torch
    import torch.distributed as dist

    global WORKLOAD
    WORKLOAD = args.workload
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

    # ---- device-resident run: tables already in HBM, time the solve only ----
    pl = mosaic.Planner.from_spec(WORKLOAD, device=local)
    res_g, res_l, res_n = pl.gpu_count, pl.quota_levels, pl.n_modules
    if world > 1:
        pl.set_shard(rank, world, allgather_bytes)
    for _ in range(args.warmup):
        res = pl.solve()
    barrier()
    pl.reset_counters()
    dev_ms, leaves, plans = [], 0, []
    with Clocks(local) as clk:
        for _ in range(args.steps):
            flush_l2(torch, dev)
            barrier()
            pl.mark(0)
            res = pl.solve()
            pl.mark(1)
            dev_ms.append(pl.marked_ms())
            leaves += res.trace.leaves
            plans.append(res.plan.predicted_iteration_time)
        barrier()
    ctr = pl.counters()
    t_local = sum(dev_ms)
    if world > 1:
        tt = torch.tensor([t_local, float(leaves)], dtype=torch.float64, device=comm_dev)
        mx = tt[:1].clone()
        sm = tt[1:].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        t_max, leaves_all = float(mx[0]), float(sm[0])
    else:
        t_max, leaves_all = t_local, float(leaves)
    value = leaves_all / (t_max / 1000.0) if t_max > 0 else 0.0

    # ---- e2e through the C ABI with host buffers (create + solve + read back) ----
    e2e_s, e2e_leaves, h2d, d2h = 0.0, 0, 0, 0
    for i in range(args.steps):
        barrier()
        t0 = time.perf_counter()
        p2 = mosaic.Planner.from_spec(WORKLOAD, device=local)
        if world > 1:
            p2.set_shard(rank, world, allgather_bytes)
        r2 = p2.solve()
        _ = [(e.module, e.gpus) for st in r2.plan.stages for e in st.entries]
        c2 = p2.counters()
        p2.close()
        barrier()
        e2e_s += time.perf_counter() - t0
        e2e_leaves += r2.trace.leaves
        h2d, d2h = c2["h2d_bytes"], c2["d2h_bytes"]
    e2e_value = e2e_leaves * world / e2e_s if e2e_s > 0 else 0.0

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (k_search) ----
    # traffic: dram__bytes_read.sum + dram__bytes_write.sum per k_search launch, from the
    # committed ncu capture of the same cfg5 solve (profiles/)
    peak, peak_kind = peaks()
    ks_ms = ctr["ksearch_ms"]
    ks_n = max(1, ctr["ksearch_launches"])
    alg_bytes = ctr.get("alg_bytes", 0)
    avg_launch_s = ks_ms / ks_n / 1000.0
    achieved = (alg_bytes / ks_n) / avg_launch_s / 1e9 if avg_launch_s > 0 else 0.0
    traffic = dram_traffic_per_launch() if WORKLOAD == "cfg5" else None

    evaluator = None if args.no_evaluator else evaluator_leg(pl, torch, dev, args.steps,
                                                              args.warmup, peak, peak_kind)

    cpu = None
    if not args.no_cpu_baseline and os.path.exists(REF_DRIVER):
        try:
            r = run_cpu_sample(1)
            cpu = {"value": r["value"], "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": f"{r['stage_evals']} stage_eval calls of cfg5 GAHC rounds 0-1 "
                             f"(8 singletons + 21 encoder pairs), {r['leaves']} leaves in "
                             f"{r['wall_s']:.2f}s, pinned to one core",
                   "cpu": host_cpu(), "host_cores": os.cpu_count()}
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / max(1, args.steps),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": DESCR.get(WORKLOAD, WORKLOAD), "modeled_gpus": res_g,
                   "quota_levels": res_l, "modules": res_n,
                   "l2": "flushed between steps (256 MiB write)",
                   "parallelism": f"frontier+round sharding over {world} GPU(s)"},
        "time_to_best_plan_s": t_max / 1000.0 / max(1, args.steps),
        "best_plan_iteration_time": plans[-1],
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "timing": "host wall clock, create+solve+readback"},
        "gpu_launches": ctr["own_launches"],
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if peak else None, "traffic": traffic,
                     "traffic_source": TRAFFIC_CSV if traffic is not None else None,
                     "kernel": "k_search (k_search_fast_min / _first builds for this model)",
                     "peak_kind": peak_kind,
                     "algorithmic_bytes": "24*k B per scored leaf (k option rows x 3 fp64, "
                                          "SURVEY.md 8d)",
                     "note": "integer/branch-bound tree search; HBM is not the binding "
                             "resource (see DESIGN.md)"},
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
