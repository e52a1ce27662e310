"""Pin the cfg5 headline plan: replay the GPU's GAHC trajectory through the REAL reference.

The reference planner does not finish the cfg5 solve in 90 min, but every
stage_eval it would issue is deterministic and independent, so the plan is pinned mask by
mask:

  1. ``gpu``  (on a B200, through the product):  solve each shape, dump the plan, the
     GAHC rounds and every EvalCache entry with its probe sequence (tau, feasible) to
     ``tests/golden/trajectory_gpu.json``.  The GAHC decisions only depend on the stage
     times of the masks in the cache, so if the reference agrees on every cached mask it
     makes the same decisions and returns the same plan.
  2. ``ref``  (here, where /root/reference exists):  run ``oracle/_ref/ref_driver SPEC
     stage MASK`` (stage_eval.hpp:302) for every cached mask, all cores in parallel,
     cheapest first, each under a wall-clock cap; results stream into
     ``tests/golden/trajectory_ref.jsonl`` as they finish.  For a mask that does not finish
     under the cap, the two probes that decide its result are run on their own:
       * ``feas MASK tau_last_ok`` — the last successful probe (cheap: feasible), which
         pins the returned allocation bit for bit (stage_eval returns the first leaf of
         the last successful probe, stage_eval.hpp:372-381);
       * ``feas MASK tau_conf``   — the final confirmation probe at t_best*(1-1e-9)
         (the expensive infeasibility proof), under its own cap.
     Also the full reference ``solve`` of each intermediate shape (preset:ofasys:8:64).
  3. ``status`` — which masks / probes are pinned, with their CPU times.

Usage:
    python tests/golden/make_cfg5_trajectory.py gpu            # on the GPU box
    python tests/golden/make_cfg5_trajectory.py ref --jobs 6 --cap 36000
    python tests/golden/make_cfg5_trajectory.py status
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
GPU_OUT = os.path.join(HERE, "trajectory_gpu.json")
REF_OUT = os.path.join(HERE, "trajectory_ref.jsonl")

# (spec, quota levels): the headline cfg5 and two intermediate shapes of it
SHAPES = [("cfg5", 32), ("preset:ofasys:8:64", 10), ("preset:ofasys:8:64", 32)]


def _hex(x: float) -> str:
    return float(x).hex()


def _alloc(st) -> list:
    return [{"m": e.module, "d": e.option.dp_degree, "u": e.option.quota_units,
             "gpus": list(e.gpus)} for e in st.entries]


def gpu(dst: str | None = None) -> None:
    sys.path.insert(0, ROOT)
    from paper_2605_18710_b200 import mosaic

    out = {}
    for spec, L in SHAPES:
        pl = mosaic.Planner.from_spec(spec, quota_levels=L, device=0)
        t0 = time.time()
        r = pl.solve()
        wall = time.time() - t0
        plan = r.plan
        cache = []
        for mask, res, probes in pl.eval_cache():
            cache.append({"mask": mask, "k": bin(mask).count("1"), "t": _hex(res.stage_time),
                          "t_dec": res.stage_time, "alloc": _alloc(res.allocation),
                          "feasibility_calls": res.stats.feasibility_calls,
                          "probes": [[_hex(t), int(ok)] for t, ok in probes]})
        out[f"{spec}@L{L}"] = {
            "spec": spec, "levels": L, "wall_s": wall,
            "iteration_time": _hex(plan.predicted_iteration_time),
            "iteration_time_dec": plan.predicted_iteration_time,
            "stages": [{"t": _hex(t), "alloc": _alloc(s)}
                       for s, t in zip(plan.stages, plan.predicted_stage_times)],
            "rounds": [{"x": rd.chosen_x, "y": rd.chosen_y, "gain": _hex(rd.applied_gain),
                        "cands": [{"x": c.mask_x, "y": c.mask_y, "pruned": int(c.pruned),
                                   "hit": int(c.cache_hit), "gain": _hex(c.gain)}
                                  for c in rd.candidates]} for rd in r.trace.rounds],
            "stage_eval_calls": r.trace.stage_eval_calls,
            "feasibility_calls": r.trace.feasibility_calls,
            "cache": cache,
        }
        print(f"{spec}@L{L}: {plan.predicted_iteration_time!r} in {wall:.2f}s, "
              f"{len(cache)} cached masks", flush=True)
        pl.close()
    dst = dst or GPU_OUT
    with open(dst, "w") as f:
        json.dump(out, f, indent=0)
    print(f"wrote {dst}")


_lock = threading.Lock()


def _done_keys() -> set:
    keys = set()
    if os.path.exists(REF_OUT):
        with open(REF_OUT) as f:
            for line in f:
                try:
                    d = json.loads(line)
                except json.JSONDecodeError:
                    continue
                keys.add(d["key"])
    return keys


def _run(key: str, args: list[str], cap: float) -> dict:
    t0 = time.time()
    try:
        p = subprocess.run([DRIVER, *args], capture_output=True, text=True, timeout=cap)
        rec = {"key": key, "args": args, "wall_s": time.time() - t0, "rc": p.returncode}
        if p.returncode in (0, 3):
            rec["out"] = json.loads(p.stdout)
        else:
            rec["stderr"] = p.stderr[-2000:]
    except subprocess.TimeoutExpired:
        rec = {"key": key, "args": args, "wall_s": time.time() - t0, "timeout": cap}
    with _lock:
        with open(REF_OUT, "a") as f:
            f.write(json.dumps(rec, separators=(",", ":")) + "\n")
    print(f"[{time.strftime('%H:%M:%S')}] {key}: "
          f"{'TIMEOUT' if 'timeout' in rec else 'rc=%d' % rec['rc']} {rec['wall_s']:.1f}s",
          flush=True)
    return rec


def _probe_jobs(name: str, sh: dict, c: dict) -> list:
    """The two probes that decide a mask's stage_eval result (see module docstring)."""
    lv = f"levels={sh['levels']}"
    mask = str(c["mask"])
    ok = [float.fromhex(t) for t, o in c["probes"] if o]
    out = [(c["k"] - 10.0, f"{name}|feas_last_ok|{mask}",
            [sh["spec"], "feas", mask, repr(ok[-1]), lv])]
    t_last, ok_last = c["probes"][-1]
    if not ok_last:
        out.append((c["k"] + 0.5, f"{name}|feas_conf|{mask}",
                    [sh["spec"], "feas", mask, repr(float.fromhex(t_last)), lv]))
    return out


def ref(jobs: int, cap: float, probe_k: int, only: str | None = None) -> None:
    with open(GPU_OUT) as f:
        traj = json.load(f)
    done = _done_keys()
    todo = []
    for name, sh in traj.items():
        if only and name != only:
            continue
        lv = f"levels={sh['levels']}"
        for c in sh["cache"]:
            todo.append((c["k"], f"{name}|stage|{c['mask']}",
                         [sh["spec"], "stage", str(c["mask"]), lv]))
            if c["k"] >= probe_k:
                todo += _probe_jobs(name, sh, c)
        if sh["spec"] != "cfg5":
            todo.append((4.5, f"{name}|solve", [sh["spec"], "solve", lv]))
    todo = [j for j in sorted(todo, key=lambda j: j[0]) if j[1] not in done]
    if only:  # a second runner for one shape: leave its full solve to the main runner
        todo = [j for j in todo if not j[1].endswith("|solve")]
    print(f"{len(todo)} jobs ({len(done)} already recorded), {jobs} workers, cap {cap:.0f}s",
          flush=True)
    with cf.ThreadPoolExecutor(jobs) as ex:
        list(ex.map(lambda j: _run(j[1], j[2], cap), todo))


def status() -> None:
    with open(GPU_OUT) as f:
        traj = json.load(f)
    recs = {}
    if os.path.exists(REF_OUT):
        with open(REF_OUT) as f:
            for line in f:
                d = json.loads(line)
                recs[d["key"]] = d
    for name, sh in traj.items():
        print(f"== {name}: GPU plan {sh['iteration_time_dec']!r}")
        for c in sh["cache"]:
            key = f"{name}|stage|{c['mask']}"
            r = recs.get(key)
            if r is None:
                st = "pending"
                for p in ("feas_last_ok", "feas_conf"):
                    q = recs.get(f"{name}|{p}|{c['mask']}")
                    if q:
                        ok = ("out" in q and float.fromhex(q["out"].get("t", "0x0p+0")) ==
                              float.fromhex(c["t"])) if p == "feas_last_ok" else "out" in q
                        st += f"; {p} " + (f"> {q['timeout']:.0f}s" if "timeout" in q else
                                          f"{q['wall_s']:.1f}s" + (" MATCH" if ok else " DIFF"))
            elif "timeout" in r:
                st = f"> {r['timeout']:.0f}s"
                for p in ("feas_last_ok", "feas_conf"):
                    q = recs.get(f"{name}|{p}|{c['mask']}")
                    if q:
                        st += f"; {p} " + (f"> {q['timeout']:.0f}s" if "timeout" in q
                                           else f"{q['wall_s']:.1f}s")
            else:
                o = r.get("out", {})
                same = ("t" in o and float.fromhex(o["t"]) == float.fromhex(c["t"])
                        and o.get("alloc") == c["alloc"])
                st = f"{r['wall_s']:.1f}s {'MATCH' if same else 'DIFF'}"
            print(f"  k={c['k']} mask={c['mask']:#x}: {st}")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("phase", choices=["gpu", "ref", "status"])
    ap.add_argument("out", nargs="?")
    ap.add_argument("--jobs", type=int, default=max(1, (os.cpu_count() or 2) - 2))
    ap.add_argument("--cap", type=float, default=36000.0)
    ap.add_argument("--only", help="restrict to one shape (e.g. preset:ofasys:8:64@L10)")
    ap.add_argument("--probe-k", type=int, default=5,
                    help="also pin the deciding probes of masks with >= this many modules")
    a = ap.parse_args()
    if a.phase == "gpu":
        gpu(a.out)
    elif a.phase == "ref":
        ref(a.jobs, a.cap, a.probe_k, a.only)
    else:
        status()
