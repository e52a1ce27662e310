"""Time to best plan for every BASELINE config: ours (wall and device events, launches per
solve) and, where oracle/_ref exists, the reference solve() on one core of this host."""
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18710_b200 import mosaic  # noqa: E402

gold = json.load(open(os.path.join(ROOT, "tests", "golden", "configs.json")))
for w in ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]:
    pl = mosaic.Planner.from_spec(w, device=0)
    reps = 3 if w == "cfg5" else 50
    for _ in range(3):
        r = pl.solve()
    walls, devs = [], []
    pl.reset_counters()
    for _ in range(reps):
        t0 = time.perf_counter()
        pl.mark(0)
        r = pl.solve()
        pl.mark(1)
        devs.append(pl.marked_ms())
        walls.append(1e3 * (time.perf_counter() - t0))
    c = pl.counters()
    ok = ""
    if w in gold and "solve" in gold[w]:
        ok = "plan==ref" if r.plan.predicted_iteration_time == float.fromhex(
            gold[w]["solve"]["iteration_time"]) else "PLAN DIFFERS"
    print(f"{w}: wall median {statistics.median(walls):.3f} ms, device {statistics.median(devs):.3f} ms, "
          f"launches/solve {c['own_launches'] / reps:.1f}, stage_evals {r.trace.stage_eval_calls}, "
          f"searches {r.trace.gpu_searches} {ok}", flush=True)
    pl.close()
drv = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
if os.path.exists(drv):
    for w in ["cfg1", "cfg2", "cfg3", "cfg4"]:
        d = json.loads(subprocess.run(["taskset", "-c", "0", drv, w, "solve", "reps=20"],
                                      capture_output=True, text=True).stdout)
        t = sorted(d.get("times", []))
        print(f"{w}: reference solve() one core median {1e3 * t[len(t) // 2]:.3f} ms", flush=True)
