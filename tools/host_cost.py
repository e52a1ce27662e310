"""Host vs device time of the batched bench sample (trace line of Planner::run_jobs)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18710_b200 import mosaic  # noqa: E402

S = json.load(open(os.path.join(ROOT, "tests", "golden", "cfg5_sample.json")))
sets = [[i for i in range(8) if m["mask"] >> i & 1] for m in S["masks"]]
pl = mosaic.Planner.from_spec("cfg5", device=0)
for _ in range(3):
    pl.search(sets, times_only=True)
pl.set_tuning(trace=3)
for _ in range(3):
    t0 = time.perf_counter()
    pl.search(sets, times_only=True)
    print(f"python wall {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr, flush=True)
for _ in range(3):
    t0 = time.perf_counter()
    p2 = mosaic.Planner.from_spec("cfg5", device=0)
    t1 = time.perf_counter()
    p2.search(sets, times_only=True)
    t2 = time.perf_counter()
    p2.close()
    print(f"e2e: create {1e3 * (t1 - t0):.3f} ms, sample {1e3 * (t2 - t1):.3f} ms, close "
          f"{1e3 * (time.perf_counter() - t2):.3f} ms", file=sys.stderr, flush=True)
