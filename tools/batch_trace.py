"""Trace of the batched bench sample: one stderr line per search of every wave."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18710_b200 import mosaic  # noqa: E402

S = json.load(open(os.path.join(ROOT, "tests", "golden", "cfg5_sample.json")))
t0 = time.perf_counter()
pl = mosaic.Planner.from_spec("cfg5", device=0)
t1 = time.perf_counter()
sets = [[i for i in range(8) if m["mask"] >> i & 1] for m in S["masks"]]
pl.search(sets)
t2 = time.perf_counter()
pl.search(sets)
t3 = time.perf_counter()
t5 = time.perf_counter()
p2 = mosaic.Planner.from_spec("cfg5", device=0)
t6 = time.perf_counter()
p2.search(sets)
t7 = time.perf_counter()
p2.close()
t8 = time.perf_counter()
print(f"create {1e3*(t1-t0):.2f} ms, first batch {1e3*(t2-t1):.2f} ms, second {1e3*(t3-t2):.2f} ms"
      f"; warm create {1e3*(t6-t5):.2f} ms, its first batch {1e3*(t7-t6):.2f} ms, close "
      f"{1e3*(t8-t7):.2f} ms", flush=True)
for k, v in [a.split("=") for a in sys.argv[1:]]:
    pl.set_tuning(**{k: float(v)})
pl.set_tuning(trace=1)
t4 = time.perf_counter()
pl.search(sets)
print(f"traced batch {1e3*(time.perf_counter()-t4):.2f} ms", flush=True)
