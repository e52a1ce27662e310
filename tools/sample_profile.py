"""Per-mask wall time / device searches of the bench sample (cfg5 k<=4 stage_evals)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18710_b200 import mosaic  # noqa: E402

S = json.load(open(os.path.join(ROOT, "tests", "golden", "cfg5_sample.json")))
pl = mosaic.Planner.from_spec("cfg5", device=0)
if len(sys.argv) > 1:
    pl.set_tuning(trace=1)
for rep in range(2):
    pl.clear_cache()
    tot = 0.0
    for m in S["masks"]:
        bits = [i for i in range(8) if m["mask"] >> i & 1]
        t0 = time.perf_counter()
        r = pl.stage_eval(bits)
        dt = time.perf_counter() - t0
        tot += dt
        if rep == 1:
            print(f"mask {m['mask']:#04x} k={m['k']} {dt*1e3:8.3f} ms searches={r.stats.gpu_searches} "
                  f"probes={r.stats.feasibility_calls} ref={m['cpu_s']:.2f}s", flush=True)
    print(f"total {tot*1e3:.2f} ms")
