"""Per-launch trace (trace=2) and per-search trace (trace=1) of the small-config solves."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18710_b200 import mosaic  # noqa: E402

for spec in sys.argv[1:] or ["cfg1", "cfg2"]:
    pl = mosaic.Planner.from_spec(spec, device=0)
    for _ in range(5):
        pl.clear_cache()
        pl.solve()
    best = 1e9
    for _ in range(20):
        pl.clear_cache()
        t0 = time.perf_counter()
        pl.solve()
        best = min(best, time.perf_counter() - t0)
    print(f"== {spec}: best solve wall {best*1e3:.3f} ms", file=sys.stderr, flush=True)
    pl.clear_cache()
    pl.set_tuning(trace=2)
    pl.solve()
    pl.clear_cache()
    pl.set_tuning(trace=1)
    pl.solve()
    pl.set_tuning(trace=0)
