"""ncu target: the launches of one cfg1 solve (after warm-up solves)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18710_b200 import mosaic  # noqa: E402

pl = mosaic.Planner.from_spec(sys.argv[1] if len(sys.argv) > 1 else "cfg1", device=0)
for _ in range(3):
    pl.solve()
pl.reset_counters()
pl.set_tuning(trace=1)
pl.solve()
print(pl.counters())
