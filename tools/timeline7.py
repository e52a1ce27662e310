"""Busy-walker timeline (trace=3) of the 7-encoder cfg5 stage_eval's big launches."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18710_b200 import mosaic  # noqa: E402

pl = mosaic.Planner.from_spec("cfg5", device=0)
pl.stage_eval([0, 1, 2])
for kv in sys.argv[1:]:
    k, v = kv.split("=")
    pl.set_tuning(**{k: float(v)})
pl.set_tuning(trace=3)
r = pl.stage_eval(list(range(7)))
print(r.stage_time.hex(), r.stats, file=sys.stderr)
