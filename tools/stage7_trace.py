"""Per-search trace of the cfg5 7-encoder stage_eval (the dominant stage of the solve)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18710_b200 import mosaic  # noqa: E402

pl = mosaic.Planner.from_spec("cfg5", device=0)
pl.stage_eval([0, 1, 2])
pl.set_tuning(trace=int(sys.argv[1]) if len(sys.argv) > 1 else 1)
r = pl.stage_eval(list(range(7)))
print(r.stage_time.hex(), r.stats, file=sys.stderr)
