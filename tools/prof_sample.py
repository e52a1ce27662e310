"""ncu target: one batched cfg5 sample (29 stage_evals) after a warm-up batch."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18710_b200 import mosaic  # noqa: E402

S = json.load(open(os.path.join(ROOT, "tests", "golden", "cfg5_sample.json")))
sets = [[i for i in range(8) if m["mask"] >> i & 1] for m in S["masks"]]
pl = mosaic.Planner.from_spec("cfg5", device=0)
pl.search(sets, times_only=True)
pl.reset_counters()
pl.search(sets, times_only=True)
print(pl.counters())
