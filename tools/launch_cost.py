"""Per-launch host / stream / kernel time of the batched bench sample (trace=2)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18710_b200 import mosaic  # noqa: E402

S = json.load(open(os.path.join(ROOT, "tests", "golden", "cfg5_sample.json")))
sets = [[i for i in range(8) if m["mask"] >> i & 1] for m in S["masks"]]
pl = mosaic.Planner.from_spec("cfg5", device=0)
for _ in range(3):
    pl.search(sets, times_only=True)
pl.set_tuning(trace=2)
pl.search(sets, times_only=True)
