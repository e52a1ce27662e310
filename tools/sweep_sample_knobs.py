"""Bench-sample (29 cfg5 stage_evals, one batch) device time under knob settings.
usage: python tools/sweep_sample_knobs.py small_tree=2e5,1e5,3e4 [trace]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18710_b200 import mosaic  # noqa: E402

S = json.load(open(os.path.join(ROOT, "tests", "golden", "cfg5_sample.json")))
sets = [[i for i in range(8) if m["mask"] >> i & 1] for m in S["masks"]]
want = [float.fromhex(m["t"]) for m in S["masks"]]
pl = mosaic.Planner.from_spec("cfg5", device=0)
for spec in sys.argv[1:]:
    if spec == "trace":
        continue
    name, vals = spec.split("=")
    for v in vals.split(","):
        pl.set_tuning(**{name: float(v)})
        best = 1e9
        for rep in range(6):
            pl.clear_cache()
            pl.reset_counters()
            r = pl.search(sets, times_only=True)
            c = pl.counters()
            best = min(best, c["device_ms"])
        assert list(r) == want, "stage times differ from the reference"
        print(f"{name}={v}: device {best:.3f} ms, launches {c['ksearch_launches']}", flush=True)
