"""Bench sample and full cfg5 solve under share_all (W option-prefix shards per large search
in one launch on this device); results checked against the reference / unsharded run."""
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
for W in [int(x) for x in sys.argv[1:]] or [0, 2, 4, 8]:
    pl.set_tuning(share_all=W)
    best = 1e9
    for _ in range(6):
        pl.clear_cache()
        pl.reset_counters()
        r = pl.search(sets, times_only=True)
        best = min(best, pl.counters()["device_ms"])
    assert list(r) == want
    pl.clear_cache()
    pl.reset_counters()
    sol = pl.solve()
    print(f"share_all={W}: sample {best:.3f} ms, solve {pl.counters()['device_ms']:.1f} ms, plan "
          f"{sol.plan.predicted_iteration_time!r}", flush=True)
