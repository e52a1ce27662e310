"""Device time of the cfg5 7-encoder stage_eval (the dominant stage of the solve) under knob
settings; every setting must return the same stage time and allocation.
usage: python tools/sweep7.py "don_tail=2 deep_after=16384" "don_tail=1" ..."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18710_b200 import mosaic  # noqa: E402

pl = mosaic.Planner.from_spec("cfg5", device=0)
pl.stage_eval([0, 1, 2])
base = None
DEFAULTS = {"don_depth": 3, "don_tail": 2, "deep_after": 16384, "don_period": 4,
            "backoff_ns": 2048, "don_depth_first": -1, "don_tail_first": -1, "tail_idle": 0, "tail_after": 256, "don_min_rest": 0, "local_handover": 1, "min_order": 4}
for setting in sys.argv[1:]:
    kv = dict(x.split("=") for x in setting.split())
    for k, v in {**DEFAULTS, **kv}.items():
        pl.set_tuning(**{k: float(v)})
    pl.clear_cache()
    pl.reset_counters()
    r = pl.stage_eval(list(range(7)))
    c = pl.counters()
    sig = (r.stage_time, [(e.module, e.option.dp_degree, e.option.quota_units, tuple(e.gpus))
                          for e in r.allocation.entries])
    if base is None:
        base = sig
    print(f"{setting:40s} device {c['device_ms']:8.1f} ms  same={sig == base}", flush=True)
