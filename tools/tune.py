"""Search-engine knob experiments through the public tuning API (mosaic_gpu_set_tuning).

    python tools/tune.py cfg5 --mask 127 --knob don_depth=2 --knob don_period=8
    python tools/tune.py cfg5 --mask 127 --share 8        # per-rank shares of an 8-way shard
    python tools/tune.py cfg4 --solve                     # full GAHC solve

Prints one line per measurement: device ms of the search kernels, launches, result.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_18710_b200 import mosaic  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("spec")
    ap.add_argument("--levels", type=int, default=0)
    ap.add_argument("--mask", type=lambda s: int(s, 0), default=None)
    ap.add_argument("--solve", action="store_true")
    ap.add_argument("--min-at", type=float.fromhex, default=None,
                    help="one MIN search below this bound (hex), no restart")
    ap.add_argument("--knob", action="append", default=[])
    ap.add_argument("--share", type=int, default=1)
    a = ap.parse_args()
    pl = mosaic.Planner.from_spec(a.spec, quota_levels=a.levels)
    knobs = dict(k.split("=") for k in a.knob)
    pl.set_tuning(**{k: float(v) for k, v in knobs.items()})
    shares = range(a.share) if a.share > 1 else [None]
    for r in shares:
        if r is not None:
            pl.set_tuning(share_rank=r, share_world=a.share)
        pl.reset_counters()
        t0 = time.time()
        if a.solve:
            out = pl.solve().plan.predicted_iteration_time
        elif a.min_at is not None:
            mods = [i for i in range(64) if a.mask >> i & 1]
            out = pl.stage_min(mods, a.min_at, restart=False)
        else:
            mods = [i for i in range(64) if a.mask >> i & 1]
            res = pl.stage_eval(mods)
            out = None if res is None else res.stage_time
        c = pl.counters()
        print(f"{a.spec} knobs={knobs} share={r}/{a.share}: {out!r} "
              f"ksearch_ms={c['ksearch_ms']:.3f} launches={c['ksearch_launches']} "
              f"wall={1e3 * (time.time() - t0):.1f}ms", flush=True)


if __name__ == "__main__":
    main()
