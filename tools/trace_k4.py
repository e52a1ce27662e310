import sys, json
sys.path.insert(0, ".")
from paper_2605_18710_b200 import mosaic
pl = mosaic.Planner.from_spec("cfg5", device=0)
bits = [i for i in range(8) if 0x1d >> i & 1]
for _ in range(3):
    pl.clear_cache(); pl.stage_eval(bits)
pl.clear_cache(); pl.set_tuning(trace=3); pl.stage_eval(bits)
