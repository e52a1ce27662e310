"""compute-sanitizer target: stage_evals and solves of cfg3 / cfg4 (batched and single
searches, MIN and FIRST, solo and shared walkers) plus the K1 evaluator."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tools")]
import numpy as np  # noqa: E402

from evalgen import random_allocations  # noqa: E402
from paper_2605_18710_b200 import mosaic  # noqa: E402

for spec in ("cfg3", "cfg4"):
    pl = mosaic.Planner.from_spec(spec, device=0)
    r = pl.solve()
    n = pl.n_modules
    pl.search([[i, j] for i in range(n) for j in range(i + 1, n)])
    pl.exact_stage(list(range(min(n, 3))))
    ent, gpus, off = random_allocations(pl, 2000, seed=1)
    st = np.zeros(len(off) - 1)
    pl.evaluate(ent, gpus, off, st)
    print(spec, r.plan.predicted_iteration_time, flush=True)
    pl.close()
