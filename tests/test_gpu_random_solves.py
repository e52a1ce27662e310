"""GAHC solves of medium random instances (4-6 modules, 16-64 GPUs, L = 10) against the
reference's own solve(): plan and full trace (every round, candidate, gain, cache hit, prune,
stage_eval_calls, feasibility_calls) bit-identical.  This is the regime of shared walkers and
batched rounds (tests/golden/random_solves.json)."""
import os

import pytest

from conftest import GOLDEN, load_golden
from test_gpu_parity import check_plan, check_trace

pytestmark = pytest.mark.gpu
mosaic = pytest.importorskip("paper_2605_18710_b200.mosaic")


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "random_solves.json")),
                    reason="fixture not generated")
def test_random_solves_bit_identical():
    rows = load_golden("random_solves.json")
    assert len(rows) >= 20
    for g in rows:
        pl = mosaic.Planner.from_spec(g["args"][0], device=0)
        r = pl.solve()
        check_plan(r.plan, g)
        check_trace(r.trace, g)
        pl.close()
