"""Beyond 128 GPUs (G = 256, 512): stage_eval of every one- and two-module set and the full
GAHC solve against the reference (tests/golden/large_clusters.json), bit for bit."""
import pytest

from conftest import alloc_tuples, hexf, load_golden, result_tuples
from test_gpu_parity import check_plan, check_trace

pytestmark = pytest.mark.gpu
mosaic = pytest.importorskip("paper_2605_18710_b200.mosaic")


def test_large_clusters_stage_eval_and_solve():
    rows = load_golden("large_clusters.json")
    by = {}
    for r in rows:
        by.setdefault(r["args"][0], []).append(r)
    for inst, rs in by.items():
        pl = mosaic.Planner.from_spec(inst, device=0)
        for r in rs:
            if r["op"] == "stage":
                g = pl.stage_eval([i for i in range(64) if r["mask"] >> i & 1])
                assert (g is not None) == bool(r["feasible"])
                if g is not None:
                    assert g.stage_time == hexf(r["t"]), (inst, r["mask"])
                    assert result_tuples(g) == alloc_tuples(r["alloc"]), (inst, r["mask"])
                    assert g.stats.feasibility_calls == r["feasibility_calls"]
            else:
                s = pl.solve()
                check_plan(s.plan, r)
                check_trace(s.trace, r)
        pl.close()
