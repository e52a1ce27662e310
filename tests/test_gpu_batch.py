"""Batched stage search (mosaic_gpu_search, A1): many module sets advance together, one
launch per wave of device searches.  Results must be identical to the one-at-a-time path
and to the reference's own stage_eval / ExactStageSolver outputs."""
import json
import os

import pytest

from conftest import GOLDEN, alloc_tuples, hexf, load_golden, result_tuples

pytestmark = pytest.mark.gpu

mosaic = pytest.importorskip("paper_2605_18710_b200.mosaic")


def bits(m):
    return [i for i in range(64) if m >> i & 1]


def _ref_records():
    out = {}
    with open(os.path.join(GOLDEN, "trajectory_ref.jsonl")) as f:
        for line in f:
            d = json.loads(line)
            if "|stage|" in d["key"] and d.get("rc") == 0 and d["key"].startswith("cfg5@L32"):
                out[int(d["key"].rsplit("|", 1)[1])] = d["out"]
    return out


def test_cfg5_sample_batch_equals_reference():
    sample = load_golden("cfg5_sample.json")["masks"]
    ref = _ref_records()
    pl = mosaic.Planner.from_spec("cfg5", device=0)
    n0 = pl.launch_count()
    rs = pl.search([bits(m["mask"]) for m in sample])
    launches = pl.launch_count() - n0
    for m, r in zip(sample, rs):
        assert r.stage_time == hexf(m["t"]), m["mask"]
        assert r.stats.feasibility_calls == m["feasibility_calls"], m["mask"]
        if m["mask"] in ref:
            assert result_tuples(r) == alloc_tuples(ref[m["mask"]]["alloc"]), m["mask"]
    # one launch per wave: far fewer than one per device search
    assert launches <= max(r.stats.gpu_searches for r in rs) + 2, launches
    pl.close()


@pytest.mark.parametrize("spec", ["cfg3", "cfg4", "random:7:5:16"])
def test_batch_equals_sequential(spec):
    pl = mosaic.Planner.from_spec(spec, device=0)
    n = pl.n_modules
    sets = [[i] for i in range(n)] + [[i, j] for i in range(n) for j in range(i + 1, n)]
    sets += [list(range(min(n, 3))), list(range(n))]
    batch = pl.search(sets)
    seq = [pl.stage_eval(s) for s in sets]
    for s, b, q in zip(sets, batch, seq):
        assert (b is None) == (q is None), s
        if b is not None:
            assert b.stage_time == q.stage_time and result_tuples(b) == result_tuples(q), s
            assert b.stats.feasibility_calls == q.stats.feasibility_calls
    ex_b = pl.search(sets[:6], exact=True)
    ex_q = [pl.exact_stage(s) for s in sets[:6]]
    for s, b, q in zip(sets, ex_b, ex_q):
        assert (b is None) == (q is None), s
        if b is not None:
            assert b.stage_time == q.stage_time and result_tuples(b) == result_tuples(q), s
    pl.close()


def test_solve_launches_fewer_than_searches():
    # GAHC rounds batch their candidates: launches per solve well below device searches
    for spec in ("cfg3", "cfg4"):
        pl = mosaic.Planner.from_spec(spec, device=0)
        pl.reset_counters()
        r = pl.solve()
        c = pl.counters()
        assert c["ksearch_launches"] < r.trace.gpu_searches, (spec, c, r.trace.gpu_searches)
        pl.close()


def test_contexts_of_different_sizes_interleave():
    # kernel attributes (dynamic shared memory) are process-wide: a small problem's context
    # must not break a larger one created earlier (regression: 'invalid argument' launches)
    big = mosaic.Planner.from_spec("cfg5", device=0)
    small = mosaic.Planner.from_spec("cfg3", device=0)
    a = big.stage_eval([0, 1, 2, 3])
    small.solve()
    b = big.stage_eval([0, 1, 2, 3])
    assert a.stage_time == b.stage_time
    small.close()
    big.close()
