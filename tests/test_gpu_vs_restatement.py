"""GPU vs the C restatement (oracle/mosaic_oracle.c, itself pinned to the real reference by
tests/test_oracle_restatement.py), on instances generated at test time: larger G and other
quota granularities than the golden fixtures cover.  Bit-exact."""
import random

import pytest

pytestmark = pytest.mark.gpu

mosaic = pytest.importorskip("paper_2605_18710_b200.mosaic")
from oracle import restatement as R  # noqa: E402


def _same(gpu, cpu):
    if cpu["status"] != 0:
        assert gpu is None
        return
    assert gpu is not None
    assert gpu.stage_time == cpu["stage_time"]
    got = [(e.module, e.option.dp_degree, e.option.quota_units, e.gpus)
           for e in gpu.allocation.entries]
    assert got == [(m, d, u, g) for m, d, u, g in cpu["alloc"]]


CASES = [(seed, n, g, L) for seed, (n, g, L) in enumerate(
    [(2, 16, 8), (3, 16, 10), (2, 32, 10), (3, 32, 8), (2, 64, 10), (3, 64, 16),
     (2, 128, 10), (3, 8, 20), (4, 8, 10), (4, 16, 5)] * 3, start=101)]


@pytest.mark.parametrize("seed,n,g,L", CASES)
def test_stage_eval_random_large_g(seed, n, g, L):
    spec = f"random:{seed}:{n}:{g}"
    pl = mosaic.Planner.from_spec(spec, quota_levels=L)
    P = R.Problem(spec, L)
    mods = list(range(n))
    _same(pl.stage_eval(mods), P.stage_eval((1 << n) - 1))
    # every pair as well (the masks GAHC evaluates)
    for a in range(n):
        for b in range(a + 1, n):
            _same(pl.stage_eval([a, b]), P.stage_eval((1 << a) | (1 << b)))


@pytest.mark.parametrize("seed,n,g,L", CASES[:10])
def test_solve_random_large_g(seed, n, g, L):
    spec = f"random:{seed}:{n}:{g}"
    r = mosaic.Planner.from_spec(spec, quota_levels=L).solve()
    c = R.Problem(spec, L).solve()
    assert r.plan.predicted_iteration_time == c["iteration_time"]
    assert len(r.plan.stages) == len(c["stages"])
    assert r.trace.feasibility_calls == c["feasibility_calls"]


def test_evaluator_fuzz_vs_restatement():
    rng = random.Random(7)
    for spec, L in [("cfg5", 0), ("random:3:6:64", 10), ("random:9:5:32", 16)]:
        pl = mosaic.Planner.from_spec(spec, quota_levels=L)
        P = R.Problem(spec, L)
        G = pl.gpu_count
        allocs, want = [], []
        for _ in range(200):
            k = rng.randint(1, pl.n_modules)
            ents = []
            for m in sorted(rng.sample(range(pl.n_modules), k)):
                opts = pl.candidate_options(m)
                if not opts:
                    continue
                c = rng.choice(opts)
                gp = sorted(rng.sample(range(G), c.opt.dp_degree))
                ents.append((m, c.opt.dp_degree, c.opt.quota_units, gp))
            if not ents:
                continue
            allocs.append(mosaic.StageAllocation([mosaic.Entry(
                m, mosaic.DeploymentOption(d, u, pl.quota_levels), g) for m, d, u, g in ents]))
            want.append(P.stage_time(ents))
        assert pl.stage_time(allocs) == want
