"""GPU parity on the cfg5 headline trajectory (and two intermediate shapes of it): every
reference result pinned so far (tests/golden/trajectory_ref.jsonl, produced by the unmodified
reference through tests/golden/make_cfg5_trajectory.py) reproduced bit for bit by the device
path, and the device's current solve still following the recorded trajectory."""
import pytest

from conftest import hexf
from trajectory import bits, done, load_gpu, load_ref

pytestmark = pytest.mark.gpu
mosaic = pytest.importorskip("paper_2605_18710_b200.mosaic")

REF = load_ref()
TRAJ = load_gpu()


def tuples(alloc):
    return [(a["m"], a["d"], a["u"], list(a["gpus"])) for a in alloc]


def res_tuples(r):
    return [(e.module, e.option.dp_degree, e.option.quota_units, list(e.gpus))
            for e in r.allocation.entries]


@pytest.fixture(scope="module")
def planners():
    out = {}
    for name, sh in TRAJ.items():
        out[name] = mosaic.Planner.from_spec(sh["spec"], quota_levels=sh["levels"], device=0)
    yield out
    for p in out.values():
        p.close()


@pytest.mark.parametrize("shape", sorted(TRAJ))
def test_pinned_stage_evals(planners, shape):
    pl = planners[shape]
    recs = [(int(k.rsplit("|", 1)[1]), r) for k, r in REF.items()
            if k.startswith(shape + "|stage|") and done(r)]
    assert recs
    got = pl.search([bits(m) for m, _ in recs])
    for (m, r), g in zip(recs, got):
        o = r["out"]
        assert (g is not None) == bool(o["feasible"]), m
        if g is not None:
            assert g.stage_time == hexf(o["t"]), (shape, m)
            assert res_tuples(g) == tuples(o["alloc"]), (shape, m)
            assert g.stats.feasibility_calls == o["feasibility_calls"], (shape, m)


@pytest.mark.parametrize("shape", sorted(TRAJ))
def test_pinned_probes(planners, shape):
    # FeasibilitySearch::run at the probes that decide a large stage's result: the last
    # successful one returns the stage_eval allocation itself
    pl = planners[shape]
    n = 0
    for key, r in REF.items():
        if not key.startswith(shape + "|feas") or not done(r):
            continue
        m = int(key.rsplit("|", 1)[1])
        o = r["out"]
        g = pl.feasibility_run(bits(m), hexf(o["tau"]))
        assert (g is not None) == bool(o["feasible"]), key
        if g is not None:
            assert g.stage_time == hexf(o["t"]) and res_tuples(g) == tuples(o["alloc"]), key
        if "feas_last_ok" in key:
            s = pl.stage_eval(bits(m))
            assert s.stage_time == hexf(o["t"]) and res_tuples(s) == tuples(o["alloc"]), key
        n += 1
    if shape.startswith("cfg5"):
        assert n >= 3


@pytest.mark.parametrize("shape", sorted(TRAJ))
def test_trajectory_is_current(planners, shape):
    # the recorded GPU trajectory is what the product does today (the pins apply to it)
    pl = planners[shape]
    r = pl.solve()
    sh = TRAJ[shape]
    assert r.plan.predicted_iteration_time == hexf(sh["iteration_time"])
    assert [res_tuples(type("R", (), {"allocation": s})) for s in r.plan.stages] == \
        [tuples(s["alloc"]) for s in sh["stages"]]
    got = [(rd.chosen_x, rd.chosen_y, [(c.mask_x, c.mask_y, int(c.pruned), int(c.cache_hit))
                                       for c in rd.candidates]) for rd in r.trace.rounds]
    want = [(rd["x"], rd["y"], [(c["x"], c["y"], c["pruned"], c["hit"]) for c in rd["cands"]])
            for rd in sh["rounds"]]
    assert got == want
    assert r.trace.stage_eval_calls == sh["stage_eval_calls"]
    assert r.trace.feasibility_calls == sh["feasibility_calls"]
    # every solve record of the reference for this shape
    ref = REF.get(f"{shape}|solve")
    if done(ref):
        assert r.plan.predicted_iteration_time == hexf(ref["out"]["iteration_time"])
