"""N4: exclusive-allocation baselines (make_baseline_plan) and the batched
plan replay (simulate, k_simulate) against golden outputs of the REAL reference
(tests/golden/simulate.json, normals.json from oracle/_ref/ref_driver).

Bars: baseline plans bit-identical (stage order, degrees, GPU lists, fp64 stage times);
replay without perturbation bit-identical; with log-normal perturbation the draws follow the
reference's RNG stream exactly and the replayed times agree to 1e-12 relative (the device
log/exp may differ from glibc by an ulp)."""
import pytest

from conftest import hexf, load_golden

mosaic = pytest.importorskip("paper_2605_18710_b200.mosaic")
REL = 1e-12


def test_normal_stream_restatement_matches_libstdcxx():
    # CPU: the C restatement of std::normal_distribution over std::mt19937_64 (the algorithm
    # k_simulate runs per seed) reproduces the reference's draws bit for bit
    rest = pytest.importorskip("oracle.restatement")
    for row in load_golden("normals.json"):
        seed, n = int(row["args"][2]), int(row["args"][3])
        assert [x.hex() for x in rest.normals(seed, n)] == [hexf(h).hex() for h in row["normals"]]


def _planner(inst, extra):
    lv = [int(x[7:]) for x in extra if x.startswith("levels=")]
    pl = mosaic.Planner.from_spec(inst, quota_levels=lv[0] if lv else 0)
    mem = [float(x[4:]) for x in extra if x.startswith("mem=")]
    if mem:
        pp = pl._owned.contents
        pp.memory_capacity = mem[0]
        pl2 = mosaic.Planner(pl._owned)
        pl2._owned, pl._owned = pl._owned, None
        pl.close()
        pl = pl2
    return pl


def _plan_tuples(plan):
    return [[(e.module, e.option.dp_degree, e.option.quota_units, list(e.gpus))
             for e in s.entries] for s in plan.stages]


def _golden_tuples(r):
    return [[(a["m"], a["d"], a["u"], a["gpus"]) for a in s["alloc"]] for s in r["stages"]]


def _cfg(args):
    c = mosaic.SimConfig()
    for a in args:
        if a.startswith("iters="):
            c.iterations = int(a[6:])
        elif a.startswith("sigma="):
            c.perturbation_sigma = float(a[6:])
        elif a.startswith("seed="):
            c.seed = int(a[5:])
        elif a == "ondemand":
            c.stream_mode = "on_demand"
    return c


def _close(a, b, exact):
    return a == b if exact else abs(a - b) <= REL * max(abs(a), abs(b))


@pytest.mark.gpu
def test_baseline_plans_bit_identical():
    rows = [x for x in load_golden("simulate.json") if x["op"] == "baseline"]
    for x in rows:
        pl = _planner(x["inst"], x["extra"])
        r = x["r"]
        if "exception" in r:
            with pytest.raises(mosaic.InfeasibleBaselineError):
                pl.make_baseline_plan(x["policy"])
        else:
            plan = pl.make_baseline_plan(x["policy"])
            assert _plan_tuples(plan) == _golden_tuples(r), (x["inst"], x["policy"])
            assert [t.hex() for t in plan.predicted_stage_times] == [
                hexf(s["t"]).hex() for s in r["stages"]]
            assert plan.predicted_iteration_time == hexf(r["iteration_time"])
        pl.close()


@pytest.mark.gpu
def test_simulate_matches_reference():
    rows = [x for x in load_golden("simulate.json") if x["op"] == "simulate"]
    for x in rows:
        pl = _planner(x["inst"], x["extra"])
        r = x["r"]
        if "exception" in r:
            pl.close()
            continue
        plan = mosaic.DeploymentPlan(stages=[
            mosaic.StageAllocation(entries=[
                mosaic.Entry(m, mosaic.DeploymentOption(d, u, pl.quota_levels), g)
                for m, d, u, g in st]) for st in _golden_tuples(r)])
        cfg = _cfg(x["cfg"])
        exact = cfg.perturbation_sigma == 0
        rep = pl.simulate(plan, cfg)[0]
        tag = (x["inst"], x["policy"], x["cfg"])
        assert _close(rep.iteration_time, hexf(r["sim_iteration_time"]), exact), tag
        assert all(_close(a, hexf(b), exact) for a, b in zip(rep.per_stage_times, r["per_stage"])), tag
        assert all(_close(a, hexf(b), exact)
                   for a, b in zip(rep.per_gpu_busy_fraction, r["busy"])), tag
        assert _close(rep.mean_busy_fraction, hexf(r["mean_busy"]), exact), tag
        assert len(rep.timeline) == len(r["timeline"]), tag
        for t, g in zip(rep.timeline, r["timeline"]):
            assert (t.gpu, t.module) == (g[0], g[1]), tag
            assert _close(t.start, hexf(g[2]), exact) and _close(t.end, hexf(g[3]), exact), tag
            assert t.quota == hexf(g[4]), tag
        pl.close()


@pytest.mark.gpu
def test_simulate_many_seeds_one_launch():
    # the batch: per-seed reports equal one-seed runs (each thread owns its RNG stream)
    pl = mosaic.Planner.from_spec("cfg4")
    plan = pl.solve().plan
    cfg = mosaic.SimConfig(iterations=4, perturbation_sigma=0.2)
    seeds = list(range(100, 164))
    batch = pl.simulate(plan, cfg, seeds)
    for i in (0, 17, 63):
        one = pl.simulate(plan, cfg, [seeds[i]])[0]
        assert batch[i].iteration_time == one.iteration_time
        assert batch[i].per_gpu_busy_fraction == one.per_gpu_busy_fraction
    with pytest.raises(mosaic.InvalidArgumentError):
        pl.simulate(plan, mosaic.SimConfig(iterations=0))
    pl.close()


@pytest.mark.gpu
def test_distmm_baseline_where_the_reference_does_not_finish():
    # cfg5: the reference enumerates every composition of 7 encoders over 128 GPUs and does
    # not finish; the closed form (pinned on the golden instances above) answers at once
    # and its plan must be valid
    pl = mosaic.Planner.from_spec("preset:ofasys:8:32")
    plan = pl.make_baseline_plan("distmm")
    assert pl.validate_plan(plan)[0] == "Ok"
    pl.close()
    pl5 = mosaic.Planner.from_spec("cfg5")
    plan5 = pl5.make_baseline_plan("distmm")
    assert pl5.validate_plan(plan5)[0] == "Ok"
    assert len(plan5.stages) == 2 and len(plan5.stages[0].entries) == 7
    pl5.close()
