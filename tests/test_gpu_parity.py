"""GPU parity: the CUDA planner against golden outputs of the REAL reference
(tests/golden/*.json, produced by tests/golden/make_golden.py from oracle/_ref).

Bar (BASELINE.json north_star): chosen plans bit-identical — stage order, module->stage
map, (d, quota_units, GPU list) per module — and stage / iteration times equal as fp64
bit patterns (stricter than the 1e-9 relative tolerance the north star allows).
"""
import pytest

from conftest import alloc_tuples, hexf, load_golden, result_tuples

pytestmark = pytest.mark.gpu

mosaic = pytest.importorskip("paper_2605_18710_b200.mosaic")


def planner(spec, levels=0, extra=(), **kw):
    if not extra:
        return mosaic.Planner.from_spec(spec, quota_levels=levels, **kw)
    # variants: rebuild from the synthetic surfaces with modified model / cluster
    base = mosaic.Planner.from_spec(spec, quota_levels=levels)
    pp = base._owned.contents
    e = [pp.e1, pp.e2, pp.e3]
    self_, add, mem = True, False, pp.memory_capacity
    for x in extra:
        if x == "noself":
            self_ = False
        elif x == "additive":
            add = True
        elif x.startswith("e="):
            e = [float(v) for v in x[2:].split(",")]
        elif x.startswith("mem="):
            mem = float(x[4:])
    pp.e1, pp.e2, pp.e3 = e
    pp.include_self = int(self_)
    pp.additive_only = int(add)
    pp.memory_capacity = mem
    for k, v in kw.items():
        setattr(pp, k, int(v))
    pl = mosaic.Planner(base._owned)
    pl._owned, base._owned = base._owned, None
    base.close()
    return pl


def check_stage(res, gold):
    if not gold["feasible"]:
        assert res is None
        return
    assert res is not None
    assert res.stage_time == hexf(gold["t"]), (res.stage_time, gold["t_dec"])
    assert result_tuples(res) == alloc_tuples(gold["alloc"])


def check_plan(plan, gold):
    assert len(plan.stages) == len(gold["stages"])
    for st, t, g in zip(plan.stages, plan.predicted_stage_times, gold["stages"]):
        assert t == hexf(g["t"])
        got = [(e.module, e.option.dp_degree, e.option.quota_units, e.gpus) for e in st.entries]
        assert got == alloc_tuples(g["alloc"])
    assert plan.predicted_iteration_time == hexf(gold["iteration_time"])


def check_trace(trace, gold):
    assert len(trace.rounds) == len(gold["rounds"])
    for r, g in zip(trace.rounds, gold["rounds"]):
        assert (r.chosen_x, r.chosen_y) == (g["x"], g["y"])
        assert r.applied_gain == hexf(g["gain"])
        assert len(r.candidates) == len(g["cands"])
        for c, gc in zip(r.candidates, g["cands"]):
            assert (c.mask_x, c.mask_y, c.pruned, c.cache_hit) == (
                gc["x"], gc["y"], bool(gc["pruned"]), bool(gc["hit"]))
            if not c.pruned:
                assert c.gain == hexf(gc["gain"])
    assert trace.stage_eval_calls == gold["stage_eval_calls"]
    assert trace.feasibility_calls == gold["feasibility_calls"]


CONFIGS = load_golden("configs.json")


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3", "cfg4"])
def test_config_solve_bit_identical(cfg):
    pl = planner(cfg)
    r = pl.solve()
    check_plan(r.plan, CONFIGS[cfg]["solve"])
    check_trace(r.trace, CONFIGS[cfg]["solve"])


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3", "cfg4"])
def test_config_solve_noprune_nocache(cfg):
    pl = planner(cfg, enable_prune=False, enable_cache=False)
    r = pl.solve()
    check_plan(r.plan, CONFIGS[cfg]["solve_noprune_nocache"])
    check_trace(r.trace, CONFIGS[cfg]["solve_noprune_nocache"])


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_config_oracle_bit_identical(cfg):
    pl = planner(cfg)
    r = pl.brute_force_optimum()
    g = CONFIGS[cfg]["oracle"]
    check_plan(r.plan, g)
    assert r.partitions_examined == g["partitions"]


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_config_options_bit_identical(cfg):
    pl = planner(cfg)
    for m, gm in enumerate(CONFIGS[cfg]["options"]["modules"]):
        got = [(c.opt.dp_degree, c.opt.quota_units, c.base_latency.hex(), c.solo_bandwidth.hex(),
                c.footprint.hex()) for c in pl.candidate_options(m)]
        want = [(r[0], r[1], float.fromhex(r[2]).hex(), float.fromhex(r[3]).hex(),
                 float.fromhex(r[4]).hex()) for r in gm["rows"]]
        assert got == want


CFG5 = load_golden("cfg5_stages.json")


def test_cfg5_stage_eval_per_mask():
    pl = planner("cfg5")
    for g in CFG5["stage"]:
        mods = [m for m in range(8) if g["mask"] >> m & 1]
        res = pl.stage_eval(mods)
        check_stage(res, g)
        assert res.stats.feasibility_calls == g["feasibility_calls"]


def test_cfg5_feasibility_probes():
    pl = planner("cfg5")
    for g in CFG5["feas"]:
        mods = [m for m in range(8) if g["mask"] >> m & 1]
        res = pl.feasibility_run(mods, float.fromhex(g["tau"]))
        check_stage(res, g)


RANDOM = load_golden("random_sets.json")


def _inst(g):
    a = g["args"]
    levels = 0
    for x in a[2:]:
        if x.startswith("levels="):
            levels = int(x[7:])
    return a[0], levels


def test_acceptance_c2_stage_vs_exact():
    for row in RANDOM["c2"]:
        spec, L = _inst(row["stage"])
        pl = planner(spec, L)
        n = int(spec.split(":")[2])
        check_stage(pl.stage_eval(range(n)), row["stage"])
        check_stage(pl.exact_stage(range(n)), row["exact"])
        pl.close()


def test_stage_eval_60_seeds():
    for row in RANDOM["stage_eval_60"]:
        spec, L = _inst(row["stage"])
        pl = planner(spec, L)
        check_stage(pl.stage_eval(range(3)), row["stage"])
        check_stage(pl.exact_stage(range(3)), row["exact"])
        pl.close()


def test_acceptance_c1_solve_and_oracle():
    for row in RANDOM["c1"] + RANDOM["c1_6mod"]:
        spec, L = _inst(row["solve"])
        pl = planner(spec, L)
        r = pl.solve()
        check_plan(r.plan, row["solve"])
        check_trace(r.trace, row["solve"])
        o = pl.brute_force_optimum()
        if row["oracle"]["feasible"]:
            check_plan(o.plan, row["oracle"])
        else:
            assert o is None
        pl.close()


def test_random_bigger_stages():
    for row in RANDOM["big"]:
        spec, L = _inst(row["stage"])
        pl = planner(spec, L)
        n = int(spec.split(":")[2])
        check_stage(pl.stage_eval(range(n)), row["stage"])
        if row["exact"] is not None:
            check_stage(pl.exact_stage(range(n)), row["exact"])
        pl.close()


PRESETS = load_golden("presets.json")


def test_presets_solve_and_prune_cache_invariance():
    for row in PRESETS:
        spec, L = _inst(row["solve"])
        pl = planner(spec, L)
        r = pl.solve()
        check_plan(r.plan, row["solve"])
        check_trace(r.trace, row["solve"])
        pl.close()
        if "solve_noprune_nocache" in row:
            pl = planner(spec, L, enable_prune=False, enable_cache=False)
            r2 = pl.solve()
            check_plan(r2.plan, row["solve_noprune_nocache"])
            pl.close()


VARIANTS = load_golden("variants.json")


def test_model_variants():
    for row in VARIANTS:
        spec, L = _inst(row["stage"])
        pl = planner(spec, L, extra=row["extra"])
        g = row["stage"]
        if g.get("status") == 2 or "exception" in g:
            with pytest.raises(mosaic.StageInfeasibleError):
                pl.stage_eval(range(3))
        else:
            check_stage(pl.stage_eval(range(3)), g)
        ge = row["exact"]
        if "exception" not in ge:
            # negative coefficients included: ExactStageSolver's sequential option cut is
            # replayed by one walker in its DFS order (planner.cpp exact_stage_job)
            check_stage(pl.exact_stage(range(3)), ge)
        gs = row["solve"]
        if "exception" in gs:
            with pytest.raises(mosaic.MosaicError):
                pl.solve()
        else:
            r = pl.solve()
            check_plan(r.plan, gs)
        pl.close()


STIME = load_golden("stime.json")


def test_evaluator_stage_time_bits():
    groups = {}
    for row in STIME:
        groups.setdefault((row["inst"], tuple(row["extra"])), []).append(row)
    for (inst, extra), rows in groups.items():
        pl = planner(inst, extra=list(extra))
        allocs = []
        for row in rows:
            ents = [mosaic.Entry(m, mosaic.DeploymentOption(d, u, pl.quota_levels), gp)
                    for m, d, u, gp in row["entries"]]
            allocs.append(mosaic.StageAllocation(ents))
        got = pl.stage_time(allocs)
        want = [hexf(r["t"]) for r in rows]
        assert got == want
        pl.close()


def test_surface_without_d1_raises_range_error():
    # candidate_options needs lookup(1, a) for the solo bandwidth (perf_model.hpp:420-422);
    # a surface profiled only from d=2 makes the reference throw SurfaceRangeError
    pts = [(d, a / 10, 1.0 / (d * a), 0.5, 1e9, 1.0) for d in (2, 4) for a in range(1, 11)]
    pl = mosaic.Planner.from_surfaces([{"id": "m", "memory_base": 0.0, "points": pts}], [], 4)
    with pytest.raises(mosaic.SurfaceRangeError):
        pl.stage_eval([0])


def test_stage_min_equals_stage_eval_time():
    pl = planner("cfg5")
    for mods in ([0, 1], [0, 1, 2], [1, 3, 5]):
        r = pl.stage_eval(mods)
        assert pl.stage_min(mods) == r.stage_time


def test_evaluator_reproduces_searched_allocations():
    # k_eval on every allocation the search returned must give back its stage time
    pl = planner("cfg4")
    res = pl.solve()
    assert pl.stage_time(res.plan.stages) == res.plan.predicted_stage_times


def _plan_of(stages, L):
    return mosaic.DeploymentPlan(stages=[
        mosaic.StageAllocation(entries=[
            mosaic.Entry(m, mosaic.DeploymentOption(d, u, L), list(g)) for m, d, u, g in st])
        for st in stages])


def test_validate_plan_matches_reference_verdicts():
    # H15 validate_plan (core.hpp:281-351) with the footprint oracle: solved plans and fuzzed
    # mutations (drop / duplicate / reorder / overcommit / co-locate / out-of-range / empty)
    rows = load_golden("validate.json")
    groups = {}
    for row in rows:
        groups.setdefault((row["inst"], tuple(row["extra"])), []).append(row)
    for (inst, extra), rs in groups.items():
        lv = [int(x[7:]) for x in extra if x.startswith("levels=")]
        rest = [x for x in extra if not x.startswith("levels=")]
        pl = planner(inst, lv[0] if lv else 0, extra=rest)
        L = pl.quota_levels
        for r in rs:
            plan = _plan_of(r["stages"], L)
            if r["exception"]:
                with pytest.raises(mosaic.SurfaceRangeError):
                    pl.validate_plan(plan)
            else:
                code, msg = pl.validate_plan(plan)
                assert code == r["code"], (inst, extra, r["kind"], msg)
        pl.close()


def test_solved_plans_validate_ok():
    # acceptance C9: every plan solve() returns passes validate_plan with footprints
    for spec, L in [("cfg1", 0), ("cfg3", 0), ("cfg4", 0), ("random:5:5:8", 4),
                    ("preset:ofasys:10:8", 0)]:
        pl = planner(spec, L)
        assert pl.validate_plan(pl.solve().plan)[0] == "Ok"
        pl.close()
