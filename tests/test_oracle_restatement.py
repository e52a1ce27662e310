"""CPU: pin the C restatement (oracle/mosaic_oracle.c) to golden outputs of the REAL
reference (tests/golden, generated from oracle/_ref by tests/golden/make_golden.py).
Everything is compared bit-exactly (fp64 bit patterns, GPU lists)."""
import pytest

from conftest import alloc_tuples, hexf, load_golden
from oracle import restatement as R


def _args(g):
    levels, extra = 0, []
    for x in g["args"][2:]:
        if x.startswith("levels="):
            levels = int(x[7:])
        elif x in ("noself", "additive") or x.startswith(("e=", "mem=")):
            extra.append(x)
    return g["args"][0], levels, extra


def check_stage(r, g):
    if not g["feasible"]:
        assert r["status"] != 0
        return
    assert r["status"] == 0
    assert r["stage_time"] == hexf(g["t"])
    assert r["alloc"] == alloc_tuples(g["alloc"])


def check_plan(r, g):
    assert r["status"] == 0
    assert r["iteration_time"] == hexf(g["iteration_time"])
    assert len(r["stages"]) == len(g["stages"])
    for s, gs in zip(r["stages"], g["stages"]):
        assert s["stage_time"] == hexf(gs["t"])
        assert s["alloc"] == alloc_tuples(gs["alloc"])


CONFIGS = load_golden("configs.json")


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_options_bits(cfg):
    P = R.Problem(cfg)
    for m, gm in enumerate(CONFIGS[cfg]["options"]["modules"]):
        got = P.options(m)
        want = [(r[0], r[1], hexf(r[2]), hexf(r[3]), hexf(r[4])) for r in gm["rows"]]
        assert got == want


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3", "cfg4"])
def test_config_solve(cfg):
    g = CONFIGS[cfg]["solve"]
    r = R.Problem(cfg).solve()
    check_plan(r, g)
    assert r["stage_eval_calls"] == g["stage_eval_calls"]
    assert r["feasibility_calls"] == g["feasibility_calls"]


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_config_oracle(cfg):
    g = CONFIGS[cfg]["oracle"]
    r = R.Problem(cfg).brute_force()
    check_plan(r, g)
    assert r["partitions"] == g["partitions"]


RANDOM = load_golden("random_sets.json")


def test_acceptance_c2():
    for row in RANDOM["c2"]:
        spec, L, _ = _args(row["stage"])
        n = int(spec.split(":")[2])
        P = R.Problem(spec, L)
        check_stage(P.stage_eval((1 << n) - 1), row["stage"])
        check_stage(P.exact((1 << n) - 1), row["exact"])


def test_stage_eval_60():
    for row in RANDOM["stage_eval_60"]:
        spec, L, _ = _args(row["stage"])
        P = R.Problem(spec, L)
        check_stage(P.stage_eval(7), row["stage"])
        check_stage(P.exact(7), row["exact"])


def test_acceptance_c1_subset():
    for row in RANDOM["c1"][:40]:
        spec, L, _ = _args(row["solve"])
        P = R.Problem(spec, L)
        check_plan(P.solve(), row["solve"])
        if row["oracle"]["feasible"]:
            check_plan(P.brute_force(), row["oracle"])


def test_variants():
    for row in load_golden("variants.json"):
        spec, L, extra = _args(row["stage"])
        P = R.Problem(spec, L, extra)
        g = row["stage"]
        r = P.stage_eval(7)
        if g.get("status") == 2:
            assert r["status"] == 2
        else:
            check_stage(r, g)


def test_cfg5_small_masks():
    gold = load_golden("cfg5_stages.json")
    P = R.Problem("cfg5")
    for g in gold["stage"]:
        if bin(g["mask"]).count("1") <= 2:
            check_stage(P.stage_eval(g["mask"]), g)


def test_stage_time_bits():
    rows = load_golden("stime.json")
    probs = {}
    for row in rows:
        key = (row["inst"], tuple(row["extra"]))
        if key not in probs:
            probs[key] = R.Problem(row["inst"], 0, row["extra"])
        ents = [(m, d, u, gp) for m, d, u, gp in row["entries"]]
        assert probs[key].stage_time(ents) == hexf(row["t"])
