"""N3: the reference's JSON v1 files (io.hpp) in and out of the planner.

CPU: loaders/validators against files the REAL reference wrote (tests/golden/io_files.json)
and round-trips.  GPU: load_scenario(...) -> solve -> plan_to_json equals the plan JSON the
reference's own solve() wrote for the same files (values bit-identical)."""
import copy
import json

import pytest

from conftest import load_golden

io = pytest.importorskip("paper_2605_18710_b200.io")
FILES = load_golden("io_files.json")


@pytest.mark.parametrize("inst", list(FILES))
def test_loaders_accept_reference_files(inst):
    f = FILES[inst]["files"]
    g = io.model_from_json(f["model"])
    c = io.cluster_from_json(f["cluster"])
    s = io.surfaces_from_json(f["profile"])
    im = io.interference_from_json(f["interference"])
    assert [m["id"] for m in g["modules"]] == [m["id"] for m in f["model"]["modules"]]
    assert c["gpu_count"] == f["cluster"]["gpu_count"]
    assert set(s) == {x["module"] for x in f["profile"]["surfaces"]}
    assert im["e1"] == f["interference"]["e1"]


def test_version_and_field_errors():
    f = FILES["cfg3"]["files"]
    bad = copy.deepcopy(f["cluster"])
    bad["version"] = 2
    with pytest.raises(io.IoError, match="unsupported version"):
        io.cluster_from_json(bad)
    bad = copy.deepcopy(f["interference"])
    del bad["e2"]
    with pytest.raises(io.IoError, match="missing field 'e2'"):
        io.interference_from_json(bad)
    bad = copy.deepcopy(f["model"])
    bad["edges"].append(["vision"])
    with pytest.raises(io.IoError, match="pair"):
        io.model_from_json(bad)
    bad = copy.deepcopy(f["cluster"])
    bad["gpu_count"] = 0
    with pytest.raises(io.IoError, match="gpu_count"):
        io.cluster_from_json(bad)


@pytest.mark.parametrize("inst", list(FILES))
def test_plan_json_round_trip(inst):
    f = FILES[inst]["files"]
    ids = [m["id"] for m in f["model"]["modules"]]
    plan = io.plan_from_json(f["plan"], ids)
    back = io.plan_to_json(plan, ids)
    assert back == json.loads(json.dumps(f["plan"]))


@pytest.mark.gpu
@pytest.mark.parametrize("inst", list(FILES))
def test_scenario_solve_matches_reference_plan_json(inst):
    f = FILES[inst]["files"]
    levels = 32 if inst.startswith("preset:ofasys") else None
    pl = io.load_scenario(f["model"], f["cluster"], f["profile"], f["interference"],
                          quota_levels=levels)
    got = io.plan_to_json(pl.solve().plan, pl.module_ids)
    assert got == f["plan"]
