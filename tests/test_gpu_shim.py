"""The drop-in proof: the reference's OWN solve() and brute_force_optimum() (unmodified
headers, compiled with tests/shim/Makefile into oracle/_ref/test_shim) running with the B200
backend at their seams (tests/shim/gpu_backend.hpp: the EvalCache seam of solve,
solver.hpp:160; stage_eval, stage_eval.hpp:302; ExactStageSolver inside brute_force_optimum,
oracle.hpp:219), compared in-process with the unmodified reference on the CPU."""
import json
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
BIN = os.path.join(ROOT, "oracle", "_ref", "test_shim")


def test_reference_planner_on_gpu_backend():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/test_shim not built (needs /root/reference at build time)")
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    bad = [x for x in lines if x.get("ok") is False]
    assert p.returncode == 0 and not bad, (bad, p.stderr[-2000:])
    checks = {(x["inst"], x["check"]) for x in lines if "check" in x}
    for inst in ("cfg1", "cfg2", "cfg3", "cfg4"):
        assert (inst, "solve") in checks and (inst, "stage_eval") in checks
    assert ("cfg1", "oracle") in checks and ("cfg2", "oracle") in checks
    assert all(x["cache_misses"] == 0 for x in lines if x.get("check") == "solve")
