"""CPU: the C-ABI library loads and exports every symbol include/mosaic_gpu.h declares;
host-side logic that needs no device (synthetic problems, record merge)."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT, load_golden

mosaic = pytest.importorskip("paper_2605_18710_b200.mosaic")


def header_symbols():
    with open(os.path.join(ROOT, "include", "mosaic_gpu.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"\b(mosaic_gpu_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = mosaic.load_library()
    syms = header_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert sorted(mosaic.EXPORTS) == syms


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", mosaic.LIB_PATH],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


@pytest.mark.parametrize("cfg,n,g,levels", [("cfg1", 2, 8, 10), ("cfg2", 3, 16, 8),
                                            ("cfg3", 4, 32, 10), ("cfg4", 6, 64, 10),
                                            ("cfg5", 8, 128, 32)])
def test_synth_problem_shapes(cfg, n, g, levels):
    L = mosaic.load_library()
    pp = C.POINTER(mosaic.ProblemC)()
    assert L.mosaic_gpu_synth_problem(cfg.encode(), 0, C.byref(pp)) == 0
    p = pp.contents
    assert (p.n_modules, p.gpu_count, p.quota_levels) == (n, g, levels)
    gold = load_golden("configs.json")[cfg]["options"]["modules"]
    assert [p.modules[i].id.decode() for i in range(n)] == [m["id"] for m in gold]
    # grid: d in powers of two <= G, a in deciles (profiler.hpp:44-54)
    nd = g.bit_length()
    assert all(p.modules[i].n_points == nd * 10 for i in range(n))
    L.mosaic_gpu_free_problem(pp)


def test_synth_rejects_unknown_spec():
    L = mosaic.load_library()
    pp = C.POINTER(mosaic.ProblemC)()
    assert L.mosaic_gpu_synth_problem(b"nope", 0, C.byref(pp)) == mosaic.RANGE
    assert b"unknown" in L.mosaic_gpu_last_error()


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(mosaic.MosaicError):
        mosaic.Planner.from_spec("cfg1")


def test_merge_ranks_rules():
    # MIN: smallest incumbent, lowest rank on ties; a restart on any rank restarts all
    recs = b"".join(mosaic.rank_record(True, v, [(1, [2])], aborted=(i == 2), leaf_value=v)
                    for i, v in enumerate([0.3, 0.5, 0.3]))
    m = mosaic.merge_ranks(recs, 3, 0, 1)
    assert (m["winner"], m["value"], m["aborted"], m["leaf_value"]) == (0, 0.3, True, 0.3)
    # FIRST: the hit earliest in reference DFS order — smaller option first, then the larger
    # take count of the first differing block; ranks without a hit never win
    recs = b"".join([mosaic.rank_record(True, 0.0, [(2, [4]), (0, [1, 3])], leaf_value=1.0),
                     mosaic.rank_record(False, 0.0),
                     mosaic.rank_record(True, 0.0, [(2, [4]), (0, [2, 0])], leaf_value=2.0),
                     mosaic.rank_record(True, 0.0, [(3, [4]), (0, [4, 0])], leaf_value=3.0)])
    f = mosaic.merge_ranks(recs, 4, 1, 2)
    assert (f["winner"], f["found"], f["leaf_value"]) == (2, True, 2.0)
    none = b"".join(mosaic.rank_record(False, 0.0) for _ in range(2))
    assert mosaic.merge_ranks(none, 2, 1, 1)["found"] is False
