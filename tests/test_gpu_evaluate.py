"""K1 evaluator (mosaic_gpu_evaluate, eval.cu) parity with the reference's stage_time
(perf_model.hpp:442-479): fp64 bit patterns, host and device arrays, edge cases and errors."""
import math
import os
import sys

import numpy as np
import pytest

from conftest import ROOT, hexf, load_golden

pytestmark = pytest.mark.gpu

mosaic = pytest.importorskip("paper_2605_18710_b200.mosaic")
sys.path.insert(0, os.path.join(ROOT, "tools"))
from evalgen import random_allocations, to_allocations  # noqa: E402
from test_gpu_parity import planner  # noqa: E402

EDGE = load_golden("stime_edge.json")


def test_edge_cases_match_reference_bits():
    # off-grid dp degrees (log2 interpolation in the rate tables), any quota unit,
    # duplicate modules, repeated / unsorted GPU ids, negative coefficients
    groups = {}
    for row in EDGE:
        groups.setdefault((row["inst"], tuple(row["extra"])), []).append(row)
    for (inst, extra), rows in groups.items():
        pl = planner(inst, extra=list(extra))

        def alloc(row):
            return mosaic.StageAllocation(
                [mosaic.Entry(m, mosaic.DeploymentOption(d, u, pl.quota_levels), gp)
                 for m, d, u, gp in row["entries"]])
        ok = [r for r in rows if r["t"] is not None]
        got = pl.stage_time([alloc(r) for r in ok])
        want = [hexf(r["t"]) for r in ok]
        bad = [(i, g, w) for i, (g, w) in enumerate(zip(got, want)) if g != w]
        assert not bad, (inst, extra, bad[:5])
        # the reference throws SurfaceRangeError exactly when a lookup it makes (a self
        # entry's base latency, a counted resident's solo bandwidth) leaves the hull
        for r in rows:
            if r["t"] is None:
                with pytest.raises(mosaic.SurfaceRangeError):
                    pl.stage_time([alloc(r)])
        pl.close()


def _torch():
    return pytest.importorskip("torch")


@pytest.mark.parametrize("spec,extra", [("cfg5", ()), ("cfg5", ("noself",)),
                                        ("cfg4", ("additive",)),
                                        ("cfg3", ("e=1e-3,-2e-4,5e-4",))])
def test_evaluate_host_device_and_reference_api_agree(spec, extra):
    torch = _torch()
    pl = planner(spec, extra=list(extra))
    ent, gpus, off = random_allocations(pl, 20000, seed=3)
    n = len(off) - 1
    st_h = np.zeros(n)
    rect_h = np.zeros(len(ent))
    pl.evaluate(ent, gpus, off, st_h, rect_h)
    dev = torch.device("cuda", 0)
    tE, tG, tO = (torch.from_numpy(x).to(dev) for x in (ent, gpus, off))
    st_d = torch.zeros(n, dtype=torch.float64, device=dev)
    rect_d = torch.zeros(len(ent), dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    pl.evaluate(tE, tG, tO, st_d, rect_d, device=True)
    assert np.array_equal(st_d.cpu().numpy(), st_h)
    assert np.array_equal(rect_d.cpu().numpy(), rect_h)
    # the reference-API path (one StageAllocation per allocation) on a slice
    allocs = to_allocations(ent, gpus, off, pl.quota_levels, 0, 300)
    st_r, rect_r = pl.stage_time(allocs, with_rectified=True)
    assert st_r == list(st_h[:300])
    assert [x for r in rect_r for x in r] == list(rect_h[:off[300]])
    s = pl.evaluate_stats()
    assert s["launches"] >= 2 and s["kernel_ms"] > 0 and s["alg_bytes"] > 0
    pl.close()


def test_evaluate_matches_restatement_oracle():
    from oracle import restatement
    if not restatement.available():
        pytest.skip("oracle restatement not built")
    pl = planner("cfg5")
    ent, gpus, off = random_allocations(pl, 400, seed=11)
    st = np.zeros(len(off) - 1)
    pl.evaluate(ent, gpus, off, st)
    prob = restatement.Problem("cfg5")
    for a in range(len(off) - 1):
        ents = []
        for e in range(off[a], off[a + 1]):
            m, d, u, ng = (int(x) for x in ent[e, :4])
            go = int(ent[e, 6:8].copy().view(np.int64)[0])
            ents.append((m, d, u, [int(x) for x in gpus[go:go + ng]]))
        assert st[a] == prob.stage_time(ents), a
    pl.close()


def test_evaluate_edge_shapes_and_errors():
    pl = planner("cfg5")
    L = pl.quota_levels
    # empty allocation -> 0.0 (stage_time's seed); entry without GPUs -> base - 1e300
    ent = mosaic.pack_eval_entries([0, 1], [4, 4], [8, 8], [0, 4], [0, 0])
    gpus = np.arange(4, dtype=np.int32)
    off = np.array([0, 0, 1, 2], dtype=np.int64)
    st = np.zeros(3)
    rect = np.zeros(2)
    pl.evaluate(ent, gpus, off, st, rect)
    assert st[0] == 0.0 and st[1] == 0.0
    assert rect[0] < -1e299
    ref = pl.stage_time([mosaic.StageAllocation(
        [mosaic.Entry(1, mosaic.DeploymentOption(4, 8, L), [0, 1, 2, 3])])])
    assert st[2] == ref[0]
    # the same quota at another granularity goes through the per-call row path
    twice = pl.stage_time([mosaic.StageAllocation(
        [mosaic.Entry(1, mosaic.DeploymentOption(4, 16, 2 * L), [0, 1, 2, 3])])])
    assert twice == ref
    cases = [
        (mosaic.pack_eval_entries([9], [4], [8], [4], [0]), mosaic.SurfaceRangeError),  # module
        (mosaic.pack_eval_entries([1], [4], [8], [4], [0], [2 * L]), mosaic.SurfaceRangeError),
        (mosaic.pack_eval_entries([1], [4], [L + 1], [4], [0]), mosaic.SurfaceRangeError),
        (mosaic.pack_eval_entries([1], [4], [8], [5], [0]), mosaic.SurfaceRangeError),  # ids
    ]
    for e, exc in cases:
        with pytest.raises(exc):
            pl.evaluate(e, gpus, np.array([0, 1], dtype=np.int64), np.zeros(1))
    g2 = np.array([0, 1, 2, 999], dtype=np.int32)
    with pytest.raises(mosaic.SurfaceRangeError):
        pl.evaluate(mosaic.pack_eval_entries([1], [4], [8], [4], [0]), g2,
                    np.array([0, 1], dtype=np.int64), np.zeros(1))
    big = mosaic.pack_eval_entries([0] * 65, [1] * 65, [1] * 65, [1] * 65, [0] * 65)
    with pytest.raises(mosaic.OracleTooLargeError):
        pl.evaluate(big, gpus, np.array([0, 65], dtype=np.int64), np.zeros(1))
    pl.close()


def test_evaluate_many_entries_deferred_path():
    # > 32 entries: the CTA kernel defers the allocation to the warp kernel; both paths must
    # agree with the per-call row path (other quota granularity: the first evaluator kernel)
    pl = planner("cfg5")
    L = pl.quota_levels
    rng = np.random.default_rng(5)
    allocs_a, allocs_b = [], []
    for n_ent in (31, 32, 33, 40, 64):
        ea, eb = [], []
        for i in range(n_ent):
            m = int(rng.integers(0, 8))
            d = int(rng.choice([1, 2, 4, 8]))
            u = int(rng.integers(8, L + 1))
            g = sorted(int(x) for x in rng.choice(128, size=d, replace=False))
            ea.append(mosaic.Entry(m, mosaic.DeploymentOption(d, u, L), g))
            eb.append(mosaic.Entry(m, mosaic.DeploymentOption(d, 2 * u, 2 * L), g))
        allocs_a.append(mosaic.StageAllocation(ea))
        allocs_b.append(mosaic.StageAllocation(eb))
    sa, ra = pl.stage_time(allocs_a, with_rectified=True)
    sb, rb = pl.stage_time(allocs_b, with_rectified=True)
    assert sa == sb and ra == rb
    pl.close()


def test_large_clusters_match_reference_bits():
    # G = 256 / 512 / 1024: the shared-memory bitmap path of k_evaluate
    rows = load_golden("stime_large_g.json")
    groups = {}
    for row in rows:
        groups.setdefault((row["inst"], tuple(row["extra"])), []).append(row)
    for (inst, extra), rs in groups.items():
        pl = planner(inst, extra=list(extra))
        allocs = [mosaic.StageAllocation(
            [mosaic.Entry(m, mosaic.DeploymentOption(d, u, pl.quota_levels), gp)
             for m, d, u, gp in r["entries"]]) for r in rs]
        assert pl.stage_time(allocs) == [hexf(r["t"]) for r in rs], (inst, extra)
        pl.close()


def _pack(allocs):
    """[(m, d, u, gpus), ...] per allocation -> the flat ABI arrays."""
    cols, gl, off = [[], [], [], [], []], [], [0]
    for a in allocs:
        for m, d, u, g in a:
            for c, v in zip(cols, (m, d, u, len(g), len(gl))):
                c.append(v)
            gl.extend(g)
        off.append(len(cols[0]))
    ent = mosaic.pack_eval_entries(*[np.array(c, dtype=np.int64) for c in cols])
    return ent, np.array(gl or [0], dtype=np.int32), np.array(off, dtype=np.int64)


def _fast_vs_full(pl, ent, gpus, off):
    """Stage times without per-entry output (k_evaluate_fast + worklist) against the full
    path (per-entry output requested: k_evaluate on everything), bit for bit."""
    n = len(off) - 1
    s0 = pl.evaluate_stats()
    st_fast = np.full(n, -7.0)
    pl.evaluate(ent, gpus, off, st_fast)
    s1 = pl.evaluate_stats()
    st_full = np.full(n, -7.0)
    pl.evaluate(ent, gpus, off, st_full, np.zeros(max(1, len(ent))))
    assert np.array_equal(st_fast.view(np.int64), st_full.view(np.int64)), \
        np.nonzero(st_fast.view(np.int64) != st_full.view(np.int64))[0][:10]
    return st_fast, s1["full_path_allocs"] - s0["full_path_allocs"]


@pytest.mark.parametrize("spec,extra", [("cfg5", ()), ("cfg4", ("additive",)),
                                        ("cfg3", ("e=1e-3,-2e-4,5e-4",)),
                                        ("cfg2", ()), ("cfg5", ("noself",))])
def test_fast_path_bits_random(spec, extra):
    # the monotone-max reformulation of k_evaluate_fast equals the per-entry maxima
    pl = planner(spec, extra=list(extra))
    ent, gpus, off = random_allocations(pl, 30000, seed=17)
    _, full = _fast_vs_full(pl, ent, gpus, off)
    if "noself" in extra:
        assert full == len(off) - 1  # without include_self the fast kernel does not apply
    else:
        assert full == 0, full        # distinct modules: every allocation on the fast path
    pl.close()


def test_fast_path_worklist_and_edges():
    # duplicate modules, repeated / unsorted GPU ids, empty allocations, entries without
    # GPUs, out-of-table options and > 32 entries mixed into one batch: those go through
    # the worklist to the full kernel, the rest stay on the fast path, all bit-exact
    pl = planner("cfg5")
    L = pl.quota_levels
    rng = np.random.default_rng(23)
    opts = [[(r.opt.dp_degree, r.opt.quota_units) for r in pl.candidate_options(m)]
            for m in range(8)]
    allocs, expect_full = [], 0
    for i in range(3000):
        kind = i % 6
        k = int(rng.integers(1, 9))
        mods = sorted(rng.choice(8, size=k, replace=False).tolist())
        a = []
        for m in mods:
            d, u = opts[m][int(rng.integers(0, len(opts[m])))]
            g = rng.choice(128, size=d, replace=False).tolist()
            a.append((m, d, u, g))
        if kind == 1:                       # duplicate module -> worklist
            a.append(a[0])
            expect_full += 1
        elif kind == 2:                     # repeated + unsorted ids in one entry
            m, d, u, g = a[-1]
            a[-1] = (m, d, u, g + g[:1])
        elif kind == 3:                     # an entry without GPUs -> worklist
            m, d, u, g = a[0]
            a[0] = (m, d, u, [])
            expect_full += 1
        elif kind == 4 and i % 12 == 4:     # empty allocation
            a = []
        elif kind == 5 and i % 30 == 5:     # > 32 entries -> worklist
            a = [(j % 8, *opts[j % 8][0], [j]) for j in range(40)]
            expect_full += 1
        allocs.append(a)
    ent, gpus, off = _pack(allocs)
    st, full = _fast_vs_full(pl, ent, gpus, off)
    assert full == expect_full, (full, expect_full)
    # and against the reference-API path on a slice
    sa = [mosaic.StageAllocation([mosaic.Entry(m, mosaic.DeploymentOption(d, u, L), g)
                                  for m, d, u, g in a]) for a in allocs[:400]]
    assert pl.stage_time(sa) == list(st[:400])
    pl.close()


def test_fast_path_reference_goldens():
    # every reference edge / large-cluster golden row through the fast path
    for name in ("stime_edge.json", "stime_large_g.json"):
        rows = load_golden(name)
        groups = {}
        for row in rows:
            if row["t"] is not None:
                groups.setdefault((row["inst"], tuple(row["extra"])), []).append(row)
        for (inst, extra), rs in groups.items():
            pl = planner(inst, extra=list(extra))
            ent, gpus, off = _pack([r["entries"] for r in rs])
            st = np.zeros(len(rs))
            pl.evaluate(ent, gpus, off, st)
            assert list(st) == [hexf(r["t"]) for r in rs], (name, inst, extra)
            pl.close()


def test_smem_peak_calibration():
    # SURVEY §8(d)'s on-chip roofline denominator: 128 B per clock per SM on a B200 is
    # 148 x 1.965 GHz x 128 B = 37.2 TB/s; the measured figure must be near it (not an
    # artefact such as loads the compiler folded away, which would read ~2x)
    bw = mosaic.smem_peak_gbs(0)
    assert 20_000 < bw < 40_000, bw
