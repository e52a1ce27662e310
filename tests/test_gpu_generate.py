"""N2: surface generation on the device (k_gen_surfaces) against the
reference's own profile files and a Python restatement of evaluate_workload.

The restatement below follows profiler.hpp:56-89 operation for operation; Python floats are
IEEE fp64 with no contraction, so it is an exact oracle for the kernel (bit-exact bar)."""
import math

import pytest

from conftest import load_golden

mosaic = pytest.importorskip("paper_2605_18710_b200.mosaic")


def evaluate_workload(w, c, d, a, demand_scale=1.0):
    # profiler.hpp:57-59 sm_efficiency, :65-89 evaluate_workload
    eta = min(1.0, 0.85 + 0.15 * a / w.sm_efficiency_knee)
    compute_time = (w.flops_per_iter / d) / (a * c.peak_compute * eta)
    io_time = (w.bytes_per_iter / d) / c.peak_bandwidth
    sync_time = 0.0
    if d > 1:
        sync_time = (c.interconnect_alpha * math.ceil(math.log2(float(d))) +
                     c.interconnect_beta * w.gradient_bytes)
    dp_eff = 1.0 + w.dp_penalty * (d - 1)
    mx = io_time if compute_time < io_time else compute_time
    latency = mx * dp_eff + sync_time + w.fixed_overhead
    sm_active = min(1.0, compute_time / latency)
    bw = min(1.0, io_time / mx * demand_scale)
    memory = w.memory_act_base + w.memory_per_quota * a + w.gradient_bytes / d
    return (d, a, latency, bw, memory, sm_active)


def test_synth_workloads_shape():
    ws, c = mosaic.synth_workloads("cfg5")
    assert len(ws) == 8 and c.gpu_count == 128 and ws[-1].id == "backbone"


@pytest.mark.parametrize("inst", list(load_golden("io_files.json")))
def test_restatement_pinned_to_reference_profile_files(inst):
    # CPU: the Python restatement reproduces every point the reference's profiler wrote
    prof = load_golden("io_files.json")[inst]["files"]["profile"]["surfaces"]
    ws, c = mosaic.synth_workloads(inst)
    for w, s in zip(ws, prof):
        for p in s["points"]:
            assert evaluate_workload(w, c, p["d"], p["a"]) == (
                p["d"], p["a"], p["latency"], p["bandwidth_util"], p["memory"], p["sm_active"])


@pytest.mark.gpu
@pytest.mark.parametrize("inst", list(load_golden("io_files.json")))
def test_device_surfaces_equal_reference_profile_files(inst):
    # the profile JSON the reference wrote for this instance (io.hpp:131-174): every point
    prof = load_golden("io_files.json")[inst]["files"]["profile"]["surfaces"]
    ws, c = mosaic.synth_workloads(inst)
    got = mosaic.generate_surfaces(ws, c)
    assert [w.id for w in ws] == [s["module"] for s in prof]
    for pts, s in zip(got, prof):
        want = sorted(((p["d"], p["a"], p["latency"], p["bandwidth_util"], p["memory"],
                        p["sm_active"]) for p in s["points"]), key=lambda t: (t[0], t[1]))
        assert pts == want


@pytest.mark.gpu
@pytest.mark.parametrize("spec", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "random:3:6:32",
                                  "random:9:4:1024", "preset:imagebind:7:8"])
def test_device_surfaces_equal_restatement(spec):
    ws, c = mosaic.synth_workloads(spec)
    got = mosaic.generate_surfaces(ws, c)
    ds = [1 << i for i in range(c.gpu_count.bit_length()) if (1 << i) <= c.gpu_count]
    for w, pts in zip(ws, got):
        assert pts == [evaluate_workload(w, c, d, i / 10.0) for d in ds for i in range(1, 11)]


@pytest.mark.gpu
def test_device_surfaces_custom_grids():
    # granularity sweeps (PAPER Fig. 14b): non-default d / a grids and demand_scale
    ws, c = mosaic.synth_workloads("cfg4")
    for ds, As, dsc in [([1, 2, 3, 5, 8, 64], [i / 32 for i in range(1, 33)], 1.0),
                        ([1, 4, 16], [0.05, 0.5, 1.0], 2.5)]:
        got = mosaic.generate_surfaces(ws, c, ds, As, dsc)
        for w, pts in zip(ws, got):
            assert pts == [evaluate_workload(w, c, d, a, dsc) for d in ds for a in As]


@pytest.mark.gpu
def test_device_surfaces_feed_the_planner():
    # generate on device -> from_surfaces -> solve == the synthetic problem's plan
    ws, c = mosaic.synth_workloads("cfg3")
    pts = mosaic.generate_surfaces(ws, c)
    ref = mosaic.Planner.from_spec("cfg3")
    pp = ref._owned.contents
    mods = [{"id": w.id, "memory_base": pp.modules[i].memory_base, "points": pts[i]}
            for i, w in enumerate(ws)]
    edges = [(pp.edges[2 * i], pp.edges[2 * i + 1]) for i in range(pp.n_edges)]
    pl = mosaic.Planner.from_surfaces(mods, edges, c.gpu_count, quota_levels=pp.quota_levels)
    a, b = pl.solve().plan, ref.solve().plan
    assert a.predicted_iteration_time == b.predicted_iteration_time
    assert [[(e.module, e.option.dp_degree, e.option.quota_units, e.gpus) for e in s.entries]
            for s in a.stages] == [[(e.module, e.option.dp_degree, e.option.quota_units, e.gpus)
                                    for e in s.entries] for s in b.stages]
