"""Sharded search end to end: two ranks on one GPU (--same-device), gloo
all-gather once per device search.  Every rank must replay the same control flow, so each
merged search result has to be identical on all ranks (a divergence deadlocks the
all-gather); the plan must equal the single-GPU / reference plan bit for bit."""
import json
import os
import subprocess
import sys

import pytest

from conftest import hexf, load_golden

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("workload,port", [("cfg3", 29561), ("cfg4", 29562)])
def test_two_ranks_same_plan(workload, port):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--workload",
           workload, "--steps", "1", "--warmup", "3", "--dist-backend", "gloo",
           "--same-device", "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=240)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2
    gold = load_golden("configs.json")[workload]["solve"]
    assert line["best_plan_iteration_time"] == hexf(gold["iteration_time"])
    # the two ranks mapped each other's search control blocks (CUDA IPC) for in-search
    # incumbent / earliest-hit sharing
    assert line["full_solve"]["peer_links"] == 1, line["full_solve"]


def test_bench_spawns_ranks_for_gpus_flag():
    # `bench.py --gpus 2` launches its own two ranks (torchrun) when not started by one; on
    # one GPU both share cuda:0 (--same-device, gloo).  The headline line must report both
    # ranks, weak scaling (each rank runs its own copy of the cfg5 sample, stage times checked
    # against the reference's inside bench.py) and the sharded full solve's plan.
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--same-device", "--dist-backend", "gloo",
           "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--no-evaluator"]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["same_config"] is True and line["value"] > 0
    assert line["scaling"] == "weak"
    traj = load_golden("trajectory_gpu.json")["cfg5@L32"]
    assert line["best_plan_iteration_time"] == hexf(traj["iteration_time"])


def test_in_library_nccl_plane_world1():
    # the library's own NCCL communicator (mosaic_gpu_nccl_id / mosaic_gpu_set_shard_nccl):
    # with one rank the full merge path (record upload, ncclAllGather, merge) runs on every
    # batched launch and the plans must not change
    from paper_2605_18710_b200 import mosaic
    gold = load_golden("configs.json")
    for w in ("cfg3", "cfg4"):
        pl = mosaic.Planner.from_spec(w, device=0)
        pl.set_shard_nccl(0, 1, mosaic.nccl_unique_id())
        r = pl.solve()
        assert r.plan.predicted_iteration_time == hexf(gold[w]["solve"]["iteration_time"])
        pl.close()


def _sig(r):
    return (r.stage_time, r.stats.feasibility_calls,
            [(e.module, e.option.dp_degree, e.option.quota_units, tuple(e.gpus))
             for e in r.allocation.entries])


@pytest.mark.parametrize("W", [2, 4, 8])
def test_share_all_shards_equal_unsharded(W):
    # every large search split into W option-prefix shards in ONE launch, merged by the
    # multi-GPU rule, with and without in-search incumbent / earliest-hit sharing between the
    # shards: stage_evals and exact stages identical to the unsharded ones, the cfg4 plan
    # equal to the reference's
    mosaic = pytest.importorskip("paper_2605_18710_b200.mosaic")
    pl = mosaic.Planner.from_spec("cfg5", device=0)
    masks = [[0, 1, 2, 3], [0, 2, 3, 4], [0, 1, 2, 3, 4], [0, 2, 3, 4, 5]]
    base = [_sig(pl.stage_eval(m)) for m in masks]
    ex_base = [_sig(pl.exact_stage(m)) for m in masks[:2]]
    for peers in (0, 1):
        pl.set_tuning(share_all=W, share_peers=peers)
        pl.clear_cache()
        assert [_sig(pl.stage_eval(m)) for m in masks] == base, (W, peers)
        assert [_sig(pl.exact_stage(m)) for m in masks[:2]] == ex_base, (W, peers)
    pl.set_tuning(share_all=0, share_peers=1)
    pl.close()
    gold = load_golden("configs.json")["cfg4"]["solve"]
    p4 = mosaic.Planner.from_spec("cfg4", device=0)
    p4.set_tuning(share_all=W)
    assert p4.solve().plan.predicted_iteration_time == hexf(gold["iteration_time"])
    p4.close()


def test_bench_strong_scaling_deals_the_sample():
    # --scaling strong: the 29 stage_evals dealt over the ranks (fixed total work)
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--same-device", "--dist-backend", "gloo",
           "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--no-evaluator",
           "--scaling", "strong"]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong" and line["value"] > 0


def test_local_handover_on_off_identical():
    # CTA-local hand-off of search pieces (shared-memory slot) on and off: identical results
    mosaic = pytest.importorskip("paper_2605_18710_b200.mosaic")
    pl = mosaic.Planner.from_spec("cfg5", device=0)
    masks = [[0, 1, 2, 3], [0, 2, 3, 4], [0, 1, 2, 3, 4]]
    res = {}
    for lh in (1, 0):
        pl.set_tuning(local_handover=lh)
        pl.clear_cache()
        res[lh] = ([_sig(pl.stage_eval(m)) for m in masks],
                   [_sig(pl.exact_stage(m)) for m in masks[:2]])
    assert res[0] == res[1]
    pl.close()
