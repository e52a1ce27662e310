"""CPU, world_size 2 over gloo: every rank's RankRecord of a sharded search crosses ranks
through an all-gather and each rank applies the engine's own merge (Engine::merge_ranks via
mosaic_gpu_merge_ranks) — the host half of the multi-GPU search (bench.py N>1).  All ranks
must leave with the same answer."""
import os

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_18710_b200 import mosaic
    import torch

    # FIRST: rank 0 hit at option 3, rank 1 at option 1 -> rank 1's hit precedes.
    # MIN: rank 0 holds 0.4, rank 1 0.4 too (tie -> lowest rank), rank 1 restarted.
    first = mosaic.rank_record(True, 0.0, [(0, [8]), (3 - 2 * rank, [5, 3])],
                               leaf_value=10.0 + rank)
    mini = mosaic.rank_record(True, 0.4, [(rank, [8])], aborted=(rank == 1),
                              leaf_value=0.4)
    out = []
    for rec, mode, k in ((first, 1, 2), (mini, 0, 1)):
        t = torch.frombuffer(bytearray(rec), dtype=torch.uint8)
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        buf = b"".join(bytes(p.numpy().tobytes()) for p in parts)
        m = mosaic.merge_ranks(buf, world, mode, k)
        out.append((m["winner"], m["found"], m["aborted"], m["leaf_value"]))
    q.put((rank, out))
    dist.destroy_process_group()


def test_gloo_world2_merge():
    pytest.importorskip("paper_2605_18710_b200.mosaic")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res[0] == res[1] == [(1, True, False, 11.0), (0, True, True, 0.4)]
