"""CPU, world_size 2 over gloo: the per-rank search records cross ranks through an
all-gather and every rank picks the same winner with the library's merge
(mosaic_gpu_merge_records) — the host half of the sharded search (bench.py N>1)."""
import os
import struct

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_18710_b200 import mosaic
    import torch

    # rank r found a FIRST hit at global item 10 - r and a MIN value 0.5 + r/10
    first = struct.pack("<Qd", 10 - rank, 0.0)
    mini = struct.pack("<Qd", rank, 0.5 + rank / 10)
    out = []
    for rec, mode in ((first, 1), (mini, 0)):
        t = torch.frombuffer(bytearray(rec), dtype=torch.uint8)
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        buf = b"".join(bytes(p.numpy().tobytes()) for p in parts)
        out.append(mosaic.merge_records(buf, world, mode))
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
    assert res[0] == res[1] == [1, 0]
