"""Synthetic batches of explicit stage allocations for the K1 evaluator (bench + tests).

Each allocation takes a random subset of the modules (sorted by index, as StageAllocation
requires); every entry uses one of its module's candidate options (candidate_options order,
stage_eval.hpp:68-93) and a window of d consecutive GPUs starting at a random GPU (wrapping).
Returned as the flat arrays mosaic_gpu_evaluate reads (include/mosaic_gpu.h).
"""
from __future__ import annotations

import numpy as np


def random_allocations(planner, n: int, seed: int = 0, max_k: int | None = None):
    rng = np.random.default_rng(seed)
    M, G = planner.n_modules, planner.gpu_count
    max_k = min(M, max_k or M)
    opt_d, opt_u, opt_n, opt_off = [], [], [], [0]
    for m in range(M):
        rows = planner.candidate_options(m)
        opt_d += [r.opt.dp_degree for r in rows]
        opt_u += [r.opt.quota_units for r in rows]
        opt_n.append(len(rows))
        opt_off.append(opt_off[-1] + len(rows))
    opt_d, opt_u = np.array(opt_d, np.int32), np.array(opt_u, np.int32)
    opt_n, opt_off = np.array(opt_n, np.int64), np.array(opt_off[:-1], np.int64)
    k = rng.integers(1, max_k + 1, size=n)
    # first k columns of a random permutation per allocation, then sorted
    perm = np.argsort(rng.random((n, M)), axis=1)
    take = np.arange(M)[None, :] < k[:, None]
    mods = np.where(take, perm, M)  # M sorts last
    mods.sort(axis=1)
    module = mods[mods < M].astype(np.int32)
    ne = module.size
    row = opt_off[module] + (rng.random(ne) * opt_n[module]).astype(np.int64)
    d, u = opt_d[row], opt_u[row]
    gpu_off = np.zeros(ne, np.int64)
    np.cumsum(d[:-1], out=gpu_off[1:])
    total = int(gpu_off[-1] + d[-1]) if ne else 0
    start = rng.integers(0, G, size=ne)
    ent_of = np.repeat(np.arange(ne), d)
    pos = np.arange(total, dtype=np.int64) - gpu_off[ent_of]
    gpus = ((start[ent_of] + pos) % G).astype(np.int32)
    alloc_off = np.zeros(n + 1, np.int64)
    np.cumsum(k, out=alloc_off[1:])
    from paper_2605_18710_b200.mosaic import pack_eval_entries
    entries = pack_eval_entries(module, d, u, d, gpu_off)
    return entries, gpus, alloc_off


def to_allocations(entries, gpus, alloc_off, levels: int, lo: int, hi: int):
    """Allocations [lo, hi) as mosaic StageAllocations (for the reference-API paths)."""
    from paper_2605_18710_b200 import mosaic
    out = []
    for a in range(lo, hi):
        ents = []
        for e in range(int(alloc_off[a]), int(alloc_off[a + 1])):
            m, d, u, ng = (int(x) for x in entries[e, :4])
            off = int(entries[e, 6:8].copy().view(np.int64)[0])
            ents.append(mosaic.Entry(m, mosaic.DeploymentOption(d, u, levels),
                                     [int(x) for x in gpus[off:off + ng]]))
        out.append(mosaic.StageAllocation(ents))
    return out
