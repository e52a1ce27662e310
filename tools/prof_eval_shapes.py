"""K1 fast-path time per allocation for allocation shapes (entries x GPUs per entry), to split
the kernel's per-allocation fixed cost from its per-id and per-slot costs."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tools")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_18710_b200 import mosaic  # noqa: E402

pl = mosaic.Planner.from_spec("cfg5", device=0)
dev = torch.device("cuda", 0)
opts = [[(r.opt.dp_degree, r.opt.quota_units) for r in pl.candidate_options(m)] for m in range(8)]
N = 1 << 20
for k, d in [(1, 1), (1, 32), (4, 1), (4, 8), (4, 32), (8, 16), (8, 64)]:
    rng = np.random.default_rng(0)
    mods = np.tile(np.arange(k), N)
    dd, uu = [], []
    for m in range(k):
        cand = [o for o in opts[m] if o[0] == d] or [opts[m][0]]
        dd.append(cand[0][0])
        uu.append(cand[0][1])
    d_arr = np.tile(np.array(dd), N)
    u_arr = np.tile(np.array(uu), N)
    ng = d_arr
    off = np.zeros(len(mods), np.int64)
    np.cumsum(ng[:-1], out=off[1:])
    total = int(off[-1] + ng[-1])
    starts = rng.integers(0, 128, size=len(mods))
    ent_of = np.repeat(np.arange(len(mods)), ng)
    pos = np.arange(total) - off[ent_of]
    gpus = ((starts[ent_of] + pos) % 128).astype(np.int32)
    ent = mosaic.pack_eval_entries(mods, d_arr, u_arr, ng, off)
    aoff = np.arange(N + 1, dtype=np.int64) * k
    tE, tG, tO = (torch.from_numpy(x).to(dev) for x in (ent, gpus, aoff))
    st = torch.empty(N, dtype=torch.float64, device=dev)
    for _ in range(3):
        pl.evaluate(tE, tG, tO, st, None, device=True)
    pl.reset_counters()
    for _ in range(5):
        pl.evaluate(tE, tG, tO, st, None, device=True)
    s = pl.evaluate_stats()
    ms = s["fast_kernel_ms"] / s["launches"]
    gbs = s["alg_bytes"] / s["launches"] / (s["kernel_ms"] / s["launches"] / 1e3) / 1e9
    print(f"k={k} d={d}: {ms:.3f} ms per 2^20 ({ms * 1e6 / N:.2f} ns/alloc), "
          f"{gbs:.0f} GB/s, full-path allocs {s['full_path_allocs']}", flush=True)
