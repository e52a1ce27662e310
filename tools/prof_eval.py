"""ncu target: a few K1 evaluator launches on 2^20 random cfg5 allocations (no solve)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tools")]
import torch  # noqa: E402

from evalgen import random_allocations  # noqa: E402
from paper_2605_18710_b200 import mosaic  # noqa: E402

pl = mosaic.Planner.from_spec(sys.argv[1] if len(sys.argv) > 1 else "cfg5", device=0)
ent, gpus, off = random_allocations(pl, 1 << 20, seed=0)
dev = torch.device("cuda", 0)
tE, tG, tO = (torch.from_numpy(x).to(dev) for x in (ent, gpus, off))
st = torch.empty(len(off) - 1, dtype=torch.float64, device=dev)
torch.cuda.synchronize()
for _ in range(3):
    pl.evaluate(tE, tG, tO, st, None, device=True)
s = pl.evaluate_stats()
print(s, "per launch ms", s["kernel_ms"] / s["launches"],
      "GB/s", s["alg_bytes"] / s["kernel_ms"] * 1e3 / 1e9)
