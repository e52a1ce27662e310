"""Sharded search on ONE device (share_all): the cfg5 7-encoder stage_eval with every large
search split into W option-prefix shards in one launch and merged by the multi-GPU rule,
with and without incumbent sharing between the shards (share_peers).  All shards share one
GPU, so device time ~ the sum of the shards' work: time(W) / time(1) is how much more work
a W-way split does.  Results must equal the unsharded stage_eval bit for bit.
usage: python tools/shard_sim.py [mask_hex] [W ...]"""
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18710_b200 import mosaic  # noqa: E402

mask = int(sys.argv[1], 16) if len(sys.argv) > 1 else 0x7f
Ws = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
mods = [i for i in range(8) if mask >> i & 1]
pl = mosaic.Planner.from_spec("cfg5", device=0)
pl.stage_eval([0, 1, 2])


def run(W, peers):
    pl.set_tuning(share_all=W if W > 1 else 0, share_peers=peers)
    pl.clear_cache()
    pl.reset_counters()
    r = pl.stage_eval(mods)
    c = pl.counters()
    sig = (r.stage_time, r.stats.feasibility_calls,
           [(e.module, e.option.dp_degree, e.option.quota_units, tuple(e.gpus))
            for e in r.allocation.entries])
    return c["device_ms"], r.stats.nodes, sig


base_ms, base_nodes, base_sig = run(1, 1)
print(f"mask {mask:#x} unsharded: {base_ms:8.1f} ms  nodes {base_nodes}", flush=True)
for W in Ws:
    if W == 1:
        continue
    for peers in (0, 1):
        ms, nodes, sig = run(W, peers)
        print(f"W={W} share_peers={peers}: {ms:8.1f} ms ({ms / base_ms:4.2f}x)  nodes {nodes} "
              f"({nodes / base_nodes:4.2f}x)  same={sig == base_sig}", flush=True)
        assert sig == base_sig, "sharded result differs from the unsharded one"
