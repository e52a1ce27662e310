"""Per-shard work of the cfg5 7-encoder stage_eval split W ways (share_all, shared incumbents):
node counts of every shard of each large launch (trace=1), max/mean = the load imbalance a
W-GPU run would see with the static option-prefix split."""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ROOT)
    from paper_2605_18710_b200 import mosaic
    pl = mosaic.Planner.from_spec("cfg5", device=0)
    pl.stage_eval([0, 1, 2])
    pl.set_tuning(share_all=int(sys.argv[2]), trace=1)
    pl.stage_eval(list(range(7)))
    sys.exit(0)
for W in [int(x) for x in sys.argv[1:]] or [2, 4, 8]:
    err = subprocess.run([sys.executable, __file__, "child", str(W)], capture_output=True,
                         text=True).stderr
    launches = {}
    for line in err.splitlines():
        m = re.search(r"\] (MIN|FIRST)\s+k=7 thr=(\S+) batch=(\d+) ctas=\d+ kernel=([\d.]+)ms .*nodes=(\d+)", line)
        if m and int(m.group(3)) == W:
            launches.setdefault((m.group(1), m.group(2), m.group(4)), []).append(int(m.group(5)))
    for (mode, thr, kms), nodes in launches.items():
        if float(kms) < 20:
            continue
        mean = sum(nodes) / len(nodes)
        print(f"W={W} {mode} thr={thr} kernel {kms} ms: shard nodes {nodes} "
              f"max/mean {max(nodes) / mean:.2f}", flush=True)
