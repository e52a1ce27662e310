"""MIN proof of the 7-encoder cfg5 stage at T* under different level orders (any order gives
the same T*; the order only changes the tree's size).  Each order runs in its own process
under a time cap (a bad order can take minutes).
usage: python tools/min_perm7.py [seed] [count] [cap_s]"""
import os
import random
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
T_HEX = "0x1.77e16c9919003p-4"
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ROOT)
    from paper_2605_18710_b200 import mosaic
    pl = mosaic.Planner.from_spec("cfg5", device=0)
    kind, val = sys.argv[2], int(sys.argv[3])
    pl.set_tuning(**{kind: val})
    pl.reset_counters()
    t = pl.stage_min(list(range(7)), float.fromhex(T_HEX), restart=False)
    assert t.hex() == T_HEX, t.hex()
    print(f"{kind}={val}: {pl.counters()['device_ms']:.1f} ms", flush=True)
    sys.exit(0)
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
count = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cap = float(sys.argv[3]) if len(sys.argv) > 3 else 8.0
random.seed(seed)
runs = [("min_order", m) for m in (0, 2, 4)] + [("min_perm", p) for p in random.sample(range(1, 5041), count)]
for kind, val in runs:
    try:
        out = subprocess.run([sys.executable, __file__, "child", kind, str(val)],
                             capture_output=True, text=True, timeout=cap)
        print(out.stdout.strip() or f"{kind}={val}: failed {out.stderr[-200:]}", flush=True)
    except subprocess.TimeoutExpired:
        print(f"{kind}={val}: > {cap:.0f} s (incl. start-up)", flush=True)
