"""Where the e2e time goes: context creation vs its first batched sample vs later ones."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18710_b200 import mosaic  # noqa: E402

S = json.load(open(os.path.join(ROOT, "tests", "golden", "cfg5_sample.json")))
sets = [[i for i in range(8) if m["mask"] >> i & 1] for m in S["masks"]]
for it in range(4):
    t0 = time.perf_counter()
    p = mosaic.Planner.from_spec("cfg5", device=0)
    t1 = time.perf_counter()
    p.reset_counters()
    for b in range(3):
        tb = time.perf_counter()
        p.search(sets)
        c = p.counters()
        p.reset_counters()
        print(f"ctx {it} batch {b}: wall {1e3*(time.perf_counter()-tb):.3f} ms, kernel "
              f"{c['ksearch_ms']:.3f} ms in {c['ksearch_launches']} launches, dev "
              f"{c['device_ms']:.3f} ms", flush=True)
    t2 = time.perf_counter()
    p.close()
    print(f"ctx {it}: create {1e3*(t1-t0):.3f} ms close {1e3*(time.perf_counter()-t2):.3f} ms")
