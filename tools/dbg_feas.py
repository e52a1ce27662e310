import sys, json
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from paper_2605_18710_b200 import mosaic
from trajectory import load_ref, load_gpu, bits, done
REF = load_ref()
pl = mosaic.Planner.from_spec("preset:ofasys:8:64", quota_levels=10, device=0)
for key, r in REF.items():
    if not key.startswith("preset:ofasys:8:64@L10|feas") or not done(r): continue
    m = int(key.rsplit("|", 1)[1]); o = r["out"]
    try:
        g = pl.feasibility_run(bits(m), float.fromhex(o["tau"]))
        print(key, "ok", g is not None, o["feasible"], flush=True)
    except Exception as e:
        print(key, "ERR", e, flush=True)
        pl.close(); pl = mosaic.Planner.from_spec("preset:ofasys:8:64", quota_levels=10, device=0)
