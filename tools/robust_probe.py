# full solves of larger synthetic instances (robustness of the hand-over policy)
import sys, time
sys.path.insert(0, '.')
import paper_2605_18710_b200.mosaic as m
for spec, L in [("preset:ofasys:8:32", 32), ("preset:ofasys:8:64", 32), ("preset:imagebind:7:64", 16),
                ("preset:ofasys:10:32", 16), ("random:11:7:64", 16)]:
    pl = m.Planner.from_spec(spec, quota_levels=L)
    t = time.time()
    r = pl.solve()
    print(spec, L, "%.3fs" % (time.time() - t), r.plan.predicted_iteration_time, flush=True)
    pl.close()
