# per-search latency floor: repeated tiny searches (cfg2 singletons), host wall vs device
import sys, time
sys.path.insert(0, '.')
import paper_2605_18710_b200.mosaic as m
pl = m.Planner.from_spec('cfg2')
for _ in range(20): pl.stage_min([0], restart=False)
pl.reset_counters()
t = time.perf_counter(); N = 200
for _ in range(N): pl.stage_min([0], restart=False)
dt = (time.perf_counter() - t) / N
c = pl.counters()
print(f"per search: wall {dt*1e6:.1f} us, k_search {c['ksearch_ms']*1e3/N:.1f} us, device span {c['device_ms']*1e3/N:.1f} us")
