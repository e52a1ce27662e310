import time, sys
sys.path.insert(0, '.')
import paper_2605_18710_b200.mosaic as m
for cfg in ['cfg1','cfg2','cfg3','cfg4']:
    t=time.time(); pl=m.Planner.from_spec(cfg); r=pl.solve(); dt=time.time()-t
    print(cfg, r.plan.predicted_iteration_time.hex(), r.plan.predicted_iteration_time, 'stages', len(r.plan.stages), 'searches', r.trace.gpu_searches, 'nodes', r.trace.nodes, 'leaves', r.trace.leaves, 'feas', r.trace.feasibility_calls, f'{dt:.3f}s', 'launches', pl.launch_count(), flush=True)
pl=m.Planner.from_spec('cfg5')
for mask in [3,7,15,31]:
    mods=[i for i in range(8) if mask>>i&1]
    t=time.time(); r=pl.stage_eval(mods); dt=time.time()-t
    print('cfg5 mask',mask, r.stage_time.hex(), r.stats, f'{dt:.3f}s', flush=True)
