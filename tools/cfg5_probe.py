import time, sys
sys.path.insert(0, '.')
import paper_2605_18710_b200.mosaic as m
pl = m.Planner.from_spec(sys.argv[1] if len(sys.argv) > 1 else 'cfg5')
for mask in [int(x) for x in (sys.argv[2].split(',') if len(sys.argv) > 2 else ['63', '127'])]:
    mods=[i for i in range(8) if mask>>i&1]
    t=time.time(); r=pl.stage_eval(mods); dt=time.time()-t
    print('mask',mask, r.stage_time.hex(), r.stage_time, r.stats, f'{dt:.3f}s', pl.counters(), flush=True)
if len(sys.argv) <= 3:
    t=time.time(); r=pl.solve(); dt=time.time()-t
    print('solve', r.plan.predicted_iteration_time, [hex(x.chosen_x|x.chosen_y) for x in r.trace.rounds], r.trace.stage_eval_calls, r.trace.feasibility_calls, r.trace.leaves, f'{dt:.3f}s', flush=True)
