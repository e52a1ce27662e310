# time-to-best-plan per config with the child look-ahead off (0), one level (1), all (12)
for LA in 0 1 12; do
  for W in cfg3 cfg4 cfg5; do
    MOSAIC_LOOKAHEAD=$LA timeout 600 python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python3 -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('LA=$LA $W ms_per_step=%.3f plan=%r'%(d['ms_per_step'], d['best_plan_iteration_time']))"
  done
done
