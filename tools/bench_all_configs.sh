# time-to-best-plan for every BASELINE config (ours), plus the reference CPU solve() on this host
for W in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python3 -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$W', 'ms_per_step=%.3f'%d['ms_per_step'], 'plan=%r'%d['best_plan_iteration_time'], 'launches=%d'%d['gpu_launches'], 'e2e_plans_s=%.0f'%d['e2e']['value'])"
done
for W in cfg1 cfg2 cfg3 cfg4; do
  taskset -c 0 ./oracle/_ref/ref_driver $W solve reps=5 | python3 -c "
import json,sys; d=json.load(sys.stdin); t=sorted(d.get('times',[]))
print('$W reference solve() median %.3f ms'%(1000*t[len(t)//2]) if t else 'n/a')"
done
