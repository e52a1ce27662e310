# full cfg4 / cfg5 solves under knob settings
for r in 1 2; do
for K in "MOSAIC_DON_PERIOD=1" "MOSAIC_DON_PERIOD=4" "MOSAIC_DON_PERIOD=8" "MOSAIC_DON_PERIOD=4 MOSAIC_DEEP_AFTER=16384"; do
  for W in cfg4 cfg5; do
    echo "$K $W $(env $K timeout 600 python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.3f'%d['ms_per_step'], d['best_plan_iteration_time'])")"
  done
done; done
