# full cfg4 / cfg5 solves vs the small-tree threshold (searches below it: 8 CTAs, no hand-overs)
for T in 2e5 1e6 5e6 5e4; do
  for W in cfg4 cfg5; do
    echo "SMALL_TREE=$T $W $(MOSAIC_SMALL_TREE=$T timeout 600 python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.3f'%d['ms_per_step'], d['best_plan_iteration_time'])")"
  done
done
