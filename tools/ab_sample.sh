# A/B(/C) of the bench sample and the 7-encoder stage: libraries under ab/ and in-tree, alternating
LIBS="${LIBS:-ab/lib_old.so paper_2605_18710_b200/libmosaic_gpu.so}"
for i in 1 2 3; do
  for L in $LIBS; do
    MOSAIC_LIB=$PWD/$L python bench.py --steps 30 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['ms_per_step'],4), d.get('time_to_best_plan_s'))"
    MOSAIC_LIB=$PWD/$L python tools/tune.py cfg5 --mask 127 2>&1 | tail -1 | sed "s|^|$L |" | cut -c1-140
  done
done
