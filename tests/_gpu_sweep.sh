for DD in 3 4 5; do for DP in 32 128; do
  echo "== depth $DD period $DP"
  MOSAIC_DON_DEPTH=$DD MOSAIC_DON_PERIOD=$DP MOSAIC_TRACE=1 timeout 120 python tests/_cfg5_probe.py cfg5 127 nosolve 2>&1 | grep -E "thr=0.0917677|thr=0.0918354|^mask" | sed 's/SolverStats.*//' | cut -c1-130
done; done
