for DP in 4 2 1; do
  echo "period $DP: full $(MOSAIC_DON_PERIOD=$DP timeout 60 python tools/prof_min.py 2>&1 | grep -o "ksearch_ms.: [0-9.]*")  rank0/8 $(MOSAIC_DON_PERIOD=$DP MOSAIC_SHARD_SIM=0/8 timeout 60 python tools/prof_min.py 2>&1 | grep -o "ksearch_ms.: [0-9.]*")"
done
MOSAIC_TRACE=1 timeout 300 python tools/cfg5_probe.py cfg5 127 nosolve 2>&1 | grep -E "thr=0.0918354" | cut -c1-90
