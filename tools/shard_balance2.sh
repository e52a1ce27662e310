for DD in 2 3; do for r in 0 5; do
  echo "depth $DD rank $r/8: $(MOSAIC_DON_DEPTH=$DD MOSAIC_SHARD_SIM=$r/8 timeout 60 python tools/prof_min.py 2>&1 | grep -o "ksearch_ms.: [0-9.]*")"
done; done
for DD in 2; do echo "depth $DD full: $(MOSAIC_DON_DEPTH=$DD timeout 60 python tools/prof_min.py 2>&1 | grep -o "ksearch_ms.: [0-9.]*")"; done
