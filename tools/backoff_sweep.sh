for B in 2048; do
  echo "backoff $B: full $(MOSAIC_BACKOFF_NS=$B timeout 60 python tools/prof_min.py 2>&1 | grep -o "ksearch_ms.: [0-9.]*")  rank0/8 $(MOSAIC_BACKOFF_NS=$B MOSAIC_SHARD_SIM=0/8 timeout 60 python tools/prof_min.py 2>&1 | grep -o "ksearch_ms.: [0-9.]*")  rank2/8 $(MOSAIC_BACKOFF_NS=$B MOSAIC_SHARD_SIM=2/8 timeout 60 python tools/prof_min.py 2>&1 | grep -o "ksearch_ms.: [0-9.]*")"
done
