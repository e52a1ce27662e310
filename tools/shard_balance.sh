# Per-rank share of the dominant MIN proof when sharded over W ranks (run sequentially on one GPU)
W=${1:-8}
for r in $(seq 0 $((W-1))); do
  echo "rank $r/$W: $(MOSAIC_SHARD_SIM=$r/$W timeout 60 python tools/prof_min.py 2>&1 | grep -o "ksearch_ms.: [0-9.]*")"
done
