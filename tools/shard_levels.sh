# per-rank share (8 ranks) of the dominant MIN proof for shard levels 1 and 2
for L in 1 2; do
  echo "level $L"; MOSAIC_SHARD_LEVEL=$L bash tools/shard_balance.sh 8
done
