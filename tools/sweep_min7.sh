M="--mask 127 --min-at 0x1.77e16c9919003p-4"
for k in "" "backoff_ns=512" "backoff_ns=8192" "backoff_ns=32768" "don_period=2" "don_period=8" "deep_after=4096" "deep_after=65536" "ring_per_walker=4"; do
  if [ -z "$k" ]; then python tools/tune.py cfg5 $M; else python tools/tune.py cfg5 $M --knob $k; fi 2>&1 | tail -1 | sed "s/^/$k: /"
done
