# Whole 7-encoder stage_eval (device ms of all its searches), knob combinations given as args
for k in "$@"; do
  [ "$k" = "-" ] && k=""
  a=""; for kv in $k; do a="$a --knob $kv"; done
  for rep in 1 2; do python tools/tune.py cfg5 --mask 127 $a 2>&1 | tail -1 | sed "s/^/[$k] /"; done
done
