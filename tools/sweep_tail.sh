# Tail splitting sweep on the 7-encoder stage (trace=3 timelines into gpurun_out/tl_*.log)
mkdir -p gpurun_out
for k in "$@"; do
  [ "$k" = "-" ] && k=""
  f=gpurun_out/tl_$(echo "$k" | tr ' =' '__').log
  python tools/timeline7.py $k > $f 2>&1
  echo "== $k"; grep -A1 "kernel=[0-9][0-9][0-9]*\.[0-9]*ms" $f | cut -c1-200
done
