set -x
for W in cfg4 cfg5; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --workload $W --steps 1 --warmup 3 --dist-backend gloo --same-device --no-cpu-baseline > gpurun_out/multi2_$W.json 2> gpurun_out/multi2_$W.err
  tail -c 700 gpurun_out/multi2_$W.json; tail -3 gpurun_out/multi2_$W.err
done
