# Sharding test on ONE GPU: 2 ranks share cuda:0 and all-gather over gloo.
# (Real multi-GPU runs use NCCL: python -m torch.distributed.run --nproc-per-node N bench.py --gpus N)
set -x
W=${1:-cfg4}
timeout ${T:-600} python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29531 bench.py --workload $W --steps 1 --warmup 3 --dist-backend gloo --same-device \
  --no-cpu-baseline
