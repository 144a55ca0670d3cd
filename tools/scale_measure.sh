#!/bin/bash
# Weak-scaling set on one box (run under gpurun --gpus 4): bench.py at N = 2
# and N = 4 ranks over NCCL, launched as the driver launches it.
TAG=${1:-scale}
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29500 + N)) bench.py --gpus $N --steps 20 --warmup 5 \
    > gpurun_out/${TAG}_bench_n$N.json 2> gpurun_out/${TAG}_bench_n$N.err; echo n$N rc=$?
done
