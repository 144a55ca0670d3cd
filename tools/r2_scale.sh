#!/bin/bash
# bench.py at N = 1, 2, 4 (driver launch), one box
TAG=${1:-r2w}
O=gpurun_out
timeout 600 python bench.py > $O/${TAG}_bench_n1.json 2> $O/${TAG}_bench_n1.err; echo n1 rc=$?
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29500 + N)) bench.py --gpus $N --steps 20 --warmup 5 \
    > $O/${TAG}_bench_n$N.json 2> $O/${TAG}_bench_n$N.err; echo n$N rc=$?
done
