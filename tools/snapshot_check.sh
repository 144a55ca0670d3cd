#!/bin/bash
# Multi-rank final-parameter assembly: bitwise check against the single-process
# run (tools/dist_check.py) and the e2e leg of bench.py at 2 and 4 ranks.
TAG=${1:-snap}
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29700 + N)) tools/dist_check.py > gpurun_out/${TAG}_dist_n$N.json 2> gpurun_out/${TAG}_dist_n$N.err
  echo dist n$N rc=$?; grep -o '"bitwise_equal": [a-z]*' gpurun_out/${TAG}_dist_n$N.json
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29710 + N)) bench.py --gpus $N --steps 20 --warmup 5 \
    > gpurun_out/${TAG}_bench_n$N.json 2> gpurun_out/${TAG}_bench_n$N.err; echo bench n$N rc=$?
done
