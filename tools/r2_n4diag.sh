#!/bin/bash
TAG=${1:-r2t}
O=gpurun_out
KG_SETUP_TIMES=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29504 bench.py --gpus 4 --steps 20 --warmup 5 > $O/${TAG}_bench_n4.json 2> $O/${TAG}_bench_n4.err; echo n4 rc=$?
timeout 900 python bench.py --parts 4 --steps 20 --warmup 5 --no-cpu-baseline > $O/${TAG}_n1_p4.json 2> $O/${TAG}_n1_p4.err; echo n1p4 rc=$?
