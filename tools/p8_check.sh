#!/bin/bash
# Diagnostic for the 8-partition job on a 4-GPU box: P = 8 partitions over 4
# ranks (2 per GPU) and over 1 rank (8 on one GPU) through bench.py --parts 8.
TAG=${1:-p8}
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 4 --parts 8 --steps 20 --warmup 5 \
  > gpurun_out/${TAG}_n4_p8.json 2> gpurun_out/${TAG}_n4_p8.err; echo n4p8 rc=$?
timeout 900 python bench.py --parts 8 --steps 20 --warmup 5 --no-cpu-baseline \
  > gpurun_out/${TAG}_n1_p8.json 2> gpurun_out/${TAG}_n1_p8.err; echo n1p8 rc=$?
