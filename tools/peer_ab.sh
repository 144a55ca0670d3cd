#!/bin/bash
# Bench A/B of the peer-memory exchange vs the NCCL all-gather at 2 and 4 ranks
# (alternating, twice each), plus the 1-GPU peer unit tests.
TAG=${1:-peerab}
timeout 300 python -m pytest tests/test_gpu_peer.py -q -p no:cacheprovider 2>&1 | tail -2
KG_PEER_GATHER=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29602 tools/dist_check.py > gpurun_out/${TAG}_dist_n2.json 2>&1; echo dist rc=$?
for N in 2 4; do
  for rep in 1 2; do
    for PG in 1 0; do
      KG_PEER_GATHER=$PG timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
        --master-addr 127.0.0.1 --master-port $((29610 + N + 10 * PG + 20 * rep)) bench.py --gpus $N --steps 20 \
        --warmup 5 --no-e2e > gpurun_out/${TAG}_bench_n${N}_pg${PG}_$rep.json 2> gpurun_out/${TAG}_bench_n${N}_pg${PG}_$rep.err
      echo bench n$N pg$PG rep$rep rc=$?
    done
  done
done
