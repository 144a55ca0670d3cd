#!/bin/bash
# Peer-memory payload exchange (csrc/kg_peer.cu) on a 4-GPU box: bitwise check
# against the single-process run at 2 and 4 ranks, then bench A/B against the
# NCCL all-gather (KG_PEER_GATHER=0).
TAG=${1:-peer}
for N in 2 4; do
  KG_PEER_GATHER=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29600 + N)) tools/dist_check.py > gpurun_out/${TAG}_dist_n$N.json 2> gpurun_out/${TAG}_dist_n$N.err
  echo dist n$N rc=$?; tail -c 300 gpurun_out/${TAG}_dist_n$N.json
done
for N in 2 4; do
  for PG in 1 0; do
    KG_PEER_GATHER=$PG timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port $((29610 + N + 10 * PG)) bench.py --gpus $N --steps 20 --warmup 5 \
      > gpurun_out/${TAG}_bench_n${N}_pg$PG.json 2> gpurun_out/${TAG}_bench_n${N}_pg$PG.err
    echo bench n$N pg$PG rc=$?
  done
done
