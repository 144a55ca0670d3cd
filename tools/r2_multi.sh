#!/bin/bash
# Round-2 multi-GPU set (gpurun --gpus 4): bitwise dist check at 2/4 ranks
# (NCCL and peer exchange), weak-scaling bench at N = 2 and 4 (driver launch),
# reference arm at N = 4, the P = 8 job over 4 ranks (diagnostic).
TAG=${1:-r2s}
O=gpurun_out
for N in 2 4; do
  for PG in 0 1; do
    KG_PEER_GATHER=$PG timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29600 + N + 10 * PG)) tools/dist_check.py > $O/${TAG}_dist_n${N}_pg$PG.json 2> $O/${TAG}_dist_n${N}_pg$PG.err
    echo dist n$N pg$PG rc=$?; tail -c 200 $O/${TAG}_dist_n${N}_pg$PG.json
  done
done
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29500 + N)) bench.py --gpus $N --steps 20 --warmup 5 \
    > $O/${TAG}_bench_n$N.json 2> $O/${TAG}_bench_n$N.err; echo bench n$N rc=$?
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29540 bench.py --impl reference --gpus 4 --steps 2 --warmup 1 \
  > $O/${TAG}_bench_ref_n4.json 2> $O/${TAG}_bench_ref_n4.err; echo ref n4 rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 4 --parts 8 --steps 20 --warmup 5 --no-e2e \
  > $O/${TAG}_n4_p8.json 2> $O/${TAG}_n4_p8.err; echo n4p8 rc=$?
