#!/bin/bash
TAG=${1:-r2v}
O=gpurun_out
KG_SETUP_TIMES=1 KG_CAPTURE_TIMES=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29504 tools/e2e_breakdown.py --repeats 3 --rounds 900 > $O/${TAG}_e2e_n4.txt 2>&1; echo n4 rc=$?
KG_SETUP_TIMES=1 KG_CAPTURE_TIMES=1 timeout 600 python tools/e2e_breakdown.py --repeats 3 --rounds 900 > $O/${TAG}_e2e_n1.txt 2>&1; echo n1 rc=$?
