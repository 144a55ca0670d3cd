#!/bin/bash
# ncu --set full of the top kernels of a short bench run (1 GPU); the plain run must exit 0 first.
TAG=$1; REGEX=${2:-"k_aggregate|k_csc_backward|k_umma_gemm"}
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/${TAG}_plain_full.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$REGEX" -s ${SKIP:-30} -c ${COUNT:-6} \
    -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu full rc=$?"
