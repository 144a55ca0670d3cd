#!/bin/bash
# ncu launch durations of the NN GEMM at FB layer shapes with parts of the kernel dropped (KG_GEMM_EXP)
for e in 0 1 2 3; do
  KG_GEMM_EXP=$e timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_umma_packed --csv python tools/gemm_probe.py 2>/dev/null | grep k_umma_packed | awk -F'","' -v e=$e '{print "exp=" e, $NF}'
done > gpurun_out/${1:-r3o}_gemm_probe.txt
