#!/bin/bash
TAG=${1:-r2y}
O=gpurun_out
for V in bps4 bps2; do
  for C in 4 5; do
    KG_LIB=paper_2201_02791_b200/lib/variants/$V.so timeout 900 python tools/bench_config4.py --config $C > $O/${TAG}_${V}_config$C.json 2>&1; echo $V c$C rc=$?
  done
done
