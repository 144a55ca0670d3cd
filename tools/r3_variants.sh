#!/bin/bash
# A/B library variants on one config: tools/r3_variants.sh TAG CONFIG V1 V2 ... ("main" = the in-tree build)
TAG=$1; C=$2; shift 2
for V in "$@"; do
  if [ "$V" = main ]; then L=; else L=paper_2201_02791_b200/lib/variants/$V.so; fi
  KG_LIB=$L timeout 900 python tools/bench_config4.py --config $C > gpurun_out/${TAG}_${V}_config$C.json 2>&1; echo $V c$C rc=$?
done
