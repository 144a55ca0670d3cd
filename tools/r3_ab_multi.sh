#!/bin/bash
# FB step and configs 4/5 for the in-tree build and variants: tools/r3_ab_multi.sh TAG V1 V2 ...
TAG=$1; shift
for V in main "$@"; do
  if [ "$V" = main ]; then L=; else L=paper_2201_02791_b200/lib/variants/$V.so; fi
  echo "$V $(KG_LIB=$L python tools/knockout.py 2>/dev/null | tail -1 | cut -c60-)"
  for C in 4 5; do KG_LIB=$L timeout 900 python tools/bench_config4.py --config $C > gpurun_out/${TAG}_${V}_config$C.json 2>/dev/null; done
done > gpurun_out/${TAG}_abm.txt
