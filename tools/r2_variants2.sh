#!/bin/bash
TAG=${1:-r2z}
O=gpurun_out
for V in default bps4 bps5 default bps4 bps5; do
  L=""; [ "$V" != default ] && L=paper_2201_02791_b200/lib/variants/$V.so
  KG_LIB=$L timeout 600 python bench.py --no-e2e --no-cpu-baseline > $O/${TAG}_${V}_bench.json 2>&1; echo $V rc=$? $(python -c "import json;d=json.load(open('$O/${TAG}_${V}_bench.json'));print(round(d['ms_per_step'],4))")
done
for C in 4 5; do
  KG_LIB=paper_2201_02791_b200/lib/variants/bps5.so timeout 900 python tools/bench_config4.py --config $C > $O/${TAG}_bps5_config$C.json 2>&1; echo bps5 c$C rc=$?
done
