#!/bin/bash
# ncu --set full of the fused CSC pass and the aggregate at configs 4 and 5
# (first eager launches of tools/bench_config4.py), reduced to CSV on the box.
TAG=${1:-r2c}
O=gpurun_out
for C in 4 5; do
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${REGEX:-k_csc_backward}" -c ${COUNT:-1} \
    -o $O/${TAG}_c${C} python tools/bench_config4.py --config $C --rounds 1 > $O/${TAG}_c${C}_ncu.log 2>&1
  echo "ncu c$C rc=$?"
  ncu -i $O/${TAG}_c${C}.ncu-rep --page raw --csv > $O/${TAG}_c${C}_raw.csv 2>/dev/null
  ncu -i $O/${TAG}_c${C}.ncu-rep --page source --csv --print-source sass > $O/${TAG}_c${C}_source.csv 2>/dev/null
  ls -la $O/${TAG}_c${C}*
  rm -f $O/${TAG}_c${C}.ncu-rep
done
