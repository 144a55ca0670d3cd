#!/bin/bash
# ncu --set full of the FB-shape (config 1) round's kernels (first launches,
# eager warm-up rounds of tools/knockout.py), reduced to CSV on the box.
TAG=${1:-r3g}
O=gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${REGEX:-k_umma_gemm|k_csc|k_aggregate}" -c ${COUNT:-12} \
  -o $O/${TAG}_fb python tools/knockout.py > $O/${TAG}_fb_ncu.log 2>&1
echo "ncu rc=$?"
ncu -i $O/${TAG}_fb.ncu-rep --page raw --csv > $O/${TAG}_fb_raw.csv 2>/dev/null
ncu -i $O/${TAG}_fb.ncu-rep --page source --csv --print-source sass > $O/${TAG}_fb_source.csv 2>/dev/null
ls -la $O/${TAG}_fb*
rm -f $O/${TAG}_fb.ncu-rep
