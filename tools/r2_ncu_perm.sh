#!/bin/bash
TAG=${1:-r2q}
O=gpurun_out
timeout 600 ncu --set full --import-source on -k regex:"k_perm_draws" -c 1 -o $O/${TAG}_perm python tools/epoch_graph_times.py 1 > $O/${TAG}_perm_ncu.log 2>&1
ncu -i $O/${TAG}_perm.ncu-rep --page raw --csv > $O/${TAG}_perm_raw.csv 2>/dev/null
ncu -i $O/${TAG}_perm.ncu-rep --page source --csv --print-source sass > $O/${TAG}_perm_source.csv 2>/dev/null
rm -f $O/${TAG}_perm.ncu-rep
