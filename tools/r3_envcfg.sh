#!/bin/bash
# configs 4/5 per-round time under environment switches: tools/r3_envcfg.sh TAG CONFIG "ENV=.." ...
TAG=$1; C=$2; shift 2
i=0
for E in "" "$@"; do
  env $E timeout 900 python tools/bench_config4.py --config $C > gpurun_out/${TAG}_c${C}_$i.json 2>/dev/null
  echo "[$E] $(python -c "import json; d=json.load(open('gpurun_out/${TAG}_c${C}_$i.json')); print(round(d['ms_per_round'],2), {k:(round(x['ms_per_launch'],3), round(x['frac_hbm'],3)) for k,x in d['kernels'].items()}, {k:v for k,v in list(d['eager_breakdown_ms'].items())[:4]})")"
  i=$((i+1))
done > gpurun_out/${TAG}_envcfg.txt
