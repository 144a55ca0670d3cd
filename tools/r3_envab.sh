#!/bin/bash
# A/B of environment switches on the FB-shape step (tools/knockout.py, no knock-out): tools/r3_envab.sh TAG "ENV=1" "ENV2=0" ...
TAG=$1; shift
for E in "" "$@"; do
  echo "[$E] $(env $E python tools/knockout.py 2>/dev/null | tail -1)"
done > gpurun_out/${TAG}_envab.txt
