#!/bin/bash
# FB-shape step A/B between the in-tree build and a variant (tools/knockout.py), alternating
TAG=$1; V=$2
for i in 1 2 3; do
  echo "main $(python tools/knockout.py 2>/dev/null | tail -1 | cut -c60-)"
  echo "$V $(KG_LIB=paper_2201_02791_b200/lib/variants/$V.so python tools/knockout.py 2>/dev/null | tail -1 | cut -c60-)"
done > gpurun_out/${TAG}_abfb.txt
