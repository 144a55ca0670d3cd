#!/bin/bash
# Build an A/B variant of the kernel library with extra nvcc defines:
#   tools/build_variant.sh NAME "-DKG_GATHER_BPS=4"   -> paper_2201_02791_b200/lib/variants/NAME.so
# then run with KG_LIB=paper_2201_02791_b200/lib/variants/NAME.so (diagnostics only).
set -e
NAME=$1; DEFS=$2
OUT=build/variants/$NAME; mkdir -p $OUT paper_2201_02791_b200/lib/variants
for f in paper_2201_02791_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=default \
       --expt-relaxed-constexpr $DEFS -c $f -o $OUT/$b.o &
done
g++ -O2 -std=c++17 -fPIC -ffp-contract=off -I/usr/local/cuda/include -c paper_2201_02791_b200/csrc/kg_host.cpp -o $OUT/kg_host.host.o &
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2201_02791_b200/lib/variants/$NAME.so $OUT/*.o -Xcompiler -fPIC -cudart static
echo built paper_2201_02791_b200/lib/variants/$NAME.so
