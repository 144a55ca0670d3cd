#!/bin/bash
# Static SASS evidence of the tcgen05 / bulk-copy kernels (no GPU needed).
cuobjdump -sass paper_2201_02791_b200/lib/libkgdist_b200.so > /tmp/kg_sass.txt && \
  grep -c UTCHMMA /tmp/kg_sass.txt
