#!/bin/bash
for st in 8 4 3 2; do echo "stages=$st $(KG_GEMM_STAGES=$st python tools/knockout.py 2>/dev/null | tail -1)"; done > gpurun_out/r3t_stages.txt
