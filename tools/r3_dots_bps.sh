#!/bin/bash
for b in 4 3 2 1; do echo "bps=$b $(KG_DOTS_BPS=$b python tools/knockout.py 2>/dev/null | tail -1)"; done > gpurun_out/r3n_dots_bps.txt
