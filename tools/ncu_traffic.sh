#!/bin/bash
# DRAM traffic per launch of the bench's roofline kernel (k_aggregate) from one
# ncu --set full capture (warm L2: --cache-control none, as in the timed
# steps), summarised into profiles/r1_roofline_traffic.json for bench.py.
# The plain command must exit 0 first.
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/traffic_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --cache-control none -k regex:"k_aggregate" -s 2 -c 4 \
    -o gpurun_out/traffic_full $CMD > gpurun_out/traffic_ncu.log 2>&1
echo "ncu rc=$?"
