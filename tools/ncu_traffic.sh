#!/bin/bash
# DRAM traffic per launch of the bench's roofline kernel (k_csc_backward, the
# fused CSC pass) from one ncu --set full capture (warm L2: --cache-control
# none, as in the timed steps), summarised into profiles/r3_roofline_traffic.json
# for bench.py (tools/traffic_json.py runs on the box; the report is deleted).
# The plain command must exit 0 first.
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/traffic_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --cache-control none -k regex:"k_csc_backward" -s 2 -c 4 \
    -o gpurun_out/traffic_full $CMD > gpurun_out/traffic_ncu.log 2>&1
echo "ncu rc=$?"
python tools/traffic_json.py gpurun_out/traffic_full.ncu-rep > gpurun_out/traffic_json.log 2>&1   # copy the printed JSON to profiles/r3_roofline_traffic.json
rm -f gpurun_out/traffic_full.ncu-rep
