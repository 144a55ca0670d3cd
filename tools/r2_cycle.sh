#!/bin/bash
# One GPU check cycle: GPU tests, FB bench, configs 4/5 (and optionally the reference suite).
TAG=${1:-r2}
nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.txt 2>&1; tail -3 gpurun_out/${TAG}_pytest.txt
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?
timeout 900 python tools/bench_config4.py --config 4 > gpurun_out/${TAG}_config4.json 2> gpurun_out/${TAG}_config4.err; echo c4 rc=$?
timeout 900 python tools/bench_config4.py --config 5 > gpurun_out/${TAG}_config5.json 2> gpurun_out/${TAG}_config5.err; echo c5 rc=$?
if [ -n "$REF_SUITE" ]; then bash tools/ref_suite.sh run gpurun_out/${TAG}_ref_suite.txt; tail -3 gpurun_out/${TAG}_ref_suite.txt; fi
