#!/bin/bash
# GPU tests (optionally a -k filter), FB knock-out baseline + in-graph kernel
# times, configs 4/5 per-round times.
TAG=${1:-r3}
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider ${PYK:+-k "$PYK"} > gpurun_out/${TAG}_pytest.txt 2>&1; tail -3 gpurun_out/${TAG}_pytest.txt
python tools/knockout.py > gpurun_out/${TAG}_knock.txt 2>&1
python tools/graph_kernel_times.py > gpurun_out/${TAG}_gkt.txt 2>&1
if [ -z "$NO_CFG" ]; then
timeout 900 python tools/bench_config4.py --config 4 > gpurun_out/${TAG}_config4.json 2> gpurun_out/${TAG}_config4.err; echo c4 rc=$?
timeout 900 python tools/bench_config4.py --config 5 > gpurun_out/${TAG}_config5.json 2> gpurun_out/${TAG}_config5.err; echo c5 rc=$?
fi
