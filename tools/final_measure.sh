#!/bin/bash
# Round-end measurement set (1 GPU): GPU tests, two bench runs, the ncu launch
# list of the bench command, the roofline kernel's traffic capture, configs 4/5
# and the eval breakdown. Outputs under gpurun_out/${TAG}_*.
TAG=${1:-final}
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.txt 2>&1; tail -2 gpurun_out/${TAG}_pytest.txt
for i in 1 2; do
  timeout 600 python bench.py > gpurun_out/${TAG}_bench_$i.json 2> gpurun_out/${TAG}_bench_$i.err; echo bench$i rc=$?
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; echo ref rc=$?
CMD="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo launches rc=$?
bash tools/ncu_traffic.sh
timeout 900 python tools/bench_config4.py --config 4 > gpurun_out/${TAG}_config4.json 2> gpurun_out/${TAG}_config4.err; echo c4 rc=$?
timeout 900 python tools/bench_config4.py --config 5 > gpurun_out/${TAG}_config5.json 2> gpurun_out/${TAG}_config5.err; echo c5 rc=$?
timeout 600 python tools/eval_bench.py > gpurun_out/${TAG}_eval.txt 2>&1; echo eval rc=$?
if [ -n "$REF_SUITE" ]; then bash tools/ref_suite.sh run gpurun_out/${TAG}_ref_suite.txt; tail -3 gpurun_out/${TAG}_ref_suite.txt; fi
