#!/bin/bash
TAG=${1:-r2x}
O=gpurun_out
KG_EAGER_WARMUP=0 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "graph or train or eager or fused or record" > $O/${TAG}_w0_pytest.txt 2>&1; tail -2 $O/${TAG}_w0_pytest.txt
KG_EAGER_WARMUP=0 timeout 600 python bench.py > $O/${TAG}_w0_bench.json 2> $O/${TAG}_w0_bench.err; echo w0 rc=$?
KG_EAGER_WARMUP=1 timeout 600 python bench.py > $O/${TAG}_w1_bench.json 2> $O/${TAG}_w1_bench.err; echo w1 rc=$?
