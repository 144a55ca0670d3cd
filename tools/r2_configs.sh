#!/bin/bash
# Config-parity GPU tests with their measured figures (JSON lines, -s).
TAG=${1:-r2}
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_dropin.py -m gpu -q -s -p no:cacheprovider \
  > gpurun_out/${TAG}_configs.txt 2>&1; tail -5 gpurun_out/${TAG}_configs.txt
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --deselect tests/test_gpu_configs.py \
  > gpurun_out/${TAG}_pytest.txt 2>&1; tail -3 gpurun_out/${TAG}_pytest.txt
(cd baseline/_ref/ref_tests && KGDIST_REF_CLI=$PWD/../ref_cli.py PYTHONPATH=../../../tools/kgdist_alias:../../.. \
  timeout 600 python ../../../tools/ref_c09_check.py > ../../../gpurun_out/${TAG}_c09.txt 2>&1); tail -2 gpurun_out/${TAG}_c09.txt
