#!/bin/bash
# One GPU check cycle: GPU tests, the reference suite against the package, one bench line.
TAG=${1:-r2}
nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader
python -c "import numpy; print('numpy', numpy.__version__)"
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.txt 2>&1; tail -3 gpurun_out/${TAG}_pytest.txt
bash tools/ref_suite.sh run gpurun_out/${TAG}_ref_suite.txt; tail -3 gpurun_out/${TAG}_ref_suite.txt
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?; cat gpurun_out/${TAG}_bench.json
