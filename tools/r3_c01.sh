#!/bin/bash
# the reference's gradient check (criterion 01), repeated in fresh processes
ROOT=$(pwd)
cd baseline/_ref/ref_tests
for i in 1 2 3 4 5 6; do
  KGDIST_REF_CLI="$ROOT/baseline/_ref/ref_cli.py" PYTHONPATH="$ROOT/tools/kgdist_alias:$ROOT" \
    timeout 300 python -m pytest -q -p no:cacheprovider test_acceptance.py -k "criterion_01" -s 2>&1 | grep "criterion 01"
done > $ROOT/gpurun_out/r3zu_c01.txt
