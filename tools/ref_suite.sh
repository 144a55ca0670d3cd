#!/bin/bash
# Run the reference's own test suite against the drop-in package on a GPU box.
#   prepare (here, with /root/reference present):  tools/ref_suite.sh prepare
#   run (GPU box):                                 tools/ref_suite.sh run OUT.txt
# The copy lives in baseline/_ref/ (git-ignored, travels with gpurun).
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
case "${1:-run}" in
  prepare)
    rm -rf "$ROOT/baseline/_ref/ref_tests"
    mkdir -p "$ROOT/baseline/_ref/ref_tests"
    cp /root/reference/pkg/tests/*.py "$ROOT/baseline/_ref/ref_tests/"
    cp /root/reference/pkg/src/kgdist/cli.py "$ROOT/baseline/_ref/ref_cli.py"
    ;;
  run)
    OUT=${2:-gpurun_out/ref_suite.txt}
    cd "$ROOT/baseline/_ref/ref_tests"
    KGDIST_REF_CLI="$ROOT/baseline/_ref/ref_cli.py" PYTHONPATH="$ROOT/tools/kgdist_alias:$ROOT" \
      timeout 1800 python -m pytest -q -rA -p no:cacheprovider . > "$ROOT/$OUT" 2>&1
    echo "ref suite exit $?" >> "$ROOT/$OUT"
    ;;
esac
