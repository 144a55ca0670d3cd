#!/bin/bash
# Ad-hoc: run a list of pytest node ids with -s, output to gpurun_out/$TAG_quick.txt
TAG=$1; shift
timeout 1500 python -m pytest "$@" -m gpu -q -s -p no:cacheprovider > gpurun_out/${TAG}_quick.txt 2>&1; tail -5 gpurun_out/${TAG}_quick.txt
