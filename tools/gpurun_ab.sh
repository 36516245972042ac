#!/bin/bash
# Same-process A/B of library variants (tests/perf_libs.py); args: config libs...
export BENCH_ALLOW_SHORT=1
TAG=$1; CFG=$2; LIBS=$3; shift 3
timeout 1200 python tests/perf_libs.py --config $CFG --libs $LIBS "$@" > gpurun_out/${TAG}.txt 2> gpurun_out/${TAG}.log; echo ab rc=$?
tail -8 gpurun_out/${TAG}.txt
