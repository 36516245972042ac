#!/bin/bash
# c2 bench line of the current tree, then one full ncu capture (with source) of trim_knn_kernel.
export BENCH_ALLOW_SHORT=1
TAG=${1:-r2d}
timeout 900 python bench.py --skip-cpu --no-group-check > gpurun_out/${TAG}_c2.json 2> gpurun_out/${TAG}_c2.log; echo c2 rc=$?
C2="python bench.py --steps 1 --warmup 0 --skip-cpu --nq 2048 --recall-q 0 --no-group-check --gamma 0.8 --streams 1"
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:trim_knn_kernel' -s 1 -c 1 -o gpurun_out/${TAG}_knn -f $C2 > gpurun_out/${TAG}_ncu.log 2>&1; echo ncu rc=$?
