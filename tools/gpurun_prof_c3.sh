#!/bin/bash
# Full ncu capture of the flat range kernel on config 3 (one 1024-query launch).
export BENCH_ALLOW_SHORT=1
C3="python bench.py --config c3 --steps 1 --warmup 0 --skip-cpu --nq 1024 --n 2000000 --gamma 0.8"
timeout 600 $C3 > gpurun_out/plain_c3.json 2> gpurun_out/plain_c3.log && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trim_range_flat -s 1 -c 1 -o gpurun_out/prof_c3 -f $C3 > gpurun_out/ncu_c3.log 2>&1
echo ncu rc=$?
