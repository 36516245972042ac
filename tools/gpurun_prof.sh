#!/bin/bash
# Launch list + one full capture of the filter and the probe-select kernels (c2).
export BENCH_ALLOW_SHORT=1
C2="python bench.py --steps 1 --warmup 0 --skip-cpu --nq 4096 --recall-q 0 --gamma 0.8"
K='regex:trim_(knn|probe|range|bl|merge|lut)'
timeout 600 $C2 > gpurun_out/plain_c2.json 2> gpurun_out/plain_c2.log && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 80 --csv --log-file gpurun_out/launches_c2.csv $C2 > gpurun_out/ncu_launch.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:trim_(knn_kernel|probe_select|probe_mma)' -s 3 -c 3 -o gpurun_out/prof_c2 -f $C2 > gpurun_out/ncu_c2.log 2>&1
echo ncu rc=$?
