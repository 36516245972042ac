#!/bin/bash
# SEG without stages: A/B on config 1 (m = 16) and a 10M-row config-5-like index (m = 48); c2 ncu of the final kernel
export BENCH_ALLOW_SHORT=1
timeout 900 python tests/perf_libs.py --config c1 --libs base=paper_2508_17828_b200/libtrim_b200.so,segns=paper_2508_17828_b200/libtrim_b200_segns.so > gpurun_out/r2x_ab_c1.txt 2> gpurun_out/r2x_ab_c1.log; echo ab c1 rc=$?
tail -4 gpurun_out/r2x_ab_c1.txt
timeout 1200 python tests/perf_libs.py --config c5 --nq 4096 --libs base=paper_2508_17828_b200/libtrim_b200.so,segns=paper_2508_17828_b200/libtrim_b200_segns.so > gpurun_out/r2x_ab_c5.txt 2> gpurun_out/r2x_ab_c5.log; echo ab c5 rc=$?
tail -4 gpurun_out/r2x_ab_c5.txt
TAG=r02d
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:trim_knn_kernel' -s 2 -c 2 -o /tmp/${TAG}_c2 -f python bench.py --config c2 --nq 2048 --gamma 0.8 --steps 1 --warmup 0 --skip-cpu --recall-q 0 --no-group-check --streams 1 > gpurun_out/${TAG}_c2_ncu.log 2>&1; echo "c2 ncu rc=$?"
ncu -i /tmp/${TAG}_c2.ncu-rep --page raw --csv > gpurun_out/${TAG}_c2_raw.csv 2>/dev/null; rm -f /tmp/${TAG}_c2.ncu-rep
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:trim_probe|trim_knn' -c 60 --csv --log-file gpurun_out/${TAG}_c2_launches.csv python bench.py --steps 1 --warmup 0 --skip-cpu --nq 4096 --recall-q 0 --no-group-check --gamma 0.8 > gpurun_out/${TAG}_launch.log 2>&1; echo launches rc=$?
