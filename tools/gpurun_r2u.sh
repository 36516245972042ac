#!/bin/bash
export BENCH_ALLOW_SHORT=1
timeout 1500 python tests/perf_libs.py --config c4 --libs head=paper_2508_17828_b200/libtrim_b200.so,nostage=paper_2508_17828_b200/libtrim_b200_ns120.so --steps 2 --reps 2 > gpurun_out/r2u_ab5.txt 2> gpurun_out/r2u_ab5.log; echo ab rc=$?
tail -5 gpurun_out/r2u_ab5.txt
timeout 1500 python tests/perf_libs.py --config c4 --gamma 0.5 --libs head=paper_2508_17828_b200/libtrim_b200.so,nostage=paper_2508_17828_b200/libtrim_b200_ns120.so --steps 2 --reps 2 > gpurun_out/r2u_ab6.txt 2> gpurun_out/r2u_ab6.log; echo ab rc=$?
tail -5 gpurun_out/r2u_ab6.txt
