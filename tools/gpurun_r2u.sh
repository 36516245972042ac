#!/bin/bash
export BENCH_ALLOW_SHORT=1
timeout 1200 python tests/perf_libs.py --config c2 --libs coarse=paper_2508_17828_b200/libtrim_b200.so,only32=paper_2508_17828_b200/libtrim_b200_only32.so,nostage=paper_2508_17828_b200/libtrim_b200_nostage.so > gpurun_out/r2u_ab3.txt 2> gpurun_out/r2u_ab3.log; echo ab rc=$?
tail -6 gpurun_out/r2u_ab3.txt
