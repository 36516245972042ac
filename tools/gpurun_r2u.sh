#!/bin/bash
export BENCH_ALLOW_SHORT=1
timeout 1200 python tests/perf_libs.py --config c2 --libs head=paper_2508_17828_b200/libtrim_b200.so,w9=paper_2508_17828_b200/libtrim_b200_w9.so,w10=paper_2508_17828_b200/libtrim_b200_w10.so > gpurun_out/r2u_ab4.txt 2> gpurun_out/r2u_ab4.log; echo ab rc=$?
tail -6 gpurun_out/r2u_ab4.txt
