#!/bin/bash
# StageCut (one-compare stage tests every 8 lookups) vs StageCheck: same-process A/B on config 2, then parity suites
export BENCH_ALLOW_SHORT=1
timeout 1200 python tests/perf_libs.py --config c2 --libs cut=paper_2508_17828_b200/libtrim_b200.so,nocut=paper_2508_17828_b200/libtrim_b200_nocut.so > gpurun_out/r2t_ab.txt 2> gpurun_out/r2t_ab.log; echo ab rc=$?
tail -12 gpurun_out/r2t_ab.txt
timeout -s KILL 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_segments.py tests/test_gpu_probe.py tests/test_gpu_shards.py -m gpu -q -x 2>&1 | tail -3
