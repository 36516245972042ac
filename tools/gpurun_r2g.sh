#!/bin/bash
# segmented flat kNN: parity tests, the flat reference-scale case, config-5 bench
export BENCH_ALLOW_SHORT=1
timeout -s KILL 900 python -m pytest tests/test_gpu_segments.py -m gpu -q -x > gpurun_out/r2g_seg.log 2>&1; echo seg rc=$?
tail -15 gpurun_out/r2g_seg.log
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_range.py -m gpu -q -x > gpurun_out/r2g_par.log 2>&1; echo parity rc=$?
tail -3 gpurun_out/r2g_par.log
timeout -s KILL 900 python -m pytest tests/test_gpu_reference_scale.py -m gpu -q -x -k config5 > gpurun_out/r2g_c5ref.log 2>&1; echo c5ref rc=$?
tail -3 gpurun_out/r2g_c5ref.log
timeout 1200 python bench.py --config c5 --nq 2048 --steps 2 --warmup 1 > gpurun_out/r2g_c5.json 2> gpurun_out/r2g_c5.log; echo c5 rc=$?
tail -c 1500 gpurun_out/r2g_c5.json
