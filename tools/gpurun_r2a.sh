#!/bin/bash
# Round-2 check of the restored tree: the multi-device ABI tests first, then the whole GPU suite, smoke and the default bench.
export BENCH_ALLOW_SHORT=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
lscpu > gpurun_out/r2a_lscpu.txt; nproc >> gpurun_out/r2a_lscpu.txt
timeout -s KILL 600 python -m pytest tests/test_gpu_multi.py tests/test_gpu_shards.py -q -x > gpurun_out/r2a_multi.log 2>&1; echo multi rc=$?
timeout -s KILL 1800 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r2a_gpu.log 2>&1; echo gpu rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.log; echo bench rc=$?
