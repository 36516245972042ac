#!/bin/bash
export BENCH_ALLOW_SHORT=1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3 > gpurun_out/pytest.log
timeout 900 python tests/perf_modes.py --variants "TRIM_RING_SLEEP_NS=0|TRIM_RING_SLEEP_NS=32|TRIM_RING_SLEEP_NS=128|TRIM_RING_SLEEP_NS=512" --gammas 0.8,0.6 > gpurun_out/modes.log 2>&1
cat gpurun_out/pytest.log gpurun_out/modes.log
