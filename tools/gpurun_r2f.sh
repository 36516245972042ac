#!/bin/bash
timeout -s KILL 1500 python -m pytest tests/test_gpu_reference_scale.py tests/test_gpu_shards.py -m gpu -q --durations=6 > gpurun_out/r2f_gpu.log 2>&1; echo gpu rc=$?
tail -12 gpurun_out/r2f_gpu.log
