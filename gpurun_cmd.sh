#!/bin/bash
export BENCH_ALLOW_SHORT=1
timeout 2400 python bench.py --config c5 --nq 2048 --steps 1 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.log; echo c5 rc=$?
tail -3 gpurun_out/bench_c5.log
