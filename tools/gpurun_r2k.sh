#!/bin/bash
export BENCH_ALLOW_SHORT=1
timeout -s KILL 900 python -m pytest tests/test_gpu_segments.py -m gpu -q -x 2>&1 | tail -3
TRIM_SEG_DEBUG=1 timeout 1500 python bench.py --config c5 --nq 2048 --steps 3 --warmup 1 > gpurun_out/r2k_c5.json 2> gpurun_out/r2k_c5.log; echo c5 rc=$?
grep "trim seg" gpurun_out/r2k_c5.log | head -2
python -c "
import json;d=json.loads(open('gpurun_out/r2k_c5.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline'],d['e2e']['value'], d['cpu_baseline']['value'])"
