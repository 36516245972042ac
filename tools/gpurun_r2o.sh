#!/bin/bash
# multi-round segmented flat kNN: parity tests, config 5 and config 1
export BENCH_ALLOW_SHORT=1
timeout -s KILL 900 python -m pytest tests/test_gpu_segments.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3
TRIM_SEG_DEBUG=1 timeout 1500 python bench.py --config c5 --nq 2048 --steps 3 --warmup 1 --skip-cpu > gpurun_out/r2o_c5.json 2> gpurun_out/r2o_c5.log; echo c5 rc=$?
grep "trim seg" gpurun_out/r2o_c5.log | head -4
TRIM_SEG_DEBUG=1 timeout 600 python bench.py --config c1 --skip-cpu > gpurun_out/r2o_c1.json 2> gpurun_out/r2o_c1.log; echo c1 rc=$?
grep "trim seg" gpurun_out/r2o_c1.log | head -4
for f in c5 c1; do python -c "
import json;d=json.loads(open('gpurun_out/r2o_$f.json').read().strip().splitlines()[-1]);print('$f',d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline'].get('list_skip_fraction'),d['e2e']['value'])"; done
