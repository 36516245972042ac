#!/bin/bash
# merge-based plan kernel: parity tests; config-5 e2e with and without continue rounds
export BENCH_ALLOW_SHORT=1
timeout -s KILL 900 python -m pytest tests/test_gpu_segments.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3
timeout 1500 python bench.py --config c5 --nq 4096 --steps 3 --warmup 1 --skip-cpu > gpurun_out/r2q_c5.json 2> gpurun_out/r2q_c5.log; echo c5 rc=$?
TRIM_SEG_ROUNDS=0 timeout 1500 python bench.py --config c5 --nq 4096 --steps 3 --warmup 1 --skip-cpu > gpurun_out/r2q_c5_r0.json 2> gpurun_out/r2q_c5_r0.log; echo c5r0 rc=$?
for f in c5 c5_r0; do python -c "
import json;d=json.loads(open('gpurun_out/r2q_$f.json').read().strip().splitlines()[-1]);print('$f',d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline'].get('list_skip_fraction'),d['e2e'])"; done
