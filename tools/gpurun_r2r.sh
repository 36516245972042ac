#!/bin/bash
export BENCH_ALLOW_SHORT=1
timeout 1500 python bench.py --config c5 --steps 2 --warmup 1 > gpurun_out/r2r_c5.json 2> gpurun_out/r2r_c5.log; echo c5 rc=$?
timeout 600 python bench.py --config c1 > gpurun_out/r2r_c1.json 2> gpurun_out/r2r_c1.log; echo c1 rc=$?
for f in c5 c1; do python -c "
import json;d=json.loads(open('gpurun_out/r2r_$f.json').read().strip().splitlines()[-1]);print('$f',d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline'].get('list_skip_fraction'),d['e2e']['value'],d['clocks'])"; done
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
