#!/bin/bash
# config 5 (one 100M-row shard) through the segmented block stream; parity at that scale
export BENCH_ALLOW_SHORT=1
TRIM_SEG_DEBUG=1 timeout 1500 python bench.py --config c5 --nq 2048 --steps 3 --warmup 1 > gpurun_out/r2j_c5.json 2> gpurun_out/r2j_c5.log; echo c5 rc=$?
grep "trim seg" gpurun_out/r2j_c5.log | head -3
python -c "
import json;d=json.loads(open('gpurun_out/r2j_c5.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline'],d['e2e']['value'], d['cpu_baseline']['value'])"
true
tail -3 gpurun_out/r2j_c5ref.log
