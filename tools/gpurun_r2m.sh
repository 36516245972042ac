#!/bin/bash
# entry-table segmented flat kNN: parity tests, config 5, config 1 with the layout forced
export BENCH_ALLOW_SHORT=1
timeout -s KILL 900 python -m pytest tests/test_gpu_segments.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3
TRIM_SEG_DEBUG=1 timeout 1500 python bench.py --config c5 --nq 2048 --steps 3 --warmup 1 --skip-cpu > gpurun_out/r2m_c5.json 2> gpurun_out/r2m_c5.log; echo c5 rc=$?
grep "trim seg" gpurun_out/r2m_c5.log | head -2
TRIM_FLAT_PARTITION_MIN_ROWS=50000 TRIM_SEG_N0=8192 TRIM_SEG_DEBUG=1 timeout 600 python bench.py --config c1 --skip-cpu > gpurun_out/r2m_c1_seg.json 2> gpurun_out/r2m_c1_seg.log; echo c1seg rc=$?
grep "trim seg" gpurun_out/r2m_c1_seg.log | head -2
for f in c5 c1_seg; do python -c "
import json;d=json.loads(open('gpurun_out/r2m_$f.json').read().strip().splitlines()[-1]);print('$f',d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline'].get('list_skip_fraction'),d['e2e']['value'])"; done
