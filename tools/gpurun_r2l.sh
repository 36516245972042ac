#!/bin/bash
# full GPU suite after the segmented flat kNN change, then the flat configs' bench lines
export BENCH_ALLOW_SHORT=1
timeout -s KILL 1800 python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/r2l_gpu.log 2>&1; echo gpu rc=$?
tail -4 gpurun_out/r2l_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2l_smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py --config c1 > gpurun_out/r2l_c1.json 2> gpurun_out/r2l_c1.log; echo c1 rc=$?
TRIM_FLAT_PARTITION_MIN_ROWS=50000 TRIM_SEG_N0=8192 TRIM_SEG_DEBUG=1 timeout 600 python bench.py --config c1 --skip-cpu > gpurun_out/r2l_c1_seg.json 2> gpurun_out/r2l_c1_seg.log; echo c1seg rc=$?
grep "trim seg" gpurun_out/r2l_c1_seg.log | head -2
timeout 1500 python bench.py --config c5 --steps 2 --warmup 1 > gpurun_out/r2l_c5.json 2> gpurun_out/r2l_c5.log; echo c5 rc=$?
timeout 900 python bench.py --config c3 --skip-cpu > gpurun_out/r2l_c3.json 2> gpurun_out/r2l_c3.log; echo c3 rc=$?
for f in c1 c1_seg c5 c3; do python -c "
import json;d=json.loads(open('gpurun_out/r2l_$f.json').read().strip().splitlines()[-1]);print('$f',d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline'].get('list_skip_fraction'),d['e2e']['value'])"; done
