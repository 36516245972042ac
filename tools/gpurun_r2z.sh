#!/bin/bash
# plan kernel (atomic compaction, slice merge): parity, config 5 / config 1
export BENCH_ALLOW_SHORT=1
timeout -s KILL 900 python -m pytest tests/test_gpu_segments.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
timeout -s KILL 900 python -m pytest tests/test_gpu_reference_scale.py -m gpu -q -x -k config5 2>&1 | tail -2
timeout 1500 python bench.py --config c5 --steps 2 --warmup 1 --skip-cpu > gpurun_out/r2z_c5.json 2> gpurun_out/r2z_c5.log; echo c5 rc=$?
timeout 600 python bench.py --config c1 --skip-cpu > gpurun_out/r2z_c1.json 2> gpurun_out/r2z_c1.log; echo c1 rc=$?
for f in c5 c1; do python -c "
import json;d=json.loads(open('gpurun_out/r2z_$f.json').read().strip().splitlines()[-1]);print('$f',d['value'],d.get('ms_per_step'),d.get('roofline',{}).get('frac'),d['e2e']['value'])"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:trim_knn' -c 12 --csv --log-file gpurun_out/r2z_c5_launches.csv python bench.py --config c5 --nq 1024 --steps 1 --warmup 0 --skip-cpu --recall-q 0 --no-group-check --streams 1 > gpurun_out/r2z_launch.log 2>&1; echo launches rc=$?
grep -E "trim_knn" gpurun_out/r2z_c5_launches.csv | awk -F'","' '{print $5, $NF}' | head -12
