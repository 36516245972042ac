#!/bin/bash
# final verification of the build: full GPU suite, smoke, the default bench line, the reference arm, c5 / c1 / c3 / c4 lines
export BENCH_ALLOW_SHORT=1
timeout -s KILL 1800 python -m pytest tests -m gpu -q -x --durations=6 > gpurun_out/r2s_gpu.log 2>&1; echo gpu rc=$?
tail -4 gpurun_out/r2s_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s_smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/r2s_c2.json 2> gpurun_out/r2s_c2.log; echo c2 rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2s_ref.json 2> gpurun_out/r2s_ref.log; echo ref rc=$?
timeout 1500 python bench.py --config c5 --steps 2 --warmup 1 > gpurun_out/r2s_c5.json 2> gpurun_out/r2s_c5.log; echo c5 rc=$?
timeout 600 python bench.py --config c1 > gpurun_out/r2s_c1.json 2> gpurun_out/r2s_c1.log; echo c1 rc=$?
timeout 900 python bench.py --config c4 > gpurun_out/r2s_c4.json 2> gpurun_out/r2s_c4.log; echo c4 rc=$?
for f in c2 ref c5 c1 c4; do python -c "
import json;d=json.loads(open('gpurun_out/r2s_$f.json').read().strip().splitlines()[-1]);print('$f',d['value'],d.get('ms_per_step'),d.get('roofline',{}).get('frac'),d['e2e']['value'])"; done
TAG=r02c
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:trim_knn_kernel|trim_knn_seg_plan' -s 0 -c 10 -o /tmp/${TAG}_c5 -f python bench.py --config c5 --nq 1024 --steps 1 --warmup 0 --skip-cpu --recall-q 0 --no-group-check --streams 1 > gpurun_out/${TAG}_c5_ncu.log 2>&1; echo "c5 ncu rc=$?"
ncu -i /tmp/${TAG}_c5.ncu-rep --page raw --csv > gpurun_out/${TAG}_c5_raw.csv 2>/dev/null; rm -f /tmp/${TAG}_c5.ncu-rep
