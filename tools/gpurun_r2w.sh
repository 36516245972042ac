#!/bin/bash
# HARD flavour (StageNone) as its own launch: A/B on config 2, full GPU suite, bench lines
export BENCH_ALLOW_SHORT=1
timeout 1200 python tests/perf_libs.py --config c2 --libs new=paper_2508_17828_b200/libtrim_b200.so,nostage=paper_2508_17828_b200/libtrim_b200_nostage.so,nocut=paper_2508_17828_b200/libtrim_b200_nocut.so > gpurun_out/r2w_ab.txt 2> gpurun_out/r2w_ab.log; echo ab rc=$?
tail -5 gpurun_out/r2w_ab.txt
timeout -s KILL 1800 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/r2w_gpu.log 2>&1; echo gpu rc=$?
tail -3 gpurun_out/r2w_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2w_smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/r2w_c2.json 2> gpurun_out/r2w_c2.log; echo c2 rc=$?
timeout 600 python bench.py --config c4 --skip-cpu > gpurun_out/r2w_c4.json 2> gpurun_out/r2w_c4.log; echo c4 rc=$?
for f in c2 c4; do python -c "
import json;d=json.loads(open('gpurun_out/r2w_$f.json').read().strip().splitlines()[-1]);print('$f',d['value'],d.get('ms_per_step'),d.get('roofline',{}).get('frac'),d['e2e']['value'],d.get('sweep'))"; done
