#!/bin/bash
# full GPU suite with the 64k-row partition threshold, then the flat configs' bench lines
export BENCH_ALLOW_SHORT=1
timeout -s KILL 1800 python -m pytest tests -m gpu -q -x --durations=6 > gpurun_out/r2n_gpu.log 2>&1; echo gpu rc=$?
tail -4 gpurun_out/r2n_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2n_smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py --config c1 > gpurun_out/r2n_c1.json 2> gpurun_out/r2n_c1.log; echo c1 rc=$?
timeout 1500 python bench.py --config c5 --steps 2 --warmup 1 > gpurun_out/r2n_c5.json 2> gpurun_out/r2n_c5.log; echo c5 rc=$?
timeout 900 python bench.py --config c3 --skip-cpu > gpurun_out/r2n_c3.json 2> gpurun_out/r2n_c3.log; echo c3 rc=$?
for f in c1 c5 c3; do python -c "
import json;d=json.loads(open('gpurun_out/r2n_$f.json').read().strip().splitlines()[-1]);print('$f',d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline'].get('list_skip_fraction'),d['e2e']['value'],d.get('sweep'))"; done
