#!/bin/bash
# final sanity of HEAD: default bench, reference arm, flat configs, segment + parity suites
export BENCH_ALLOW_SHORT=1
timeout 900 python bench.py > gpurun_out/r2y_c2.json 2> gpurun_out/r2y_c2.log; echo c2 rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2y_ref.json 2> gpurun_out/r2y_ref.log; echo ref rc=$?
timeout 600 python bench.py --config c1 --skip-cpu > gpurun_out/r2y_c1.json 2> gpurun_out/r2y_c1.log; echo c1 rc=$?
timeout 1500 python bench.py --config c5 --steps 2 --warmup 1 --skip-cpu > gpurun_out/r2y_c5.json 2> gpurun_out/r2y_c5.log; echo c5 rc=$?
timeout 900 python bench.py --config g1 --skip-cpu > gpurun_out/r2y_g1.json 2> gpurun_out/r2y_g1.log; echo g1 rc=$?
for f in c2 ref c1 c5 g1; do python -c "
import json;d=json.loads(open('gpurun_out/r2y_$f.json').read().strip().splitlines()[-1]);print('$f',d['value'],d.get('ms_per_step'),d.get('roofline',{}).get('frac'),d['e2e']['value'],d.get('gpu_launches'))"; done
timeout -s KILL 900 python -m pytest tests/test_gpu_segments.py tests/test_gpu_parity.py tests/test_capi.py -m gpu -q -x 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
