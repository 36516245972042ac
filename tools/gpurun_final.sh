#!/bin/bash
# last check of the shipped build
export BENCH_ALLOW_SHORT=1
timeout -s KILL 900 python -m pytest tests/test_gpu_segments.py tests/test_gpu_parity.py tests/test_gpu_range.py tests/test_gpu_graph.py tests/test_capi.py -m gpu -q -x 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/final_c2.json 2> gpurun_out/final_c2.log; echo c2 rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/final_c2.json').read().strip().splitlines()[-1]);print(d['value'],d.get('ms_per_step'),d['roofline']['frac'],d['e2e']['value'])"
