#!/bin/bash
# last check of the shipped build (clean rebuild of HEAD): full GPU suite, smoke, default bench
export BENCH_ALLOW_SHORT=1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > gpurun_out/final_gpu.log 2>&1; echo gpu rc=$?
tail -2 gpurun_out/final_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/final_c2.json 2> gpurun_out/final_c2.log; echo c2 rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/final_c2.json').read().strip().splitlines()[-1]);print(d['value'],d.get('ms_per_step'),d['roofline']['frac'],d['e2e']['value'],d['cpu_baseline']['value'])"
