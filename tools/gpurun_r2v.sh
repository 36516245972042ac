#!/bin/bash
# StageCut + StageNone (record-selected): A/B on config 2, parity suites, flat configs
export BENCH_ALLOW_SHORT=1
timeout 1200 python tests/perf_libs.py --config c2 --libs new=paper_2508_17828_b200/libtrim_b200.so,nostage=paper_2508_17828_b200/libtrim_b200_nostage.so,nocut=paper_2508_17828_b200/libtrim_b200_nocut.so > gpurun_out/r2v_ab.txt 2> gpurun_out/r2v_ab.log; echo ab rc=$?
tail -5 gpurun_out/r2v_ab.txt
timeout -s KILL 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_segments.py tests/test_gpu_probe.py tests/test_gpu_shards.py tests/test_gpu_multi.py -m gpu -q -x 2>&1 | tail -3
timeout 1500 python bench.py --config c5 --steps 2 --warmup 1 --skip-cpu > gpurun_out/r2v_c5.json 2> gpurun_out/r2v_c5.log; echo c5 rc=$?
timeout 600 python bench.py --config c1 --skip-cpu > gpurun_out/r2v_c1.json 2> gpurun_out/r2v_c1.log; echo c1 rc=$?
for f in c5 c1; do python -c "
import json;d=json.loads(open('gpurun_out/r2v_$f.json').read().strip().splitlines()[-1]);print('$f',d['value'],d.get('ms_per_step'),d.get('roofline',{}).get('frac'),d['e2e']['value'])"; done
