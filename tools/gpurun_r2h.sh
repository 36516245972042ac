#!/bin/bash
# segmented flat kNN: parity tests + plan statistics on a 10M-row config-5-like index
export BENCH_ALLOW_SHORT=1
timeout -s KILL 900 python -m pytest tests/test_gpu_segments.py -m gpu -q -x > gpurun_out/r2h_seg.log 2>&1; echo seg rc=$?
tail -25 gpurun_out/r2h_seg.log
TRIM_SEG_DEBUG=1 timeout 900 python bench.py --config c5 --n 10000000 --nq 2048 --steps 2 --warmup 1 --skip-cpu --no-group-check > gpurun_out/r2h_c5s.json 2> gpurun_out/r2h_c5s.log; echo c5s rc=$?
grep "trim seg" gpurun_out/r2h_c5s.log | head -5
python -c "
import json;d=json.loads(open('gpurun_out/r2h_c5s.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline']['list_skip_fraction'],d['e2e']['value'])"
