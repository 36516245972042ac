#!/bin/bash
# segmented flat kNN: plan statistics vs the number of blocks (10M-row config-5-like index)
export BENCH_ALLOW_SHORT=1
for nb in 8192 16384; do
TRIM_FLAT_PARTITION_BLOCKS=$nb TRIM_SEG_DEBUG=1 timeout 900 python bench.py --config c5 --n 10000000 --nq 2048 --steps 2 --warmup 1 --skip-cpu --no-group-check > gpurun_out/r2i_c5s_$nb.json 2> gpurun_out/r2i_c5s_$nb.log; echo c5s $nb rc=$?
grep "trim seg" gpurun_out/r2i_c5s_$nb.log | head -3
python -c "
import json;d=json.loads(open('gpurun_out/r2i_c5s_$nb.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline']['list_skip_fraction'],d['e2e']['value'])"
done
timeout -s KILL 900 python -m pytest tests/test_gpu_segments.py tests/test_gpu_range.py -m gpu -q -x 2>&1 | tail -3
