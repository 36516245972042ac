#!/bin/bash
# full GPU suite + smoke + default bench (QPS headline) + reference arm
export BENCH_ALLOW_SHORT=1
timeout -s KILL 1800 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/r2e_gpu.log 2>&1; echo gpu rc=$?
tail -3 gpurun_out/r2e_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e_smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/r2e_c2.json 2> gpurun_out/r2e_c2.log; echo c2 rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2e_ref.json 2> gpurun_out/r2e_ref.log; echo ref rc=$?
