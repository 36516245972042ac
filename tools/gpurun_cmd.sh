#!/bin/bash
# The round's GPU checks (run via: gpurun --timeout 3000 -- ./gpurun_cmd.sh):
# parity suite, smoke, and the default bench line.
export BENCH_ALLOW_SHORT=1
timeout -s KILL 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log; echo bench rc=$?
