#!/bin/bash
# LUT build in code-major order: parity subset + c2/c4/c1 bench lines.
export BENCH_ALLOW_SHORT=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_range.py tests/test_gpu_graph.py tests/test_gpu_probe.py tests/test_gpu_multi.py -q -x > gpurun_out/r2c_tests.log 2>&1; echo tests rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py --skip-cpu --no-group-check > gpurun_out/r2c_c2.json 2> gpurun_out/r2c_c2.log; echo c2 rc=$?
timeout 900 python bench.py --config c4 --skip-cpu --steps 3 > gpurun_out/r2c_c4.json 2> gpurun_out/r2c_c4.log; echo c4 rc=$?
timeout 900 python bench.py --config c1 --skip-cpu > gpurun_out/r2c_c1.json 2> gpurun_out/r2c_c1.log; echo c1 rc=$?
