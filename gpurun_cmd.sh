#!/bin/bash
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest.log
timeout 600 python tests/perf_modes.py --gammas 0.8,0.6 --reps 3 2>&1 | grep gamma | tail -2
cat gpurun_out/pytest.log
