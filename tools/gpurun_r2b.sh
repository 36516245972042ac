#!/bin/bash
# Round 2: the reworked bench (torch fixture in both arms, shared config dict,
# one-process multi-device mode, 1-thread CPU figure) — default line, the
# reference arm, --gpus 1 --group, and torchrun one-rank shard.
export BENCH_ALLOW_SHORT=1
timeout 900 python bench.py > gpurun_out/r2b_c2.json 2> gpurun_out/r2b_c2.log; echo c2 rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2b_ref.json 2> gpurun_out/r2b_ref.log; echo ref rc=$?
timeout 600 python bench.py --gpus 1 --group --skip-cpu --steps 3 > gpurun_out/r2b_group.json 2> gpurun_out/r2b_group.log; echo group rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --force-shard --skip-cpu --steps 3 > gpurun_out/r2b_shard.json 2> gpurun_out/r2b_shard.log; echo shard rc=$?
