#!/bin/bash
# Round-1 re-check of the non-default bench lines from a fresh build, plus the
# id-sharded path (NCCL all-gather + device merge) at one rank under torchrun.
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --force-shard --skip-cpu > gpurun_out/bench_c2_shard1.json 2> gpurun_out/bench_c2_shard1.log; echo shard rc=$?
for c in c3 c4 g1; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.log; echo $c rc=$?
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_c2_ref.json 2> gpurun_out/bench_c2_ref.log; echo ref rc=$?
