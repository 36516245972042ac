#!/bin/bash
# multi-round segmented flat kNN: full GPU suite, smoke, bench lines (c2 default, c1, c5), ncu of c5 / c1
export BENCH_ALLOW_SHORT=1
timeout -s KILL 1800 python -m pytest tests -m gpu -q -x --durations=6 > gpurun_out/r2p_gpu.log 2>&1; echo gpu rc=$?
tail -4 gpurun_out/r2p_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2p_smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/r2p_c2.json 2> gpurun_out/r2p_c2.log; echo c2 rc=$?
timeout 600 python bench.py --config c1 > gpurun_out/r2p_c1.json 2> gpurun_out/r2p_c1.log; echo c1 rc=$?
timeout 1500 python bench.py --config c5 --steps 2 --warmup 1 > gpurun_out/r2p_c5.json 2> gpurun_out/r2p_c5.log; echo c5 rc=$?
for f in c2 c1 c5; do python -c "
import json;d=json.loads(open('gpurun_out/r2p_$f.json').read().strip().splitlines()[-1]);print('$f',d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline'].get('list_skip_fraction'),d['e2e']['value'])"; done
TAG=r02b
run() { # name, bench args, kernel regex, skip, count
  local n=$1 a=$2 k=$3 s=$4 c=${5:-1}
  timeout 1200 ncu --set full --clock-control none --import-source on -k "$k" -s $s -c $c -o /tmp/${TAG}_${n} -f python bench.py $a --steps 1 --warmup 0 --skip-cpu --recall-q 0 --no-group-check --streams 1 > gpurun_out/${TAG}_${n}_ncu.log 2>&1; echo "$n ncu rc=$?"
  ncu -i /tmp/${TAG}_${n}.ncu-rep --page raw --csv > gpurun_out/${TAG}_${n}_raw.csv 2>/dev/null
  rm -f /tmp/${TAG}_${n}.ncu-rep
}
run c5 "--config c5 --nq 1024" 'regex:trim_knn_kernel|trim_knn_seg_plan' 0 10
run c1 "--config c1 --gamma 0.0" 'regex:trim_knn_kernel|trim_knn_seg_plan|trim_flat_dist' 0 11
du -sh gpurun_out
