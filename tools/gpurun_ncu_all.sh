#!/bin/bash
# One ncu --set full capture of the dominant kernel per workload (traffic, occupancy, stalls),
# plus the c2 launch list. Each capture only after the same command ran clean without ncu.
# The reports are exported to CSV on the box and deleted (gpurun_out/ returns <= 64 MiB).
export BENCH_ALLOW_SHORT=1
TAG=${1:-r2}
run() { # name, bench args, kernel regex, skip, count, keep source page (0/1)
  local n=$1 a=$2 k=$3 s=$4 c=${5:-1} src=${6:-0}
  timeout 900 python bench.py $a --steps 1 --warmup 0 --skip-cpu --recall-q 0 --no-group-check --streams 1 > gpurun_out/${TAG}_${n}_plain.json 2> gpurun_out/${TAG}_${n}_plain.log || { echo "$n plain failed"; return; }
  timeout 1200 ncu --set full --clock-control none --import-source on -k "$k" -s $s -c $c -o /tmp/${TAG}_${n} -f python bench.py $a --steps 1 --warmup 0 --skip-cpu --recall-q 0 --no-group-check --streams 1 > gpurun_out/${TAG}_${n}_ncu.log 2>&1; echo "$n ncu rc=$?"
  ncu -i /tmp/${TAG}_${n}.ncu-rep --page raw --csv > gpurun_out/${TAG}_${n}_raw.csv 2>/dev/null
  if [ "$src" = 1 ]; then ncu -i /tmp/${TAG}_${n}.ncu-rep --page source --csv > gpurun_out/${TAG}_${n}_source.csv 2>/dev/null; fi
  rm -f /tmp/${TAG}_${n}.ncu-rep
}
run c2 "--config c2 --nq 2048 --gamma 0.8" 'regex:trim_knn_kernel' 1 1 1
run c1 "--config c1 --gamma 0.0" 'regex:trim_knn_kernel|trim_flat_dist' 0 2
run c4 "--config c4 --gamma 0.9" 'regex:trim_knn_kernel|trim_flat_dist' 0 2
run c3 "--config c3 --nq 1024 --gamma 0.8" 'regex:trim_range_flat_kernel|trim_range_kernel' 0
run c5 "--config c5 --nq 1024" 'regex:trim_knn_kernel|trim_knn_seg_plan' 0 5
C2="python bench.py --steps 1 --warmup 0 --skip-cpu --nq 4096 --recall-q 0 --no-group-check --gamma 0.8"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:trim_' -c 80 --csv --log-file gpurun_out/${TAG}_c2_launches.csv $C2 > gpurun_out/${TAG}_launch.log 2>&1; echo launches rc=$?
C1="python bench.py --config c1 --steps 1 --warmup 0 --skip-cpu --recall-q 0 --no-group-check --gamma 0.0"
TRIM_FLAT_PARTITION_MIN_ROWS=50000 TRIM_SEG_N0=8192 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:trim_' -c 400 --csv --log-file gpurun_out/${TAG}_c1seg_launches.csv $C1 > gpurun_out/${TAG}_launch_c1seg.log 2>&1; echo c1seg launches rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:trim_' -c 100 --csv --log-file gpurun_out/${TAG}_c1_launches.csv $C1 > gpurun_out/${TAG}_launch_c1.log 2>&1; echo c1 launches rc=$?
du -sh gpurun_out
