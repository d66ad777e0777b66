#!/bin/bash
# Round-2 evidence on the GPU box: launch lists (time + DRAM bytes per launch) for C3/C2/C4,
# `ncu --set full` of the main C3 kernels (each after a plain run), bench lines for C2-C5
# and the reference arm.  Usage: bash tools/ev_r02.sh r02d
set -u
R=${1:-r02d}
D=gpurun_out/ev; mkdir -p $D
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct
timeout 400 python bench.py --steps 20 --warmup 3 > $D/bench_${R}_C3.json 2> $D/bench_C3.err; echo "bench C3 rc=$?"
for c in C2 C4; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $D/bench_${R}_$c.json 2> $D/bench_$c.err; echo "bench $c rc=$?"
done
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $D/bench_${R}_C5.json 2> $D/bench_C5.err; echo "bench C5 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $D/bench_${R}_reference.json 2> $D/bench_ref.err; echo "reference rc=$?"
for c in C3 C2 C4; do
  timeout 120 python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $D/plain_$c.log 2>&1 || { echo "plain $c failed"; continue; }
  timeout 300 ncu --metrics $M --clock-control none --csv --log-file $D/launches_${R}_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $D/ncu_$c.log 2>&1
  echo "$c launches rc=$?"
done
for k in k_p1 k_p2 k_p3; do
  timeout 300 ncu -f --set full --clock-control none --import-source on -k regex:"$k" -s 2 -c 1 -o $D/full_${R}_$k python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $D/ncu_full_$k.log 2>&1
  echo "$k full rc=$?"
  ncu -i $D/full_${R}_$k.ncu-rep --page raw --csv > $D/raw_${R}_C3_$k.csv 2>/dev/null
done
ls -la $D
