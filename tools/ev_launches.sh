#!/bin/bash
# Round evidence, part 1: per-launch ncu lists (time + DRAM bytes) for C3/C2/C4 and one
# `ncu --set full` capture per main C3 kernel, each after a plain run of the same command.
# Usage (on the GPU box): bash tools/ev_launches.sh r01h
set -u
R=${1:-r01m}
D=gpurun_out/ev; mkdir -p $D
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct
for c in C3 C2 C4; do
  timeout 120 python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $D/plain_$c.log 2>&1 || { echo "plain $c failed"; continue; }
  timeout 240 ncu --metrics $M --clock-control none --csv --log-file $D/launches_${R}_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $D/ncu_$c.log 2>&1
  echo "$c launches rc=$?"
done
for k in k_p1 k_p2 k_p3; do
  timeout 240 ncu -f --set full --clock-control none -k regex:"$k" -s 2 -c 1 -o /tmp/full_$k python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $D/ncu_full_$k.log 2>&1
  echo "$k full rc=$?"
  ncu -i /tmp/full_$k.ncu-rep --page raw --csv > $D/raw_${R}_C3_$k.csv 2>/dev/null
done
