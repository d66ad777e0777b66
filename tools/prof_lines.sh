#!/bin/bash
# Source-level ncu of the C3 place kernels: per-line instruction / stall tables (all lines) and raw metrics.
# Usage: bash tools/prof_lines.sh <tag>   -> gpurun_out/<tag>/
set -u
D=gpurun_out/${1:-prof}; mkdir -p $D
for k in k_p1 "k_p2.*DecR1" k_p3 "k_p2.*DecR2"; do
  n=$(echo $k | tr -cd 'a-zA-Z0-9_')
  timeout 600 ncu -f --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"$k" -s 2 -c 1 -o /tmp/src_$n python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $D/ncu_$n.log 2>&1; echo "$n=$?"
  python tools/ncu_lines.py /tmp/src_$n.ncu-rep 3000 > $D/all_lines_$n.txt 2>&1
  ncu -i /tmp/src_$n.ncu-rep --page raw --csv > $D/raw_C3_$n.csv 2>/dev/null
done
