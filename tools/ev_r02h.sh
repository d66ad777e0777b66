#!/bin/bash
# `ncu --set full` of the C3 kernels round 2's first capture left out: the
# level-3 big-bucket place (k_p2<DecR2>), the count passes (k_c1, k_cnt_rec)
# and the scan, each after a plain run.  Usage: bash tools/ev_r02h.sh r02h
set -u
R=${1:-r02h}
D=gpurun_out/ev; mkdir -p $D
timeout 120 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $D/plain_C3.log 2>&1 || { echo "plain failed"; exit 1; }
cap() {  # name regex skip
  timeout 300 ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$2" -s $3 -c 1 \
    -o $D/full_${R}_$1 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $D/ncu_full_$1.log 2>&1
  echo "$1 full rc=$?"
  ncu -i $D/full_${R}_$1.ncu-rep --page raw --csv > $D/raw_${R}_C3_$1.csv 2>/dev/null
  ncu -i $D/full_${R}_$1.ncu-rep --page details --csv > $D/details_${R}_C3_$1.csv 2>/dev/null
  rm -f $D/full_${R}_$1.ncu-rep  # (64 MiB copy-back limit)
}
cap k_p2_big "k_p2.*DecR2" 2
cap k_c1 "k_c1" 2
cap k_cnt_rec "k_cnt_rec" 2
cap k_scan "k_scan_lookback" 4
ls -la $D
