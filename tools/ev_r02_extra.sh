#!/bin/bash
# Round-2 extra evidence: C5 per-kernel launch list (main kernels only, one transpose after
# warm-up) and `ncu --set full` of the level-3 big-bucket place kernel on C3.
set -u
D=gpurun_out/ev2; mkdir -p $D
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct
timeout 900 python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-graph > $D/plain_C5.log 2>&1; echo "plain C5 rc=$?"
timeout 1500 ncu --metrics $M --clock-control none -k regex:"k_c1|k_p1|k_cnt|k_p2|k_p3|k_scan|k_segfix" --csv --log-file $D/launches_r02e_C5.csv python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-graph > $D/ncu_C5.log 2>&1; echo "C5 launches rc=$?"
timeout 120 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $D/plain_C3.log 2>&1; echo "plain C3 rc=$?"
timeout 300 ncu -f --set full --clock-control none --import-source on -k regex:"DecR2" -s 2 -c 1 -o $D/full_r02e_k_p2big python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $D/ncu_full_big.log 2>&1; echo "big full rc=$?"
ncu -i $D/full_r02e_k_p2big.ncu-rep --page raw --csv > $D/raw_r02e_C3_k_p2big.csv 2>/dev/null
ls -la $D
