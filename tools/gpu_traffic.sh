#!/bin/bash
# Launch lists (ncu, per-kernel DRAM bytes) for C2/C3/C4 after a plain run of the same command.
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,l1tex__throughput.avg.pct_of_peak_sustained_active
for c in C3 C2 C4; do
  python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_$c.log 2>&1 && \
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_r01d_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$c.log 2>&1
  echo "$c rc=$?"
done
