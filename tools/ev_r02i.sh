#!/bin/bash
# Round-2 (i) evidence: GPU suite on the fast-loop build, C3 bench, source-level ncu of the
# three place kernels (per-line instruction / stall / bank-conflict summaries).
set -u
D=gpurun_out/r02i; mkdir -p $D
timeout 1500 python -m pytest tests -x -q -m "gpu and not slow" > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $D/pytest_gpu.log | cut -c1-200
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $D/bench_C3_device.json 2> $D/bench.err; echo "bench rc=$?"
for k in k_p1 "k_p2.*DecR1" k_p3; do
  n=$(echo $k | tr -cd 'a-z0-9_')
  timeout 600 ncu -f --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"$k" -s 2 -c 1 -o /tmp/src_$n python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $D/ncu_$n.log 2>&1; echo "$n=$?"
  python tools/ncu_lines.py /tmp/src_$n.ncu-rep 70 > $D/lines_C3_$n.txt 2>&1
  ncu -i /tmp/src_$n.ncu-rep --page raw --csv > $D/raw_C3_$n.csv 2>/dev/null
done
ls -la $D
