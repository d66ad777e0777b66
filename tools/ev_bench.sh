#!/bin/bash
# Round evidence, part 2: bench lines (C3 default = the driver's line, the reference arm,
# C2/C4 with e2e + CPU baseline, C5 device-only).  Usage (GPU box): bash tools/ev_bench.sh
set -u
D=gpurun_out/ev; mkdir -p $D
timeout 400 python bench.py > $D/bench_C3.json 2> $D/bench_C3.err; echo "C3 rc=$?"
timeout 400 python bench.py --impl reference > $D/bench_reference.json 2> $D/bench_reference.err; echo "ref rc=$?"
for c in C2 C4; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 > $D/bench_$c.json 2> $D/bench_$c.err; echo "$c rc=$?"; done
timeout 400 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $D/bench_C5.json 2> $D/bench_C5.err; echo "C5 rc=$?"
for f in $D/bench_*.json; do tail -1 $f | cut -c1-300; done
