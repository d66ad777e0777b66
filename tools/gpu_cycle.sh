#!/bin/bash
# One GPU round trip: parity tests (fast + full-size) and a short C3 bench.
# Usage: tools/gpu_cycle.sh [extra shell run on the box after the bench]
cd /root/repo
make -s -C paper_2501_06872_b200/csrc > /tmp/mk.log 2>&1 || { grep -B2 -A6 error /tmp/mk.log | head -40; echo BUILD_FAIL; exit 1; }
EXTRA="${1:-true}"
timeout 3000 /usr/local/graft/bin/gpurun --timeout 1500 -- "timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=\$?; tail -3 gpurun_out/pytest_gpu.log | cut -c1-300; timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_q.log 2>&1; echo bench_rc=\$?; tail -1 gpurun_out/bench_q.log | python3 -c \"import json,sys; d=json.loads(sys.stdin.read()); print('ms', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],4), {k:(round(v,3) if isinstance(v,float) else v) for k,v in d['roofline']['kernels'].items()})\"; $EXTRA" 2>&1 | grep -v "^\[gpurun\] sending"
