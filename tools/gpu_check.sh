#!/bin/bash
# Rebuild libgt.so; on success run the GPU parity tests + a short C3 bench on the B200 box.
set -u
cd /root/repo
make -s -C paper_2501_06872_b200/csrc > /tmp/mk.log 2>&1
if grep -q "error" /tmp/mk.log; then grep -B2 -A5 error /tmp/mk.log | head -40; echo BUILD_FAIL; exit 1; fi
EXTRA="${1:-}"
timeout 2400 /usr/local/graft/bin/gpurun --timeout 1200 -- "timeout 600 python -m pytest tests -x -q -m 'gpu and not slow' > gpurun_out/pytest_gpu.log 2>&1; echo rc=\$?; tail -2 gpurun_out/pytest_gpu.log; $EXTRA timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench3.log 2>&1; echo bench_rc=\$?; grep fprof gpurun_out/bench3.log | tail -1 | cut -c1-400; tail -1 gpurun_out/bench3.log | python3 -c \"import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d['roofline']['frac'],4), {k:(round(v,3) if isinstance(v,float) else v) for k,v in d['roofline']['kernels'].items()})\"" 2>&1 | grep -v "^\[gpurun\] sending" | tail -8
