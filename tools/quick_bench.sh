#!/bin/bash
# quick per-config bench lines: ms/step and per-kernel ms (usage: tools/quick_bench.sh C3 C2 ...)
for c in "$@"; do
  st=8; [ "$c" = C5 ] && st=3
  timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernels']; print('$c', round(d['ms_per_step'],3), round(k['step1_ms'],2), round(k['step2_ms'],2), round(k['step3_ms'],2), [round(x['ms'],3) for x in k['per_kernel']])"
done
