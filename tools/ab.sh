#!/bin/bash
# A/B of experiment bits on one config: tools/ab.sh C3 "0 1" [steps]
c=${1:-C3}; exps=${2:-"0 1"}; st=${3:-10}
for rep in 1 2; do
for x in $exps; do
  timeout 300 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --no-e2e --experiment $x 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernels']; print('$c exp=$x', round(d['ms_per_step'],3), round(k['step1_ms'],3), round(k['step2_ms'],3), round(k['step3_ms'],3), [round(x['ms'],3) for x in k['per_kernel']])"
done; done
