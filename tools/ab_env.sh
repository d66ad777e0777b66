#!/bin/bash
# A/B of env settings on one config: tools/ab_env.sh C5 "X=0" "GT_K2=16" ...
c=$1; shift
st=8; [ "$c" = C5 ] && st=3
for cfg in "$@"; do
  r=$(env $cfg timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernels']; print(round(d['ms_per_step'],3), round(k['step1_ms'],2), round(k['step2_ms'],2), round(k['step3_ms'],2), k['digit_bits'], k['big_buckets'], [round(x['ms'],3) for x in k['per_kernel']])")
  echo "$c $cfg : $r"
done
