for cfg in "GT_K2=16" "GT_K2=32"; do
  for c in C4 C3; do
  r=$(env $cfg timeout 200 python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernels']; print(round(d['ms_per_step'],3), round(k['step1_ms'],3), round(k['step2_ms'],3), round(k['step3_ms'],3), [round(x['ms'],3) for x in k['per_kernel']])")
  echo "$cfg $c : $r"
  done
done
