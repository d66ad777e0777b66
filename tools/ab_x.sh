for cfg in "X=0" "X=1"; do
  for c in C3 C4; do
  r=$(env $cfg timeout 200 python bench.py --config $c --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernels']; print(round(d['ms_per_step'],3), [round(x['ms'],3) for x in k['per_kernel']])")
  echo "$cfg $c : $r"
  done
done
