for cfg in "GT_SPLIT=9,8,7 GT_W3=16" "GT_SPLIT=9,8,7 GT_W3=32" "GT_SPLIT=9,7,8 GT_W3=16" "GT_SPLIT=9,7,8 GT_W3=32" "GT_SPLIT=8,8,8 GT_W3=32"; do
  r=$(env $cfg timeout 200 python bench.py --config C3 --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernels']; print(round(d['ms_per_step'],3), k['digit_bits'], round(k['step1_ms'],3), round(k['step2_ms'],3), round(k['step3_ms'],3), [round(x['ms'],3) for x in k['per_kernel']], k['big_buckets'])")
  echo "$cfg : $r"
done
