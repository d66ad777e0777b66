for args in "" "--split 9,9,8 --force-wide" "--split 10,9,7 --force-wide" "--split 9,10,7 --force-wide" "--force-wide"; do
  timeout 300 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $args 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernels']; print('$args', round(d['ms_per_step'],3), k['digit_bits'], round(k['step1_ms'],3), round(k['step2_ms'],3), round(k['step3_ms'],3), [round(x['ms'],3) for x in k['per_kernel']])"
done
for args in "" "--split 8,8,8" "--split 9,8,7 --force-wide"; do
  timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $args 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernels']; print('C3 $args', round(d['ms_per_step'],3), k['digit_bits'], [round(x['ms'],3) for x in k['per_kernel']])"
done
