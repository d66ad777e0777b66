set -u
mkdir -p gpurun_out/ev
for k in k_p1 k_p2 k_p3; do
  timeout 240 ncu -f --set full --clock-control none -k regex:"$k" -s 2 -c 1 -o /tmp/full_$k python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev/ncu_full_$k.log 2>&1
  echo "$k full rc=$?"
  ncu -i /tmp/full_$k.ncu-rep --page raw --csv > gpurun_out/ev/raw_r01k_C3_$k.csv 2>/dev/null
done
timeout 400 python bench.py > gpurun_out/ev/bench_C3.json 2> gpurun_out/ev/bench_C3.err; echo "C3 rc=$?"
