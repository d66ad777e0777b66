# Source-level ncu capture of the main C3 kernels; reduces each report to text on the box
# (full reports exceed gpurun's copy-back limit).  Usage: bash tools/ncu_src.sh [kernels...]
set -u
KS="${*:-k_p1 k_p2 k_p3}"
CFG="${CFG:-C3}"
python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1; echo plain=$?
for k in $KS; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$k" -s 2 -c 1 -o /tmp/src_${CFG}_$k python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${CFG}_$k.log 2>&1; echo $k=$?
  python tools/ncu_lines.py /tmp/src_${CFG}_$k.ncu-rep 60 > gpurun_out/lines_${CFG}_$k.txt 2>&1
  ncu -i /tmp/src_${CFG}_$k.ncu-rep --page source --csv --print-source cuda,sass > /tmp/srcdump_${CFG}_$k.csv 2>/dev/null; gzip -c /tmp/srcdump_${CFG}_$k.csv > gpurun_out/srcdump_${CFG}_$k.csv.gz
  ncu -i /tmp/src_${CFG}_$k.ncu-rep --page raw --csv > gpurun_out/raw_${CFG}_$k.csv 2>/dev/null
  ls -la /tmp/src_${CFG}_$k.ncu-rep gpurun_out/srcdump_${CFG}_$k.csv.gz
done
