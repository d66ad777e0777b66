#!/bin/bash
# Final evidence of round 2 (fast rank/stage/write-out loops; usage: ev_final_r02.sh [tag]): full GPU suite,
# smoke(), then tools/ev_r02.sh (bench C2-C5 + reference arm, launch lists, ncu --set full).
set -u
D=gpurun_out/ev; mkdir -p $D
timeout 2400 python -m pytest tests -q -m gpu > $D/${1:-r02n}_pytest_gpu_full.log 2>&1; echo "pytest rc=$?"; tail -2 $D/${1:-r02n}_pytest_gpu_full.log | cut -c1-200
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/${1:-r02n}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $D/${1:-r02n}_smoke.log
bash tools/ev_r02.sh ${1:-r02n}
rm -f $D/*.ncu-rep
