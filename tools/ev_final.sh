#!/bin/bash
# Round-end evidence on the final build (GPU box): full GPU suite, smoke, launch lists +
# ncu full of the main kernels (ev_launches.sh), bench lines (ev_bench.sh).
set -u
mkdir -p gpurun_out/ev
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/ev/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ev/pytest_gpu.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/ev/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/ev/smoke.log
bash tools/ev_launches.sh ${1:-r01m}
bash tools/ev_bench.sh | grep rc=
