#!/bin/bash
# Round-2 final evidence: full GPU suite (incl. slow full-size tests), smoke(), the C3 bench
# line, the sharded step at one rank (torch.distributed + the gt_transpose_multi C-ABI leg).
set -u
D=gpurun_out/fin; mkdir -p $D
timeout 3000 python -m pytest tests -q -m gpu > $D/pytest_gpu_full.log 2>&1; echo "pytest rc=$?"; tail -3 $D/pytest_gpu_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $D/smoke.log
timeout 600 python bench.py > $D/bench_C3.json 2> $D/bench_C3.err; echo "bench rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --force-dist --capi --steps 10 --warmup 3 > $D/bench_sharded1_C3.json 2> $D/bench_sharded1.err; echo "sharded rc=$?"
tail -2 $D/bench_sharded1.err
