"""Probe: per-kernel times of the transpose on a seeded permuted R-MAT graph
of a given scale / edge count (tools/wide_probe.py SCALE LOG2_EDGES [reps])."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_06872_b200 import gen, transpose_device  # noqa: E402

scale, le = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = gen.GraphConfig(f"rmat-s{scale}-e2^{le}", "rmat", 1 << scale, 1 << le, scale=scale, permute=True, seed=7)
off, edg = gen.generate_device(cfg)
t_off = torch.empty_like(off)
t_edg = torch.empty_like(edg)
for r in range(reps):
    _, _, st = transpose_device(off, edg, cfg.num_vertices, t_offsets=t_off, t_edges=t_edg, want_stats=True)
    torch.cuda.synchronize()
    E = cfg.num_edges
    print(f"s{scale} E=2^{le} rep{r}: total {st.ms_total:.2f} ms ({st.ms_total * 1e9 / E:.2f} ps/edge) "
          f"steps {st.ms_step1:.2f}/{st.ms_step2:.2f}/{st.ms_step3:.2f} kernels "
          f"{[round(x, 2) for x in st.ms_kernel]} bits {list(st.bits)} big {st.n_big_buckets}", flush=True)
