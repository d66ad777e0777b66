"""Debug helper: one small graph through the wide v3 form (GT_WIDE=1)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("GT_WIDE", "1")
from oracle import oracle  # noqa: E402  (test infrastructure)
from paper_2501_06872_b200 import CsrGraph, transpose_gpu  # noqa: E402

rng = np.random.default_rng(1)
nv, ne = int(sys.argv[1]) if len(sys.argv) > 1 else 3000, int(sys.argv[2]) if len(sys.argv) > 2 else 40000
src = rng.integers(0, nv, ne)
dst = rng.integers(0, nv, ne)
g = CsrGraph.from_edge_pairs(src, dst, nv)
out = transpose_gpu(g)
toff, tedg = oracle.transpose_c(g.offsets, g.edges, nv)
print("offsets ok", np.array_equal(out.graph.offsets, toff), "edges ok", np.array_equal(out.graph.edges, tedg),
      out.details)
