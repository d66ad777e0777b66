"""Small transposes for compute-sanitizer (racecheck / memcheck / synccheck):
C1, a hub graph (level-3 big buckets), the wide form, and the sharded
building blocks, in both rank modes, each checked against the oracle.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import oracle  # noqa: E402  (test infrastructure: the checker)
from paper_2501_06872_b200 import CsrGraph, gen, pipeline_config, set_rank_mode, transpose_gpu  # noqa: E402
from paper_2501_06872_b200.multi import GpuShardBackend, plan_shards, transpose_sharded_local  # noqa: E402


def check(g, out_off, out_edg, what):
    o, e = oracle.transpose_c(g.offsets, g.edges, g.num_vertices)
    ok = np.array_equal(out_off, o) and np.array_equal(out_edg, e)
    print(f"{what}: {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        raise SystemExit(1)


def main():
    cfg = gen.CONFIGS["C1"]
    off, edg = gen.generate_np(cfg)
    c1 = CsrGraph(cfg.num_vertices, cfg.num_edges, off, edg)
    rng = np.random.default_rng(4)
    nv = 30_000
    src = np.sort(rng.integers(0, nv, 400_000))
    dst = np.where(rng.random(src.size) < 0.4, 123, np.minimum((nv * rng.random(src.size) ** 4).astype(np.int64), nv - 1))
    hub = CsrGraph.from_edge_pairs(src, dst, nv)
    for mode in (0, 1):
        set_rank_mode(mode)
        for name, g in (("C1", c1), ("hub", hub)):
            out = transpose_gpu(g)
            check(g, out.graph.offsets, out.graph.edges, f"{name} rank-mode {mode}")
        with pipeline_config(force_wide=True):
            out = transpose_gpu(hub)
            check(hub, out.graph.offsets, out.graph.edges, f"hub wide rank-mode {mode}")
        toff, tedg = transpose_sharded_local(hub, plan_shards(hub.offsets, 2), GpuShardBackend())
        check(hub, toff, tedg, f"hub sharded P=2 rank-mode {mode}")
    set_rank_mode(-1)
    print("all cases ok")


if __name__ == "__main__":
    main()
