"""Generate tests/golden/hdv_cases.npz by running the REAL reference's step 0
(``potra.sample_hdv``, hlh.py:167-218; ``coverage_exact``, hlh.py:221-228).

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_hdv_golden.py

Each case: a graph (this script's seeds: skewed-endpoint graphs shaped like
the reference's test_hlh.py helper, random multigraphs, a hub above 2^16
in-edges, Fig. 1, empty graphs) and a (k, sample_fraction, seed, threads)
choice; the reference's hdv_ids (order included), coverage_estimate,
sample_size and exact coverage are recorded.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

import potra  # noqa: E402  (the reference, from PYTHONPATH)


def make(src, dst, nv):
    return potra.CsrGraph.from_edge_pairs(np.asarray(src, np.int64), np.asarray(dst, np.int64), nv)


def skewed(nv, ne, hot, share, seed):
    rng = np.random.default_rng(seed)
    dst = rng.integers(0, nv, size=ne)
    dst[rng.random(ne) < share] = hot
    return make(rng.integers(0, nv, size=ne), dst, nv)


def graphs():
    rng = np.random.default_rng(20261020)
    out = {
        "fig1": make([0, 0, 1, 1, 2, 3], [1, 2, 2, 3, 3, 0], 4),
        "skew_20k": skewed(20_000, 50_000, 7, 0.9, 1),
        "skew_5k": skewed(5000, 20_000, 3, 0.4, 2),
        "skew_100k": skewed(100_000, 200_000, 11, 0.2, 4),
        "hub_over_2p16": skewed(1000, 200_000, 17, 0.5, 5),
        "no_edges_v17": make([], [], 17),
        "empty_v0": potra.CsrGraph(0, 0, np.zeros(1, np.uint64), np.empty(0, np.uint32)),
    }
    for i in range(6):
        nv = int(rng.integers(50, 3000))
        ne = int(rng.integers(0, 30_000))
        src = rng.integers(0, nv, ne)
        dst = np.minimum((nv * rng.random(ne) ** 4).astype(np.int64), nv - 1)
        out[f"random_{i}"] = make(src, dst, nv)
    return out


CHOICES = [  # (k, sample_fraction, seed, threads)
    (1, 0.5, 3, 2), (5, 0.2, 9, 2), (20, 1.0, 0, 1), (100, 1.0, 0, 2), (1000, 1.0, 0, 1),
    (50, 0.01, 0, 1), (50, 0.01, 7, 16), (300, 0.05, 123, 7), (0, 0.3, 1, 1), (10**9, 0.5, 5, 3),
]


def main():
    arrays = {}
    names = []
    for gname, g in graphs().items():
        arrays[f"{gname}__nv"] = np.array([g.num_vertices], np.int64)
        arrays[f"{gname}__off"] = g.offsets
        arrays[f"{gname}__edg"] = g.edges
        for ci, (k, frac, seed, threads) in enumerate(CHOICES):
            plan = potra.sample_hdv(g, k, sample_fraction=frac, seed=seed, threads=threads)
            name = f"{gname}__c{ci}"
            names.append(name)
            arrays[f"{name}__args"] = np.array([k, seed, threads], np.int64)
            arrays[f"{name}__frac"] = np.array([frac], np.float64)
            arrays[f"{name}__ids"] = plan.hdv_ids.astype(np.uint64)
            arrays[f"{name}__est"] = np.array([plan.coverage_estimate], np.float64)
            arrays[f"{name}__size"] = np.array([plan.sample_size], np.int64)
            arrays[f"{name}__exact"] = np.array([potra.coverage_exact(g, plan)], np.float64)
            for i, v in enumerate(plan.hdv_ids.tolist()):  # the reference's own lookups agree with the order
                assert potra.hash_lookup(plan, v) == i
    arrays["__names__"] = np.array(names)
    np.savez_compressed(HERE / "hdv_cases.npz", **arrays)
    print("wrote", len(names), "step-0 cases")


if __name__ == "__main__":
    main()
