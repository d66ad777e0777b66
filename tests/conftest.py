import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libgt.so")
    config.addinivalue_line("markers", "slow: full-size configs (C2/C3) on the GPU box")


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden_cases():
    z = np.load(GOLDEN / "cases.npz")
    out = {}
    for name in z["__names__"].tolist():
        out[name] = dict(
            nv=int(z[f"{name}__nv"][0]),
            off=z[f"{name}__off"],
            edg=z[f"{name}__edg"],
            toff=z[f"{name}__toff"],
            tedg=z[f"{name}__tedg"],
        )
    return out


@pytest.fixture(scope="session")
def golden_hashes():
    return json.loads((GOLDEN / "hashes.json").read_text())


def sha(*arrays) -> str:
    import hashlib

    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def random_graph(rng, max_vertices=1000, max_edges=10_000):
    """Random multigraph with self-loops, parallel edges, isolated vertices
    (same kind as the reference's conftest.random_graph, conftest.py:16-26)."""
    from paper_2501_06872_b200.graph import CsrGraph

    nv = int(rng.integers(1, max_vertices + 1))
    ne = int(rng.integers(0, max_edges + 1))
    src = rng.integers(0, nv, size=ne)
    if rng.random() < 0.5:
        dst = rng.integers(0, nv, size=ne)
    else:
        dst = np.minimum((nv * rng.random(ne) ** 3).astype(np.int64), nv - 1)
    return CsrGraph.from_edge_pairs(src, dst, nv)


def skewed_reference_graph():
    """potra.relabel_random(potra.generate_skewed(300000, 4000000, 1.1, seed=7),
    seed=8) restated in numpy (graph.py:187-222, 225-249): Zipf destinations by
    inverse CDF (searchsorted, 2^24-draw chunks), uniform sources, a seeded
    permutation of both endpoints, canonical CSR."""
    from paper_2501_06872_b200 import CsrGraph

    nv, ne, zipf = 300_000, 4_000_000, 1.1
    rng = np.random.default_rng(7)
    cdf = np.cumsum(np.arange(1, nv + 1, dtype=np.float64) ** -zipf)
    cdf /= cdf[-1]
    src = rng.integers(0, nv, size=ne, dtype=np.int64)
    dst = np.searchsorted(cdf, rng.random(ne), side="right")
    g = CsrGraph.from_edge_pairs(src, dst, nv)
    perm = np.random.default_rng(8).permutation(nv).astype(np.int64)
    owners = np.repeat(np.arange(nv, dtype=np.int64), np.diff(g.offsets.astype(np.int64)))
    return CsrGraph.from_edge_pairs(perm[owners], perm[g.edges.astype(np.int64)], nv)
