"""Web-like generator (config C4): properties of the numpy restatement.  The
device generator is compared with it bit for bit in test_gpu_parity.py."""

import numpy as np

from conftest import ROOT  # noqa: F401  (sys.path)
from paper_2501_06872_b200 import gen

WP = gen.WebParams(hubs=1 << 10, window=256)


def test_thresholds_monotone_and_capped():
    dt, ht, sq = gen.web_tables(1 << 16, 1 << 20, WP)
    assert dt.dtype == np.uint64 and ht.dtype == np.uint64
    assert np.all(dt[1:] >= dt[:-1]) and np.all(ht[1:] >= ht[:-1])
    assert dt[-1] == np.uint64(2**64 - 1) and ht[-1] == np.uint64(2**64 - 1)
    assert dt.shape[0] == WP.deg_max and ht.shape[0] == WP.hubs
    assert sq > 0


def test_degrees_and_edge_count():
    dt, _, sq = gen.web_tables(1 << 16, 1 << 20, WP)
    deg = gen.web_degrees_np(1 << 16, 7, dt, sq)
    assert deg.min() >= 1
    src, dst = gen.web_pairs_np(1 << 16, 1 << 20, 7, WP)
    assert src.shape[0] == int(deg.sum())
    assert abs(src.shape[0] / (1 << 20) - 1) < 0.1  # rescaled to the target edge count
    assert np.array_equal(np.bincount(src, minlength=1 << 16), deg.astype(np.int64))
    assert np.all(np.diff(src.astype(np.int64)) >= 0)  # generation order = source order


def test_locality_and_hubs():
    V = 1 << 16
    src, dst = gen.web_pairs_np(V, 1 << 20, 7, WP)
    d = (dst.astype(np.int64) - src.astype(np.int64)) % V
    local = np.minimum(d, V - d) <= WP.window
    assert 0.83 < local.mean() < 0.90  # p_local = 0.85 (+ hubs that fall in the window)
    hubs = gen.web_hub_ids(V, WP.hubs, 7)
    assert np.unique(hubs).shape[0] == WP.hubs  # distinct (Feistel bijection)
    far = dst[~local]
    assert np.isin(far, hubs).all()
    # Zipf(1.2) over ranks: the rank-0 hub is the most popular far destination
    vals, cnt = np.unique(far, return_counts=True)
    assert vals[np.argmax(cnt)] == hubs[0]


def test_deterministic():
    a = gen.web_pairs_np(1 << 12, 1 << 16, 3, WP)
    b = gen.web_pairs_np(1 << 12, 1 << 16, 3, WP)
    c = gen.web_pairs_np(1 << 12, 1 << 16, 4, WP)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert not np.array_equal(a[1], c[1])
