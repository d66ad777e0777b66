"""The CPU oracle (test infrastructure) pinned against the reference's outputs.

tests/golden/*.npz|json were produced by the real reference
(potra.transpose_oracle etc.) — see tests/golden/make_golden.py."""

import numpy as np
import pytest

from conftest import ROOT, sha

import sys

sys.path.insert(0, str(ROOT))
from oracle import oracle  # noqa: E402


def test_numpy_oracle_matches_reference_goldens(golden_cases):
    for name, c in golden_cases.items():
        toff, tedg = oracle.transpose_np(c["off"], c["edg"], c["nv"])
        assert toff.dtype == np.uint64 and tedg.dtype == np.uint32
        assert np.array_equal(toff, c["toff"]), name
        assert np.array_equal(tedg, c["tedg"]), name


def test_c_oracle_matches_reference_goldens(golden_cases):
    for name, c in golden_cases.items():
        toff, tedg = oracle.transpose_c(c["off"], c["edg"], c["nv"])
        assert np.array_equal(toff, c["toff"]), name
        assert np.array_equal(tedg, c["tedg"]), name


@pytest.mark.parametrize("threads", [1, 2, 3, 8])
def test_cpu_baseline_ports_match_goldens(golden_cases, threads):
    for name, c in golden_cases.items():
        if len(c["edg"]) == 0 and c["nv"] == 0:
            continue
        toff, tedg = oracle.transpose_scantrans_c(c["off"], c["edg"], c["nv"], threads)
        assert np.array_equal(toff, c["toff"]) and np.array_equal(tedg, c["tedg"]), (name, "scantrans")
        toff, tedg = oracle.transpose_atomic_sorted_c(c["off"], c["edg"], c["nv"], threads)
        assert np.array_equal(toff, c["toff"]) and np.array_equal(tedg, c["tedg"]), (name, "atomic+sort")


def test_c1_oracle_hash_matches_reference(golden_hashes):
    from paper_2501_06872_b200 import gen

    cfg = gen.CONFIGS["C1"]
    off, edg = gen.generate_np(cfg)
    assert sha(off, edg) == golden_hashes["C1"]["input"]
    toff, tedg = oracle.transpose_c(off, edg, cfg.num_vertices)
    assert sha(toff, tedg) == golden_hashes["C1"]["oracle"]
    toff2, tedg2 = oracle.transpose_np(off, edg, cfg.num_vertices)
    assert sha(toff2, tedg2) == golden_hashes["C1"]["oracle"]
    assert golden_hashes["C1"]["atomic_sorted_equals_oracle"] and golden_hashes["C1"]["scantrans_equals_oracle"]


def test_edge_balanced_bounds_match_reference(golden_hashes):
    from paper_2501_06872_b200 import gen

    off, _ = gen.generate_np(gen.CONFIGS["C1"])
    for parts, want in golden_hashes["C1_edge_balanced_bounds"].items():
        assert oracle.edge_balanced_bounds_np(off, int(parts)).tolist() == want
        assert oracle.edge_balanced_bounds_c(off, int(parts)).tolist() == want
    probe = np.array([0, 5, 5, 6, 20, 21, 30], dtype=np.uint64)
    assert oracle.edge_balanced_bounds_c(probe, 3).tolist() == golden_hashes["survey_probe_bounds_parts3"]


def test_prefix_sum_port_matches_reference(golden_hashes):
    import ctypes

    counts = np.random.default_rng(19).integers(0, 1000, size=100_000)
    c32 = counts.astype(np.uint32)
    out = np.empty(c32.size + 1, dtype=np.uint64)
    lib = oracle.load()
    assert lib.gto_scan_exclusive(oracle._p(c32), c32.size, oracle._p(out), 7) == 0
    assert sha(out) == golden_hashes["prefix_sum_100k_seed19"]


def test_scantrans_refuses_2_32_edges_like_reference():
    # baselines.py:278-281: |E| >= 2^32 -> CounterOverflowError; the port returns EOVERFLOW
    lib = oracle.load()
    off = np.array([0, 1 << 32], dtype=np.uint64)
    rc = lib.gto_transpose_scantrans(oracle._p(off), None, 1, 1 << 32, None, None, 2)
    assert rc == oracle.GTO_EOVERFLOW


def test_reference_importable_cross_check():
    """When the reference is importable (build container), re-derive one golden live."""
    pytest.importorskip("numba")
    try:
        sys.path.insert(0, "/root/reference/pkg/src")
        import potra  # noqa: F401
    except Exception:
        pytest.skip("reference not importable here")
    rng = np.random.default_rng(5)
    for _ in range(20):
        nv = int(rng.integers(1, 500))
        ne = int(rng.integers(0, 3000))
        g = potra.CsrGraph.from_edge_pairs(rng.integers(0, nv, ne), rng.integers(0, nv, ne), nv)
        t = potra.transpose_oracle(g)
        toff, tedg = oracle.transpose_c(g.offsets, g.edges, nv)
        assert np.array_equal(toff, t.offsets) and np.array_equal(tedg, t.edges)


@pytest.mark.parametrize("threads", [1, 3, 8])
@pytest.mark.parametrize("method", [None, "atomic", "hlh"])
def test_potra_port_sorted_matches_goldens(golden_cases, threads, method):
    """OpenMP port of transpose_potra (hlh.py:441-588) + sort_neighbor_lists == transpose_oracle."""
    for name, c in golden_cases.items():
        if c["nv"] == 0:
            continue
        toff, tedg, info = oracle.transpose_potra_c(c["off"], c["edg"], c["nv"], threads, k=min(64, c["nv"]),
                                                    force_method=method, sort=True)
        assert np.array_equal(toff, c["toff"]) and np.array_equal(tedg, c["tedg"]), (name, method)
        if method is not None:
            assert info["method_chosen"] == method


def test_potra_port_step0_matches_sample_restatement():
    """The port's HDV selection = sample_hdv_np (pinned by tests/golden/hdv_cases.npz)."""
    from paper_2501_06872_b200 import gen

    off, edg = gen.generate_np(gen.CONFIGS["C1"])
    for k, frac, seed, thr in [(100, 0.01, 0, 4), (1000, 0.05, 7, 3), (50, 1.0, 0, 2)]:
        ids, est, size = oracle.sample_hdv_np(edg, 1 << 16, k, frac, seed, thr)
        _, _, info = oracle.transpose_potra_c(off, edg, 1 << 16, thr, k=k, sample_fraction=frac, seed=seed,
                                              force_method="hlh")
        assert info["k"] == len(ids) and info["sample_size"] == size
        assert abs(info["coverage_estimate"] - est) < 1e-12


@pytest.mark.parametrize("name", ["C1"])
def test_host_generator_matches_numpy_generator(name):
    """oracle.generate_c (bench.py's reference-arm input) == gen.generate_np, bit for bit."""
    import dataclasses

    from paper_2501_06872_b200 import gen

    cfgs = [gen.CONFIGS[name],
            dataclasses.replace(gen.CONFIGS["C2"], num_vertices=1 << 14, num_edges=1 << 18),
            dataclasses.replace(gen.CONFIGS["C3"], num_vertices=1 << 13, num_edges=1 << 17, scale=13)]
    for cfg in cfgs:
        o1, e1 = gen.generate_np(cfg)
        o2, e2 = oracle.generate_c(cfg, 4)
        assert np.array_equal(o1, o2) and np.array_equal(e1, e2), cfg.name


def test_skewed_4m_generator_restatement_and_oracle(golden_hashes):
    """The restated skewed_4m generator (conftest.skewed_reference_graph)
    reproduces the reference's input bit for bit, and the C oracle's transpose
    of it hashes to the reference's transpose_oracle output."""
    from conftest import sha, skewed_reference_graph

    g = skewed_reference_graph()
    assert sha(g.offsets, g.edges) == golden_hashes["skewed_4m"]["input"]
    o, e = oracle.transpose_c(g.offsets, g.edges, g.num_vertices)
    assert sha(o, e) == golden_hashes["skewed_4m"]["oracle"]
