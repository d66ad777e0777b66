"""Step 0 (the HDV sample): the numpy restatement and the
GPU path against the reference's own outputs (tests/golden/hdv_cases.npz,
made by tests/golden/make_hdv_golden.py from potra.sample_hdv)."""

import sys

import numpy as np
import pytest

from conftest import ROOT

sys.path.insert(0, str(ROOT))
from oracle import oracle  # noqa: E402  (test infrastructure)


@pytest.fixture(scope="module")
def hdv_cases():
    z = np.load(ROOT / "tests" / "golden" / "hdv_cases.npz")
    out = []
    for name in z["__names__"]:
        g = str(name).split("__")[0]
        k, seed, threads = z[f"{name}__args"].tolist()
        out.append(dict(name=str(name), nv=int(z[f"{g}__nv"][0]), off=z[f"{g}__off"], edg=z[f"{g}__edg"], k=k,
                        seed=seed, threads=threads, frac=float(z[f"{name}__frac"][0]), ids=z[f"{name}__ids"],
                        est=float(z[f"{name}__est"][0]), size=int(z[f"{name}__size"][0]),
                        exact=float(z[f"{name}__exact"][0])))
    return out


def test_oracle_sample_hdv_matches_reference(hdv_cases):
    for c in hdv_cases:
        ids, est, size = oracle.sample_hdv_np(c["edg"], c["nv"], c["k"], c["frac"], c["seed"], c["threads"])
        assert np.array_equal(ids, c["ids"]), c["name"]
        assert est == c["est"] and size == c["size"], c["name"]


def test_budget_and_eq1():
    from paper_2501_06872_b200 import HdvBudget, hdv_count
    from paper_2501_06872_b200.hdv import fit_table_budget

    # Eq. 1 (model.py:66-75): 1 MiB, 12-byte records at load 0.5, 13 B x 4 threads per HDV
    b = HdvBudget(cache_bytes=1 << 20, threads=4)
    k = hdv_count(b).k
    assert k == (1 << 20) // (24 + 52)
    assert hdv_count(b).implied_bytes <= b.cache_bytes
    kf = fit_table_budget(k, 0.5, 4, 1 << 20)
    cap = 1 << max(1, (int(np.ceil(kf / 0.5)) - 1).bit_length())
    assert 0 < kf <= k and 12 * cap + 13 * 4 * kf <= (1 << 20)
    for bad in (dict(cache_bytes=0), dict(cache_bytes=10, load_factor=0.0), dict(cache_bytes=10, threads=0)):
        with pytest.raises(ValueError):
            HdvBudget(**bad)


@pytest.mark.gpu
def test_gpu_sample_hdv_matches_reference(hdv_cases):
    from paper_2501_06872_b200 import CsrGraph, coverage_exact, hash_lookup, sample_hdv
    from paper_2501_06872_b200.hdv import hash_lookup_gpu

    for c in hdv_cases:
        g = CsrGraph(c["nv"], int(c["edg"].shape[0]), c["off"].astype(np.uint64), c["edg"].astype(np.uint32))
        plan = sample_hdv(g, c["k"], sample_fraction=c["frac"], seed=c["seed"], threads=c["threads"])
        assert plan.hdv_ids.dtype == np.uint64
        assert np.array_equal(plan.hdv_ids, c["ids"]), c["name"]
        assert plan.coverage_estimate == c["est"] and plan.sample_size == c["size"], c["name"]
        assert plan.k == len(c["ids"]) and plan.k / plan.capacity <= 0.5
        for i, v in enumerate(plan.hdv_ids.tolist()[:50]):
            assert hash_lookup(plan, v) == i
        if c["nv"]:
            q = np.arange(c["nv"], dtype=np.uint32)
            got = hash_lookup_gpu(plan, q)
            want = np.full(c["nv"], -1, np.int64)
            want[plan.hdv_ids.astype(np.int64)] = np.arange(plan.k)
            assert np.array_equal(got, want), c["name"]
        assert coverage_exact(g, plan) == c["exact"], c["name"]


@pytest.mark.gpu
def test_gpu_sample_hdv_errors_and_potra_step0():
    from paper_2501_06872_b200 import CsrGraph, HdvBudget, sample_hdv, transpose_gpu, transpose_potra

    rng = np.random.default_rng(5)
    nv, ne = 100_000, 2_000_000
    dst = rng.integers(0, nv, ne)
    dst[rng.random(ne) < 0.3] = 77
    g = CsrGraph.from_edge_pairs(rng.integers(0, nv, ne), dst, nv)
    with pytest.raises(ValueError):
        sample_hdv(g, 1, sample_fraction=0.0)
    with pytest.raises(ValueError):
        sample_hdv(g, -1)
    out0 = transpose_potra(g, 8, HdvBudget(cache_bytes=1 << 16, threads=8), seed=3)  # default: no step 0
    assert out0.details["k"] is None and out0.details["plan"] is None
    out = transpose_potra(g, 8, HdvBudget(cache_bytes=1 << 16, threads=8), seed=3, force_method="hlh")
    d = out.details
    assert d["method_chosen"] == "gpu" and d["k"] > 0 and d["plan"].hdv_ids[0] == 77
    assert d["sample_size"] == 1000 and 0.2 < d["coverage_estimate"] < 0.45
    ids, est, size = oracle.sample_hdv_np(g.edges, nv, d["k"], 0.01, 3, 8)
    assert np.array_equal(d["plan"].hdv_ids, ids) and d["coverage_estimate"] == est
    assert out.graph == transpose_gpu(g).graph and "step0" in out.phase_times
