"""GPU verify_output / sort_neighbor_lists against the reports the reference's
verify_output gave on the same inputs (tests/golden/make_io_golden.py), and
the argument contract of the reference-shaped entry points (CPU)."""

import json

import numpy as np
import pytest

from conftest import GOLDEN


def _variants():
    rep = json.loads((GOLDEN / "verify_cases.json").read_text())
    z = np.load(GOLDEN / "verify_cases.npz")
    return rep, z


def test_api_argument_contract():
    from paper_2501_06872_b200 import CsrGraph, transpose_atomic, transpose_gpu, transpose_potra

    g = CsrGraph(2, 1, np.array([0, 1, 1], dtype=np.uint64), np.array([1], dtype=np.uint32))
    with pytest.raises(ValueError, match="force_method"):
        transpose_potra(g, 1, force_method="bogus")
    with pytest.raises(ValueError):
        transpose_potra(g, 0)
    with pytest.raises(ValueError):
        transpose_atomic(g, 0)
    with pytest.raises(ValueError):
        transpose_gpu(g, 0)


def test_verify_mode_contract():
    from paper_2501_06872_b200 import CsrGraph, TransposeOutput, verify_output

    g = CsrGraph(2, 1, np.array([0, 1, 1], dtype=np.uint64), np.array([1], dtype=np.uint32))
    out = TransposeOutput(graph=g, phase_times={}, aux_footprint_bytes=0, method="x", sorted=True)
    with pytest.raises(ValueError, match="unknown verify mode"):
        verify_output(g, out, mode="bogus")


@pytest.mark.gpu
def test_verify_output_matches_reference_reports():
    from paper_2501_06872_b200 import CsrGraph, TransposeOutput, verify_output

    rep, z = _variants()
    nv = z["in_offsets"].size - 1
    g = CsrGraph(nv, z["in_edges"].size, z["in_offsets"], z["in_edges"], "CSR")
    n = 0
    for name, v in rep.items():
        t = CsrGraph(nv, z[f"{name}_edges"].size, z[f"{name}_offsets"], z[f"{name}_edges"], "CSC")
        out = TransposeOutput(graph=t, phase_times={}, aux_footprint_bytes=0, method="x", sorted=v["sorted"])
        for key, want in v["reports"].items():
            mode, sv = key.split("/")
            r = verify_output(g, out, mode=mode, seed=5, sample_vertices=int(sv))
            assert (r.passed, r.mismatch_vertex, r.message) == (want["passed"], want["mismatch_vertex"],
                                                                want["message"]), (name, key)
            assert r.mode == mode
            n += 1
    assert n == 20


@pytest.mark.gpu
def test_sort_neighbor_lists_canonicalises():
    from paper_2501_06872_b200 import CsrGraph, TransposeOutput, sort_neighbor_lists

    _, z = _variants()
    nv = z["in_offsets"].size - 1
    scr = CsrGraph(nv, z["scrambled_unsorted_edges"].size, z["scrambled_unsorted_offsets"],
                   z["scrambled_unsorted_edges"], "CSC")
    out = TransposeOutput(graph=scr, phase_times={"step1": 1.0}, aux_footprint_bytes=7, method="m", sorted=False)
    s = sort_neighbor_lists(out, 4)
    assert s.sorted and s.method == "m" and s.aux_footprint_bytes == 7 and "sort" in s.phase_times
    assert np.array_equal(s.graph.offsets, z["exact_offsets"]) and np.array_equal(s.graph.edges, z["exact_edges"])
    assert s.graph.edges.dtype == np.uint32 and s.graph.orientation == "CSC"


@pytest.mark.gpu
def test_sort_lists_random_multigraph(golden_cases):
    """Arbitrary list orders (not produced by a transpose) come back sorted."""
    from paper_2501_06872_b200 import CsrGraph, TransposeOutput, sort_neighbor_lists

    rng = np.random.default_rng(3)
    for name in list(golden_cases)[:10]:
        c = golden_cases[name]
        e = c["edg"].copy()
        off = c["off"].astype(np.int64)
        for v in rng.choice(c["nv"], size=min(50, c["nv"]), replace=False):
            seg = e[off[v]:off[v + 1]]
            e[off[v]:off[v + 1]] = seg[::-1]
        g = CsrGraph(c["nv"], e.size, c["off"], e)
        s = sort_neighbor_lists(TransposeOutput(graph=g, phase_times={}, aux_footprint_bytes=0, method="x",
                                                sorted=False), 1)
        want = e.copy()
        for v in range(c["nv"]):
            want[off[v]:off[v + 1]] = np.sort(want[off[v]:off[v + 1]])
        assert np.array_equal(s.graph.edges, want), name


@pytest.mark.gpu
def test_transpose_potra_shape(golden_cases):
    from paper_2501_06872_b200 import CsrGraph, transpose_atomic, transpose_potra

    c = next(iter(golden_cases.values()))
    g = CsrGraph(c["nv"], c["edg"].size, c["off"], c["edg"])
    p = transpose_potra(g, 8, force_method="hlh", seed=3)
    a = transpose_atomic(g, 8)
    for out in (p, a):
        assert out.sorted and np.array_equal(out.graph.offsets, c["toff"]) and np.array_equal(out.graph.edges, c["tedg"])
    assert p.details["method_chosen"] == "gpu" and "step0" in p.phase_times


@pytest.mark.gpu
def test_full_oracle_is_independent_of_the_pipeline(golden_cases):
    """verify_output(full-oracle) builds its expected CSC with gt_verify_transpose
    (histogram + global key sort), which equals the reference goldens, accepts
    the product's output and rejects a corrupted copy of it."""
    import torch

    from paper_2501_06872_b200 import CsrGraph, transpose_gpu, verify_output
    from paper_2501_06872_b200.verify import reference_transpose_device

    for name, c in golden_cases.items():
        off = torch.from_numpy(c["off"].astype(np.uint64).view(np.int64)).cuda()
        edg = torch.from_numpy(c["edg"].astype(np.uint32).view(np.int32)).cuda()
        o, e = reference_transpose_device(off, edg, c["nv"])
        assert np.array_equal(o.cpu().numpy().view(np.uint64), c["toff"]), name
        assert np.array_equal(e.cpu().numpy().view(np.uint32), c["tedg"]), name
    rng = np.random.default_rng(8)
    src = rng.integers(0, 3000, 100_000)
    dst = np.minimum((3000 * rng.random(100_000) ** 3).astype(np.int64), 2999)
    g = CsrGraph.from_edge_pairs(src, dst, 3000)
    out = transpose_gpu(g)
    assert verify_output(g, out, mode="full-oracle").passed
    bad = out.graph.edges.copy()
    i = int(out.graph.offsets[0])  # vertex 0 (the hub): swap two of its sources
    bad[i], bad[i + 1] = bad[i + 1], bad[i] if bad[i] != bad[i + 1] else bad[i] + 1
    t = CsrGraph(3000, g.num_edges, out.graph.offsets, bad, "CSC")
    out.graph = t
    r = verify_output(g, out, mode="full-oracle")
    assert not r.passed and r.mismatch_vertex == 0
