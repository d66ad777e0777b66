"""GPU parity: libgt.so (through the C ABI / transpose_gpu) against the CPU
oracle and the reference's golden outputs.  Bit-exact: identical CSC offsets
(uint64) and identical neighbour arrays (uint32), lists ascending by source."""

import ctypes
import os
import sys

import numpy as np
import pytest

from conftest import ROOT, random_graph, sha

sys.path.insert(0, str(ROOT))
from oracle import oracle  # noqa: E402  (test infrastructure)

pytestmark = pytest.mark.gpu

RANK_MODES = [0, 1]  # 0 = smem-atomic ranking (default when the self-test passes), 1 = safe OR-mask


@pytest.fixture(params=RANK_MODES, ids=["atomic-rank", "safe-rank"])
def rank_mode(request):
    from paper_2501_06872_b200 import set_rank_mode

    set_rank_mode(request.param)
    yield request.param
    set_rank_mode(-1)


def _graph(nv, off, edg):
    from paper_2501_06872_b200 import CsrGraph

    return CsrGraph(nv, int(edg.shape[0]), off.astype(np.uint64), edg.astype(np.uint32))


def test_selftest_lane_order():
    from paper_2501_06872_b200 import selftest_rank_order

    assert selftest_rank_order(1 << 24) == 0


def test_golden_cases(golden_cases, rank_mode):
    from paper_2501_06872_b200 import transpose_gpu

    for name, c in golden_cases.items():
        g = _graph(c["nv"], c["off"], c["edg"])
        out = transpose_gpu(g)
        assert out.sorted and out.method == "gpu"
        assert out.graph.orientation == "CSC"
        assert out.graph.offsets.dtype == np.uint64 and out.graph.edges.dtype == np.uint32
        assert np.array_equal(out.graph.offsets, c["toff"]), name
        assert np.array_equal(out.graph.edges, c["tedg"]), name


def test_random_suite_vs_oracle(rank_mode):
    from paper_2501_06872_b200 import lists_are_sorted, transpose_gpu

    rng = np.random.default_rng(2024 + rank_mode)
    for i in range(60):
        g = random_graph(rng, max_vertices=3000, max_edges=40_000)
        toff, tedg = oracle.transpose_c(g.offsets, g.edges, g.num_vertices)
        out = transpose_gpu(g)
        assert np.array_equal(out.graph.offsets, toff), i
        assert np.array_equal(out.graph.edges, tedg), i
        assert lists_are_sorted(out.graph)


def test_involution():
    from paper_2501_06872_b200 import transpose_gpu

    rng = np.random.default_rng(7)
    for _ in range(10):
        g = random_graph(rng, max_vertices=500, max_edges=5000)
        back = transpose_gpu(transpose_gpu(g).graph).graph
        # transposing twice gives the canonical (sorted-list) form of g
        co, ce = oracle.transpose_c(*oracle.transpose_c(g.offsets, g.edges, g.num_vertices), g.num_vertices)
        assert np.array_equal(back.offsets, co) and np.array_equal(back.edges, ce)
        assert back.orientation == "CSR"


def test_c1_matches_reference_hash(golden_hashes, rank_mode):
    from paper_2501_06872_b200 import gen, transpose_gpu

    cfg = gen.CONFIGS["C1"]
    off, edg = gen.generate_np(cfg)
    out = transpose_gpu(_graph(cfg.num_vertices, off, edg))
    assert sha(out.graph.offsets, out.graph.edges) == golden_hashes["C1"]["oracle"]


def test_device_generator_matches_numpy(golden_hashes):
    import torch

    from paper_2501_06872_b200 import gen

    cfg = gen.CONFIGS["C1"]
    off_d, edg_d = gen.generate_device(cfg)
    torch.cuda.synchronize()
    off = off_d.cpu().numpy().view(np.uint64)
    edg = edg_d.cpu().numpy().view(np.uint32)
    assert sha(off, edg) == golden_hashes["C1"]["input"]
    # permuted RMAT and ER at a reduced edge count: device == numpy
    for kind_cfg, E in ((gen.GraphConfig("p", "rmat", 1 << 13, 1 << 17, scale=13, permute=True, seed=9), 1 << 17),
                        (gen.GraphConfig("q", "rmat", 1 << 12, 1 << 16, scale=12, permute=True, seed=3), 1 << 16),
                        (gen.GraphConfig("e", "er", 100_003, 1 << 18, seed=11), 1 << 18)):
        o_d, e_d = gen.generate_device(kind_cfg, num_edges=E)
        o_n, e_n = gen.generate_np(kind_cfg)
        assert np.array_equal(o_d.cpu().numpy().view(np.uint64), o_n)
        assert np.array_equal(e_d.cpu().numpy().view(np.uint32), e_n)


def test_edge_cases():
    from paper_2501_06872_b200 import CsrGraph, transpose_gpu

    # no edges, several vertex counts (test_baselines.py:151-160, test_io.py:31-37)
    for nv in (0, 1, 17, 70_000):
        g = CsrGraph(nv, 0, np.zeros(nv + 1, np.uint64), np.empty(0, np.uint32))
        out = transpose_gpu(g)
        assert np.array_equal(out.graph.offsets, np.zeros(nv + 1, np.uint64)) and out.graph.num_edges == 0
    # every edge to one vertex, large (multi-job big-bucket path)
    rng = np.random.default_rng(3)
    for nv, ne in ((50, 2_000_000), (1 << 20, 3_000_000)):
        src = np.sort(rng.integers(0, nv, ne))
        g = CsrGraph.from_edge_pairs(src, np.full(ne, nv // 3), nv)
        out = transpose_gpu(g)
        toff, tedg = oracle.transpose_c(g.offsets, g.edges, nv)
        assert np.array_equal(out.graph.offsets, toff) and np.array_equal(out.graph.edges, tedg)
    # one source with all edges (a single out-list spanning many tiles)
    g = CsrGraph.from_edge_pairs(np.full(1_000_000, 5), rng.integers(0, 1 << 18, 1_000_000), 1 << 18)
    out = transpose_gpu(g)
    toff, tedg = oracle.transpose_c(g.offsets, g.edges, g.num_vertices)
    assert np.array_equal(out.graph.offsets, toff) and np.array_equal(out.graph.edges, tedg)
    # many isolated sources between edges (long zero-degree runs)
    nv = 3_000_000
    src = rng.choice(nv, 5000, replace=False)
    g = CsrGraph.from_edge_pairs(np.repeat(src, 40), rng.integers(0, nv, 200_000), nv)
    out = transpose_gpu(g)
    toff, tedg = oracle.transpose_c(g.offsets, g.edges, nv)
    assert np.array_equal(out.graph.offsets, toff) and np.array_equal(out.graph.edges, tedg)


@pytest.mark.parametrize("nv,ne,skew", [(1 << 16, 1 << 22, 3.0), (1_000_003, 1 << 23, 1.0), (1 << 21, 1 << 24, 6.0)])
def test_medium_graphs(nv, ne, skew, rank_mode):
    from paper_2501_06872_b200 import CsrGraph, transpose_gpu

    rng = np.random.default_rng(nv ^ ne)
    src = rng.integers(0, nv, ne)
    dst = np.minimum((nv * rng.random(ne) ** skew).astype(np.int64), nv - 1)
    perm = rng.permutation(nv)
    g = CsrGraph.from_edge_pairs(src, perm[dst], nv)
    out = transpose_gpu(g)
    toff, tedg = oracle.transpose_c(g.offsets, g.edges, nv)
    assert np.array_equal(out.graph.offsets, toff)
    assert np.array_equal(out.graph.edges, tedg)
    assert out.details["big_buckets"] >= 0


def test_prefix_sum_gpu(golden_hashes):
    from paper_2501_06872_b200 import prefix_sum_gpu

    counts = np.random.default_rng(19).integers(0, 1000, size=100_000)
    assert sha(prefix_sum_gpu(counts)) == golden_hashes["prefix_sum_100k_seed19"]
    assert prefix_sum_gpu(np.array([2, 0, 3])).tolist() == [0, 2, 2, 5]  # test_baselines.py:19-21
    assert prefix_sum_gpu(np.zeros(0, np.int64)).tolist() == [0]
    big = np.random.default_rng(1).integers(0, 1 << 31, size=3_000_000)
    assert np.array_equal(prefix_sum_gpu(big).astype(np.int64), np.concatenate([[0], np.cumsum(big)]))


def test_host_entry_point_e2e():
    """gt_transpose_host: host buffers in/out through the C ABI."""
    from paper_2501_06872_b200 import _lib

    rng = np.random.default_rng(11)
    g = random_graph(rng, max_vertices=20_000, max_edges=300_000)
    toff = np.empty(g.num_vertices + 1, np.uint64)
    tedg = np.empty(g.num_edges, np.uint32)
    st = _lib.GtStats()
    rc = _lib.lib.gt_transpose_host(g.offsets.ctypes.data_as(ctypes.c_void_p), g.edges.ctypes.data_as(ctypes.c_void_p),
                                    g.num_vertices, g.num_edges, toff.ctypes.data_as(ctypes.c_void_p),
                                    tedg.ctypes.data_as(ctypes.c_void_p), 0, ctypes.byref(st))
    _lib.check(rc, "gt_transpose_host")
    o, e = oracle.transpose_c(g.offsets, g.edges, g.num_vertices)
    assert np.array_equal(toff, o) and np.array_equal(tedg, e)


def test_host_batch_entry_point():
    """gt_transpose_host_many: a batch of host graphs of different sizes (an
    empty one and a hub-heavy one included), copies overlapped with kernels;
    every result equals the oracle."""
    from paper_2501_06872_b200 import CsrGraph, transpose_gpu_many

    rng = np.random.default_rng(12)
    gs = [random_graph(rng, max_vertices=20_000, max_edges=300_000) for _ in range(3)]
    gs.append(CsrGraph(17, 0, np.zeros(18, np.uint64), np.zeros(0, np.uint32)))
    src = rng.integers(0, 50_000, 1_500_000)
    dst = np.minimum((50_000 * rng.random(1_500_000) ** 5).astype(np.int64), 49_999)
    gs.append(CsrGraph.from_edge_pairs(src, dst, 50_000))
    gs.append(gs[0])
    outs = transpose_gpu_many(gs)
    assert len(outs) == len(gs)
    for i, (g, out) in enumerate(zip(gs, outs)):
        o, e = oracle.transpose_c(g.offsets, g.edges, g.num_vertices)
        assert np.array_equal(out.graph.offsets, o) and np.array_equal(out.graph.edges, e), i
        assert out.sorted and out.method == "gpu"
    assert transpose_gpu_many([]) == []


def _host_pipeline_cases():
    from paper_2501_06872_b200 import CsrGraph

    rng = np.random.default_rng(23)
    cases = [("random", random_graph(rng, max_vertices=20_000, max_edges=300_000))]
    nv = 70_001  # not a multiple of the coarse bucket width
    src = np.sort(rng.integers(0, nv, 900_000))
    dst = np.where(rng.random(src.size) < 0.3, 4242, np.minimum((nv * rng.random(src.size) ** 4).astype(np.int64), nv - 1))
    cases.append(("hub", CsrGraph.from_edge_pairs(src, dst, nv)))
    # one source holds almost every edge: the other source chunks are empty
    src = np.concatenate([np.full(200_000, 5), rng.integers(0, 3000, 50)])
    cases.append(("star", CsrGraph.from_edge_pairs(src, rng.integers(0, 3000, src.size), 3000)))
    # destinations only in the first and last coarse buckets: empty bucket groups
    dst = np.where(rng.random(100_000) < 0.5, rng.integers(0, 50, 100_000), rng.integers(99_900, 100_000, 100_000))
    cases.append(("two-ends", CsrGraph.from_edge_pairs(rng.integers(0, 100_000, 100_000), dst, 100_000)))
    return cases


@pytest.mark.parametrize("chunks,groups", [(1, 1), (2, 3), (3, 8), (8, 2), (5, 64)])
def test_host_pipeline(chunks, groups):
    """The pipelined gt_transpose_host (source chunks run level 1 as senders
    while later chunks copy in; bucket groups copy back while later groups
    run levels 2-3), forced on small graphs through gt_config; pageable and
    pinned host buffers; every result equals the oracle."""
    import torch

    from paper_2501_06872_b200 import pipeline_config, transpose_host

    for name, g in _host_pipeline_cases():
        o, e = oracle.transpose_c(g.offsets, g.edges, g.num_vertices)
        with pipeline_config(host_chunks=chunks, host_groups=groups):
            out = transpose_host(g)
            assert np.array_equal(out.graph.offsets, o) and np.array_equal(out.graph.edges, e), name
            pin_o = torch.empty(g.num_vertices + 1, dtype=torch.int64).pin_memory()
            pin_e = torch.empty(max(g.num_edges, 1), dtype=torch.int32).pin_memory()
            to = pin_o.numpy().view(np.uint64)
            te = pin_e.numpy().view(np.uint32)[: g.num_edges]
            transpose_host(g, out=(to, te))
            assert np.array_equal(to, o) and np.array_equal(te, e), name


def test_host_pipeline_default_size():
    """A graph above the pipelined call's size threshold (2^24 edges) takes it
    by default (2 source chunks, 2 bucket groups) and equals the oracle, with
    and without stats; the serial call (host_chunks = -1) gives the same."""
    from paper_2501_06872_b200 import CsrGraph, _lib, pipeline_config, transpose_host

    rng = np.random.default_rng(29)
    nv, ne = 3_000_000, (1 << 24) + (1 << 25) + 12345
    src = rng.integers(0, nv, ne)
    dst = np.minimum((nv * rng.random(ne) ** 2).astype(np.int64), nv - 1)
    g = CsrGraph.from_edge_pairs(src, dst, nv)
    del src, dst
    o, e = oracle.transpose_c(g.offsets, g.edges, g.num_vertices)
    out = transpose_host(g)
    assert np.array_equal(out.graph.offsets, o) and np.array_equal(out.graph.edges, e)
    toff = np.empty(nv + 1, np.uint64)
    tedg = np.empty(ne, np.uint32)
    st = _lib.GtStats()
    rc = _lib.lib.gt_transpose_host(g.offsets.ctypes.data_as(ctypes.c_void_p), g.edges.ctypes.data_as(ctypes.c_void_p),
                                    nv, ne, toff.ctypes.data_as(ctypes.c_void_p), tedg.ctypes.data_as(ctypes.c_void_p),
                                    0, ctypes.byref(st))
    _lib.check(rc, "gt_transpose_host")
    assert st.n_launches > 0 and st.ms_total > 0
    assert np.array_equal(toff, o) and np.array_equal(tedg, e)
    with pipeline_config(host_chunks=-1):
        out = transpose_host(g)
    assert np.array_equal(out.graph.offsets, o) and np.array_equal(out.graph.edges, e)


def test_host_offsets_mismatch():
    """gt_transpose_host rejects offsets[V] != num_edges before any copy."""
    from paper_2501_06872_b200 import _lib

    off = np.array([0, 2, 3], np.uint64)
    edg = np.array([1, 0, 0, 1], np.uint32)
    toff = np.empty(3, np.uint64)
    tedg = np.empty(4, np.uint32)
    rc = _lib.lib.gt_transpose_host(off.ctypes.data_as(ctypes.c_void_p), edg.ctypes.data_as(ctypes.c_void_p), 2, 4,
                                    toff.ctypes.data_as(ctypes.c_void_p), tedg.ctypes.data_as(ctypes.c_void_p), 0, None)
    assert rc == -1  # GT_EINVAL


@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_shard_pipeline_single_gpu(parts):
    """The multi-GPU building blocks, run for every rank on one GPU in sequence
    (no kernel waits on another): sender partitions + receiver transposes."""
    from paper_2501_06872_b200.multi import GpuShardBackend, plan_shards, transpose_sharded_local

    rng = np.random.default_rng(parts)
    nv, ne = 200_003, 2_000_000
    src = rng.integers(0, nv, ne)
    dst = np.minimum((nv * rng.random(ne) ** 2).astype(np.int64), nv - 1)
    from paper_2501_06872_b200 import CsrGraph

    g = CsrGraph.from_edge_pairs(src, dst, nv)
    plan = plan_shards(g.offsets, parts)
    toff, tedg = transpose_sharded_local(g, plan, GpuShardBackend())
    o, e = oracle.transpose_c(g.offsets, g.edges, nv)
    assert np.array_equal(toff, o) and np.array_equal(tedg, e)


@pytest.mark.slow
@pytest.mark.parametrize("cfg_name", ["C2", "C3"])
def test_full_size_configs(cfg_name):
    """Full BASELINE sizes: generated on device, checked against the C oracle
    bit for bit, plus size-independent properties."""
    import torch

    from paper_2501_06872_b200 import gen, transpose_device

    if os.environ.get("GT_SKIP_FULL") == "1":
        pytest.skip("GT_SKIP_FULL=1")
    cfg = gen.CONFIGS[cfg_name]
    off_d, edg_d = gen.generate_device(cfg)
    t_off, t_edg, st = transpose_device(off_d, edg_d, cfg.num_vertices, want_stats=True)
    torch.cuda.synchronize()
    off = off_d.cpu().numpy().view(np.uint64)
    edg = edg_d.cpu().numpy().view(np.uint32)
    got_off = t_off.cpu().numpy().view(np.uint64)
    got_edg = t_edg.cpu().numpy().view(np.uint32)
    del off_d, edg_d, t_off, t_edg
    torch.cuda.empty_cache()
    assert got_off[-1] == cfg.num_edges
    o, e = oracle.transpose_c(off, edg, cfg.num_vertices)
    assert np.array_equal(got_off, o)
    assert np.array_equal(got_edg, e)


def _web_cfg(V, target, hubs=1 << 10, window=256, seed=11):
    from paper_2501_06872_b200 import gen

    scale = V.bit_length() - 1
    return gen.GraphConfig(f"web-v2^{scale}", "web", V, target, scale=scale, seed=seed,
                           web=gen.WebParams(hubs=hubs, window=window))


def test_web_generator_device_matches_numpy():
    from paper_2501_06872_b200 import gen

    cfg = _web_cfg(1 << 16, 1 << 20)
    s_d, d_d = gen.web_pairs_device(cfg)
    s_n, d_n = gen.web_pairs_np(cfg.num_vertices, cfg.num_edges, cfg.seed, cfg.web)
    assert np.array_equal(s_d.cpu().numpy().view(np.uint32), s_n)
    assert np.array_equal(d_d.cpu().numpy().view(np.uint32), d_n)


@pytest.mark.parametrize("V,target", [(1 << 16, 1 << 20), (1 << 26, 1 << 26)])
def test_web_graph_transpose(V, target, rank_mode):
    """Web-like graphs; |V| = 2^26 takes the 10|10|6 digit split (1024-digit
    level-2 pass) of config C4 at a small edge count."""
    from paper_2501_06872_b200 import gen, transpose_device

    cfg = _web_cfg(V, target, hubs=min(1 << 16, V >> 6), window=4096 if V > 1 << 20 else 256)
    off_d, edg_d = gen.generate_device(cfg)
    t_off, t_edg, st = transpose_device(off_d, edg_d, V, want_stats=True)
    if V == 1 << 26:
        assert list(st.bits) == [10, 10, 6]
    off = off_d.cpu().numpy().view(np.uint64)
    edg = edg_d.cpu().numpy().view(np.uint32)
    o, e = oracle.transpose_c(off, edg, V)
    assert np.array_equal(t_off.cpu().numpy().view(np.uint64), o)
    assert np.array_equal(t_edg.cpu().numpy().view(np.uint32), e)


@pytest.mark.slow
def test_full_size_c4():
    """Config C4 (web-like, |V| = 2^26, |E| ~ 2^30) generated on the device,
    transposed, and checked against the C oracle bit for bit."""
    import torch

    from paper_2501_06872_b200 import gen, transpose_device

    if os.environ.get("GT_SKIP_FULL") == "1":
        pytest.skip("GT_SKIP_FULL=1")
    cfg = gen.CONFIGS["C4"]
    off_d, edg_d = gen.generate_device(cfg)
    E = int(edg_d.numel())
    t_off, t_edg, st = transpose_device(off_d, edg_d, cfg.num_vertices, want_stats=True)
    torch.cuda.synchronize()
    off = off_d.cpu().numpy().view(np.uint64)
    edg = edg_d.cpu().numpy().view(np.uint32)
    got_off = t_off.cpu().numpy().view(np.uint64)
    got_edg = t_edg.cpu().numpy().view(np.uint32)
    del off_d, edg_d, t_off, t_edg
    torch.cuda.empty_cache()
    assert got_off[-1] == E and abs(E / (1 << 30) - 1) < 0.1
    o, e = oracle.transpose_c(off, edg, cfg.num_vertices)
    assert np.array_equal(got_off, o)
    assert np.array_equal(got_edg, e)


def test_wide_pipeline(golden_cases, rank_mode):
    """The wide v3 form (64-bit positions, R2 = source array + low-digit bytes;
    taken by graphs with E >= 2^32 or 29-bit IDs such as C5), forced on small
    graphs: goldens, random graphs, hub graphs (big-bucket path), skewed medium
    graphs, and a 2^29-vertex graph with the C5 digit split (11|10|8, 15
    source-high bits per coarse bucket)."""
    from paper_2501_06872_b200 import CsrGraph, pipeline_config, transpose_gpu

    with pipeline_config(force_wide=True):
        _wide_cases(golden_cases, rank_mode, CsrGraph, transpose_gpu)


def _wide_cases(golden_cases, rank_mode, CsrGraph, transpose_gpu):
    for name, c in golden_cases.items():
        out = transpose_gpu(_graph(c["nv"], c["off"], c["edg"]))
        assert np.array_equal(out.graph.offsets, c["toff"]), name
        assert np.array_equal(out.graph.edges, c["tedg"]), name
    rng = np.random.default_rng(515 + rank_mode)
    for i in range(30):
        g = random_graph(rng, max_vertices=3000, max_edges=40_000)
        out = transpose_gpu(g)
        toff, tedg = oracle.transpose_c(g.offsets, g.edges, g.num_vertices)
        assert np.array_equal(out.graph.offsets, toff) and np.array_equal(out.graph.edges, tedg), i
    cases = []
    for nv, ne, skew in ((1 << 16, 1 << 22, 3.0), (1 << 21, 1 << 24, 6.0), (1_000_003, 1 << 23, 1.0)):
        src = rng.integers(0, nv, ne)
        dst = np.minimum((nv * rng.random(ne) ** skew).astype(np.int64), nv - 1)
        cases.append((nv, src, rng.permutation(nv)[dst]))
    src = np.sort(rng.integers(0, 50, 2_000_000))
    cases.append((50, src, np.full(src.size, 17)))  # every edge to one vertex
    nv = 1 << 29  # C5's ID width and digit split at 2^25 edges
    src = rng.integers(0, nv, 1 << 25)
    dst = np.minimum((nv * rng.random(1 << 25) ** 2.0).astype(np.int64), nv - 1)
    cases.append((nv, src, (dst * 2654435761) % nv))  # odd multiplier: a bijection of [0, 2^29)
    for nv, s, d in cases:
        g = CsrGraph.from_edge_pairs(s, d, nv)
        out = transpose_gpu(g)
        toff, tedg = oracle.transpose_c(g.offsets, g.edges, nv)
        assert np.array_equal(out.graph.offsets, toff), nv
        assert np.array_equal(out.graph.edges, tedg), nv
        if nv == 1 << 29:
            assert tuple(out.details["digit_bits"]) == (11, 10, 8)


def test_rmat_lean_generator_matches_pairs_path():
    """gt_gen_rmat_csr + two transposes (the C5 generation path) gives the same
    CSR as the pair generator + CSR build (and as the numpy generator)."""
    from paper_2501_06872_b200 import gen

    cfg = gen.GraphConfig("rmat-s16-perm", "rmat", 1 << 16, 1 << 20, scale=16, permute=True, seed=21)
    o1, e1 = gen.generate_device(cfg, lean=True)
    o2, e2 = gen.generate_device(cfg, lean=False)
    assert np.array_equal(o1.cpu().numpy(), o2.cpu().numpy())
    assert np.array_equal(e1.cpu().numpy(), e2.cpu().numpy())
    on, en = gen.generate_np(cfg)
    assert np.array_equal(o1.cpu().numpy().view(np.uint64), on)
    assert np.array_equal(e1.cpu().numpy().view(np.uint32), en)


@pytest.mark.slow
def test_full_size_c5():
    """Config C5 (R-MAT scale 29, edge factor 16, IDs permuted: 8.6e9 edges, E >= 2^32)
    on one GPU: lean generation, transpose (wide v3 form), and the C
    oracle on the host, bit for bit."""
    import gc

    import torch

    from paper_2501_06872_b200 import gen, transpose_device

    if os.environ.get("GT_SKIP_FULL") == "1" or os.environ.get("GT_SKIP_C5") == "1":
        pytest.skip("GT_SKIP_FULL / GT_SKIP_C5")
    free, total = torch.cuda.mem_get_info()
    if total < 150 * (1 << 30):
        pytest.skip("C5 needs a 180 GB-class GPU")
    cfg = gen.CONFIGS["C5"]
    V, E = cfg.num_vertices, cfg.num_edges
    off_d, edg_d = gen.generate_device(cfg)
    t_off, t_edg, st = transpose_device(off_d, edg_d, V, want_stats=True)
    torch.cuda.synchronize()
    off = off_d.cpu().numpy().view(np.uint64)
    edg = edg_d.cpu().numpy().view(np.uint32)
    del off_d, edg_d
    got_off = t_off.cpu().numpy().view(np.uint64)
    got_edg = t_edg.cpu().numpy().view(np.uint32)
    del t_off, t_edg
    torch.cuda.empty_cache()
    assert off[-1] == E and got_off[-1] == E
    o, e = oracle.transpose_c(off, edg, V)
    del off, edg
    gc.collect()
    assert np.array_equal(got_off, o)
    assert np.array_equal(got_edg, e)


@pytest.mark.parametrize("cfg", [{}, {"split": (6, 6, 6)}, {"split": (8, 8, 2)}, {"force_wide": True}],
                         ids=["default", "split-6-6-6", "split-8-8-2", "wide"])
def test_pipeline_configs(golden_cases, cfg):
    """The explicit pipeline configuration (gt_set_config: digit split, wide
    form) stays bit-exact: goldens, random graphs and a hub-heavy graph
    (level-3 big-bucket path), against the oracle."""
    from paper_2501_06872_b200 import CsrGraph, pipeline_config, transpose_gpu

    with pipeline_config(**cfg):
        for name in sorted(golden_cases)[:20]:
            c = golden_cases[name]
            out = transpose_gpu(_graph(c["nv"], c["off"], c["edg"]))
            assert np.array_equal(out.graph.offsets, c["toff"]), name
            assert np.array_equal(out.graph.edges, c["tedg"]), name
        rng = np.random.default_rng(77)
        for i in range(6):
            g = random_graph(rng, max_vertices=50_000, max_edges=400_000)
            out = transpose_gpu(g)
            o, e = oracle.transpose_c(g.offsets, g.edges, g.num_vertices)
            assert np.array_equal(out.graph.offsets, o) and np.array_equal(out.graph.edges, e), i
        nv, ne = 1 << 18, 1 << 23
        src = np.sort(rng.integers(0, nv, ne))
        dst = np.minimum((nv * rng.random(ne) ** 6).astype(np.int64), nv - 1)
        g = CsrGraph.from_edge_pairs(src, dst, nv)
        out = transpose_gpu(g)
        o, e = oracle.transpose_c(g.offsets, g.edges, nv)
        assert np.array_equal(out.graph.offsets, o) and np.array_equal(out.graph.edges, e)
        if "split" in cfg:
            assert tuple(out.details["digit_bits"]) == cfg["split"]
        assert out.details["big_buckets"] > 0 or cfg.get("force_wide")
