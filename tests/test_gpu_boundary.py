"""GPU tests of the C-ABI boundary contract (include/gt.h): stream ordering
(CUDA-graph capture + replay), per-stream workspaces (two concurrent streams),
the status word, gt_transpose_multi over NCCL at P = 1, the multi-GPU
building blocks, the overflow error, and the reference's skewed_4m golden."""

import ctypes
import os
import sys
import threading

import numpy as np
import pytest

from conftest import ROOT, sha, skewed_reference_graph

sys.path.insert(0, str(ROOT))
from oracle import oracle  # noqa: E402  (test infrastructure)

pytestmark = pytest.mark.gpu


def _rand_graph(seed, nv=300_007, ne=3_000_000, skew=3.0):
    from paper_2501_06872_b200 import CsrGraph

    rng = np.random.default_rng(seed)
    src = rng.integers(0, nv, ne)
    dst = np.minimum((nv * rng.random(ne) ** skew).astype(np.int64), nv - 1)
    return CsrGraph.from_edge_pairs(src, rng.permutation(nv)[dst], nv)


def _dev(torch, g):
    off = torch.from_numpy(g.offsets.view(np.int64)).cuda()
    edg = torch.from_numpy(g.edges.view(np.int32)).cuda()
    return off, edg


def _check(t_off, t_edg, g):
    o, e = oracle.transpose_c(g.offsets, g.edges, g.num_vertices)
    assert np.array_equal(t_off.cpu().numpy().view(np.uint64), o)
    assert np.array_equal(t_edg.cpu().numpy().view(np.uint32), e)


def test_cuda_graph_capture_and_replay():
    """gt_transpose enqueues without host synchronisation: it can be captured in
    a CUDA graph, and every replay reproduces the transpose bit for bit."""
    import torch

    from paper_2501_06872_b200 import transpose_device, transpose_status

    g = _rand_graph(5)
    off, edg = _dev(torch, g)
    t_off = torch.empty(g.num_vertices + 1, dtype=torch.int64, device="cuda")
    t_edg = torch.empty(g.num_edges, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        transpose_device(off, edg, g.num_vertices, t_offsets=t_off, t_edges=t_edg, stream=s)  # warm-up: sizes caches
    s.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        transpose_device(off, edg, g.num_vertices, t_offsets=t_off, t_edges=t_edg, stream=s)
    for _ in range(3):
        with torch.cuda.stream(s):
            t_off.fill_(-1)
            t_edg.fill_(-1)
            graph.replay()
        torch.cuda.synchronize()
        transpose_status(stream=s)
        _check(t_off, t_edg, g)


def test_two_concurrent_streams():
    """Two transposes in flight at once on different streams (from two host
    threads) use separate cached workspaces and both match the oracle."""
    import torch

    from paper_2501_06872_b200 import transpose_device, transpose_status

    gs = [_rand_graph(11), _rand_graph(12, nv=150_001, ne=4_000_000, skew=6.0)]
    devs = [_dev(torch, g) for g in gs]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [None, None]
    errs = []

    def run(i):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(streams[i]):
                for _ in range(3):
                    outs[i] = transpose_device(devs[i][0], devs[i][1], gs[i].num_vertices, stream=streams[i])[:2]
        except Exception as exc:  # pragma: no cover - reported below
            errs.append(exc)

    th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for i in range(2):
        streams[i].synchronize()
        transpose_status(stream=streams[i])
        _check(outs[i][0], outs[i][1], gs[i])


def test_transpose_multi_c_abi_one_rank():
    """gt_transpose_multi (NCCL driven from libgt.so) with one rank equals the
    oracle: level 1, the count all-gather, the NCCL send/recv of R1 and the
    receiver's levels 2-3."""
    import torch

    from paper_2501_06872_b200.multi import MultiComm

    g = _rand_graph(21, nv=1 << 20, ne=1 << 24, skew=2.0)
    off, edg = _dev(torch, g)
    comm = MultiComm(0, 1)
    try:
        t_off, t_edg, info = comm.transpose(off, edg, g.num_vertices, g.num_edges, 0, g.num_vertices)
        torch.cuda.synchronize()
        assert info.dst_begin == 0 and info.dst_end == g.num_vertices and info.global_base == 0
        assert info.num_local_edges == g.num_edges
        _check(t_off, t_edg, g)
        # capacity too small: GT_ENOMEM -> MemoryError, with the required size reported
        with pytest.raises(MemoryError):
            comm.transpose(off, edg, g.num_vertices, g.num_edges, 0, g.num_vertices, capacity=10)
    finally:
        comm.close()


@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_shard_pipeline_single_gpu(parts):
    """The multi-GPU building blocks, run for every rank on one GPU in sequence
    (no kernel waits on another): sender level 1, owner ranges balanced on the
    bucket totals, receiver levels 2-3 over the runs of every sender."""
    from paper_2501_06872_b200.multi import GpuShardBackend, plan_shards, transpose_sharded_local

    g = _rand_graph(parts, nv=200_003, ne=2_000_000, skew=2.0)
    plan = plan_shards(g.offsets, parts)
    toff, tedg = transpose_sharded_local(g, plan, GpuShardBackend())
    o, e = oracle.transpose_c(g.offsets, g.edges, g.num_vertices)
    assert np.array_equal(toff, o) and np.array_equal(tedg, e)


def test_shard_pipeline_wide_and_edge_cases():
    """Sharded pipeline on the wide form (forced), with an empty source shard
    and a hub graph (level-3 big buckets on the receivers)."""
    from paper_2501_06872_b200 import CsrGraph, pipeline_config
    from paper_2501_06872_b200.multi import GpuShardBackend, plan_shards, transpose_sharded_local

    rng = np.random.default_rng(3)
    nv = 40_000
    src = np.sort(rng.integers(20_000, nv, 1_000_000))  # sources below 20000 are empty
    dst = np.where(rng.random(src.size) < 0.3, 17, rng.integers(0, nv, src.size))
    g = CsrGraph.from_edge_pairs(src, dst, nv)
    o, e = oracle.transpose_c(g.offsets, g.edges, nv)
    for wide in (False, True):
        with pipeline_config(force_wide=wide):
            for parts in (2, 5):
                toff, tedg = transpose_sharded_local(g, plan_shards(g.offsets, parts), GpuShardBackend())
                assert np.array_equal(toff, o) and np.array_equal(tedg, e), (wide, parts)


def test_status_word_without_stats():
    """Without stats the call returns after enqueueing; gt_transpose_status
    reports GT_OK once the stream is done."""
    import torch

    from paper_2501_06872_b200 import _lib, transpose_device

    g = _rand_graph(31, nv=10_007, ne=200_000)
    off, edg = _dev(torch, g)
    t_off, t_edg, st = transpose_device(off, edg, g.num_vertices)
    assert st is None
    torch.cuda.synchronize()
    v = ctypes.c_int(7)
    assert _lib.lib.gt_transpose_status(ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), ctypes.byref(v)) == 0
    assert v.value == 0
    _check(t_off, t_edg, g)


def test_skewed_4m_reference_hash(golden_hashes):
    """The reference-made skewed_4m golden: the restated generator reproduces the
    reference's input bit for bit, and the GPU transpose hashes to the
    reference's transpose_oracle output."""
    from paper_2501_06872_b200 import transpose_gpu

    g = skewed_reference_graph()
    assert sha(g.offsets, g.edges) == golden_hashes["skewed_4m"]["input"]
    out = transpose_gpu(g)
    assert sha(out.graph.offsets, out.graph.edges) == golden_hashes["skewed_4m"]["oracle"]


@pytest.mark.slow
def test_counter_overflow_raises():
    """One vertex with 2^32 + 5 in-edges (the reference's 32-bit counters
    overflow, baselines.py:189-192): transpose_device raises
    CounterOverflowError (stats path), and the stream-ordered path reports it
    through gt_transpose_status."""
    import torch

    from paper_2501_06872_b200 import transpose_device, transpose_status
    from paper_2501_06872_b200.errors import CounterOverflowError

    if os.environ.get("GT_SKIP_FULL") == "1":
        pytest.skip("GT_SKIP_FULL=1")
    free, total = torch.cuda.mem_get_info()
    if free < 80 * (1 << 30):
        pytest.skip("needs ~70 GB of device memory")
    E = (1 << 32) + 5
    off = torch.tensor([0, E // 2, E], dtype=torch.int64, device="cuda")  # 2 sources, 2 destinations
    edg = torch.zeros(E, dtype=torch.int32, device="cuda")  # every edge to vertex 0
    with pytest.raises(CounterOverflowError):
        transpose_device(off, edg, 2, want_stats=True)
    transpose_device(off, edg, 2)
    torch.cuda.synchronize()
    with pytest.raises(CounterOverflowError):
        transpose_status()


def test_debug_mode_checks(golden_cases):
    """transpose_gpu / transpose_potra(debug=True): the reference's debug
    asserts on the device pass on real outputs and fire on corrupted ones
    (a slot never written, a wrong source, two sources out of order)."""
    import torch

    from paper_2501_06872_b200 import transpose_gpu, transpose_potra
    from paper_2501_06872_b200.transpose import _debug_check

    for name in sorted(golden_cases)[:30]:
        c = golden_cases[name]
        from paper_2501_06872_b200 import CsrGraph

        g = CsrGraph(c["nv"], int(c["edg"].size), c["off"].astype(np.uint64), c["edg"].astype(np.uint32))
        out = transpose_gpu(g, debug=True)
        if c["nv"]:
            assert out.details["debug"]["unwritten"] == 0, name
    g = _rand_graph(41, nv=20_011, ne=400_000, skew=4.0)
    out = transpose_potra(g, 4, debug=True)
    assert out.details["debug"] == {"unwritten": 0, "descents": 0, "offset_diff": g.num_vertices + 1,
                                    "multiset_diff": g.num_vertices}
    off, edg = _dev(torch, g)
    t_off = torch.from_numpy(out.graph.offsets.view(np.int64)).cuda()
    good = out.graph.edges.copy()
    hub_start = int(out.graph.offsets[int(np.argmax(np.diff(out.graph.offsets.astype(np.int64))))])
    cases = {}
    bad = good.copy(); bad[hub_start + 3] = 0xFFFFFFFF; cases["written more than once"] = bad
    bad = good.copy(); bad[hub_start + 3] ^= 1; cases["multiset"] = bad
    bad = good.copy(); bad[hub_start], bad[hub_start + 1] = good[hub_start + 1] + 1, good[hub_start]
    cases["not the multiset"] = bad
    for msg, b in cases.items():
        with pytest.raises(AssertionError, match=msg.split()[0]):
            _debug_check(off, edg, t_off, torch.from_numpy(b.view(np.int32)).cuda(), g.num_vertices, torch)
    bad = good.copy(); bad[hub_start], bad[hub_start + 1] = good[hub_start + 1], good[hub_start]
    if good[hub_start] != good[hub_start + 1]:
        with pytest.raises(AssertionError, match="out of order"):
            _debug_check(off, edg, t_off, torch.from_numpy(bad.view(np.int32)).cuda(), g.num_vertices, torch)


@pytest.mark.slow
def test_c5_one_rank_share_at_p8():
    """Config C5 (8.6e9 edges) sharded over 8 ranks: all eight senders' level 1
    on this GPU, then one rank's receiver (its bucket range, runs from every
    sender) — its CSC slice equals the corresponding slice of the C oracle's
    full transpose, bit for bit."""
    import gc

    import torch

    from paper_2501_06872_b200 import gen, release_workspace
    from paper_2501_06872_b200.multi import GpuShardBackend, plan_shards, shard_geometry, shard_owners

    if os.environ.get("GT_SKIP_FULL") == "1" or os.environ.get("GT_SKIP_C5") == "1":
        pytest.skip("GT_SKIP_FULL / GT_SKIP_C5")
    free, total = torch.cuda.mem_get_info()
    if total < 150 * (1 << 30):
        pytest.skip("C5 needs a 180 GB-class GPU")
    cfg = gen.CONFIGS["C5"]
    V, E, P, r = cfg.num_vertices, cfg.num_edges, 8, 3
    off_d, edg_d = gen.generate_device(cfg)
    release_workspace()
    torch.cuda.empty_cache()
    off_h = off_d.cpu().numpy().view(np.uint64)
    plan = plan_shards(off_h, P)
    geom = shard_geometry(V, E)
    row = int(geom.seg_hi_row)
    be = GpuShardBackend()
    sent = []
    for s in range(P):
        e0, e1 = int(plan.edge_bounds[s]), int(plan.edge_bounds[s + 1])
        sent.append(be.send(off_d, edg_d[e0:e1], V, E, e0, geom))
    counts_all = torch.stack([x[1] for x in sent]).contiguous()
    C = counts_all.cpu().numpy()
    bounds = shard_owners(C.sum(axis=0), P).astype(np.int64)
    lo, hi = int(bounds[r]), int(bounds[r + 1])
    recv = torch.cat([x[0][int(C[s, :lo].sum()):int(C[s, :hi].sum())] for s, x in enumerate(sent)])
    seg = torch.cat([x[2][lo * row:hi * row] for x in sent]).contiguous()
    del sent
    gc.collect()
    torch.cuda.empty_cache()
    base, nrec = int(C[:, :lo].sum()), int(C[:, lo:hi].sum())
    assert abs(nrec / (E / P) - 1) < 0.05  # owners balanced on the bucket totals
    t_off, t_edg, _ = be.receive(recv, seg, counts_all, P, V, E, lo, hi, nrec, base, geom)
    got_off = t_off.cpu().numpy().view(np.uint64)
    got_edg = t_edg.cpu().numpy().view(np.uint32)
    del recv, seg, t_off, t_edg
    release_workspace()
    edg_h = edg_d.cpu().numpy().view(np.uint32)
    del off_d, edg_d
    torch.cuda.empty_cache()
    o, e = oracle.transpose_c(off_h, edg_h, V)
    del edg_h
    gc.collect()
    shift = int(geom.bucket_shift)
    v_lo, v_hi = min(V, lo << shift), min(V, hi << shift)
    assert np.array_equal(got_off, o[v_lo:v_hi + 1])
    assert np.array_equal(got_edg, e[base:base + nrec])


def _slab_case(V, E, nsrc, seed):
    """CSR on the device with sources in [0, nsrc) and destinations anywhere in
    [0, V) (plus hubs in the first and the last slab); the expected CSC lists
    from numpy (lexsort by (destination, source)), the expected offsets from
    the device in-degree scan."""
    import torch

    rng = np.random.default_rng(seed)
    src = np.sort(rng.integers(0, nsrc, E))
    dst = rng.integers(0, V, E, dtype=np.int64)
    dst[rng.random(E) < 0.2] = V - 1
    dst[rng.random(E) < 0.1] = 3
    o = np.lexsort((dst, src))
    src, dst = src[o], dst[o]  # CSR order: by source, lists ascending
    deg = np.bincount(src, minlength=nsrc)
    off_small = np.zeros(nsrc + 1, np.int64)
    np.cumsum(deg, out=off_small[1:])
    off = torch.full((V + 1,), E, dtype=torch.int64, device="cuda")
    off[: nsrc + 1] = torch.from_numpy(off_small).cuda()
    edg = torch.from_numpy(dst.astype(np.uint32).view(np.int32)).cuda()
    order = np.lexsort((src, dst))
    return off, edg, src[order].astype(np.uint32)


@pytest.mark.parametrize("V", [(1 << 29) + 1000, (1 << 30) + 7])
def test_slab_mode_beyond_29_bits(V):
    """num_vertices > 2^29 (the reference's uint32 contract goes to 2^32): slab
    mode — per 2^29-ID destination slab a filtered level 1 over the whole edge
    stream, then levels 2-3 — gives transpose_oracle's CSC."""
    import torch

    from paper_2501_06872_b200 import _lib, transpose_device

    E = 1 << 21
    off, edg, want_edges = _slab_case(V, E, 5000, V & 0xffff)
    t_off, t_edg, st = transpose_device(off, edg, V, want_stats=True)
    assert np.array_equal(t_edg.cpu().numpy().view(np.uint32), want_edges)
    exp = torch.empty(V + 1, dtype=torch.int64, device="cuda")
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(_lib.lib.gt_in_degree_offsets(ctypes.c_void_p(edg.data_ptr()), E, V, ctypes.c_void_p(exp.data_ptr()), s),
               "gt_in_degree_offsets")
    first = ctypes.c_uint64(0)
    _lib.check(_lib.lib.gt_first_diff_u64(ctypes.c_void_p(exp.data_ptr()), ctypes.c_void_p(t_off.data_ptr()), V + 1,
                                          ctypes.byref(first), s), "gt_first_diff_u64")
    assert first.value == V + 1


@pytest.mark.slow
def test_slab_mode_full_uint32_range():
    """num_vertices = 2^32 - 3 (eight slabs, the full uint32 ID range): lists
    against numpy, offsets against the device in-degree scan."""
    import gc

    import torch

    from paper_2501_06872_b200 import _lib, release_workspace, transpose_device

    free, total = torch.cuda.mem_get_info()
    if free < 120 * (1 << 30):
        pytest.skip("needs ~110 GB of device memory")
    V, E = (1 << 32) - 3, 1 << 22
    off, edg, want_edges = _slab_case(V, E, 70_000, 9)
    t_off, t_edg, _ = transpose_device(off, edg, V, want_stats=True)
    assert np.array_equal(t_edg.cpu().numpy().view(np.uint32), want_edges)
    del off, t_edg
    gc.collect()
    release_workspace()
    torch.cuda.empty_cache()
    exp = torch.empty(V + 1, dtype=torch.int64, device="cuda")
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(_lib.lib.gt_in_degree_offsets(ctypes.c_void_p(edg.data_ptr()), E, V, ctypes.c_void_p(exp.data_ptr()), s),
               "gt_in_degree_offsets")
    first = ctypes.c_uint64(0)
    _lib.check(_lib.lib.gt_first_diff_u64(ctypes.c_void_p(exp.data_ptr()), ctypes.c_void_p(t_off.data_ptr()), V + 1,
                                          ctypes.byref(first), s), "gt_first_diff_u64")
    assert first.value == V + 1


def test_caller_workspace():
    """A caller-owned workspace of exactly gt_workspace_size bytes gives the same
    CSC; one byte less is GT_ENOMEM (MemoryError) before any kernel runs."""
    import torch

    from paper_2501_06872_b200 import _lib

    g = _rand_graph(51, nv=70_001, ne=1_500_000, skew=4.0)
    off, edg = _dev(torch, g)
    need = ctypes.c_uint64(0)
    _lib.check(_lib.lib.gt_workspace_size(g.num_vertices, g.num_edges, ctypes.byref(need)), "gt_workspace_size")
    ws = torch.empty(int(need.value), dtype=torch.uint8, device="cuda")
    t_off = torch.empty(g.num_vertices + 1, dtype=torch.int64, device="cuda")
    t_edg = torch.empty(g.num_edges, dtype=torch.int32, device="cuda")
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    args = [ctypes.c_void_p(off.data_ptr()), ctypes.c_void_p(edg.data_ptr()), g.num_vertices, g.num_edges,
            ctypes.c_void_p(t_off.data_ptr()), ctypes.c_void_p(t_edg.data_ptr()), ctypes.c_void_p(ws.data_ptr())]
    assert _lib.lib.gt_transpose(*args, int(need.value), s, None) == 0
    torch.cuda.synchronize()
    _check(t_off, t_edg, g)
    assert _lib.lib.gt_transpose(*args, int(need.value) - 1, s, None) == _lib.GT_ENOMEM
