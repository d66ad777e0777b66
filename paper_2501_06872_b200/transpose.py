"""Drop-in GPU transposition with the reference's operator contract.

Mirrors the reference entry points of the hot path
(``transpose_atomic(g, threads, ...)`` baselines.py:168-209 and
``transpose_potra(g, threads, ...)`` hlh.py:441-588, each followed by
``sort_neighbor_lists`` baselines.py:457-475): a ``CsrGraph`` in, a
``TransposeOutput`` out whose graph is bit-identical to
``transpose_oracle(g)`` (graph.py:136-148) — uint64 offsets, uint32 neighbour
IDs, orientation flipped, every list ascending by source — with
``sorted=True`` and no sort pass.

The work runs in libgt.so (hand-written sm_100a kernels behind a C ABI).
torch is used only for device memory and streams.  There is no CPU fallback:
missing library or device raises :class:`GpuUnavailableError`.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import GpuUnavailableError
from .graph import CsrGraph, flip_orientation

__all__ = [
    "TransposeOutput",
    "transpose_gpu",
    "transpose_gpu_many",
    "transpose_host",
    "transpose_potra",
    "transpose_atomic",
    "transpose_device",
    "prefix_sum_gpu",
    "edge_balanced_vertex_bounds",
    "selftest_rank_order",
    "set_rank_mode",
    "transpose_status",
    "set_config",
    "pipeline_config",
    "release_workspace",
]


@dataclass
class TransposeOutput:
    """Result of one transposition run plus its cost accounting
    (baselines.py:39-53, same fields)."""

    graph: object
    phase_times: dict
    aux_footprint_bytes: int
    method: str
    sorted: bool
    details: dict = field(default_factory=dict)


def _torch():
    try:
        import torch
    except ImportError as exc:  # pragma: no cover - torch is in the image
        raise GpuUnavailableError(f"torch is required for device memory: {exc}") from None
    if not torch.cuda.is_available():
        raise GpuUnavailableError("no CUDA device visible (transpose_gpu has no CPU path)")
    return torch


def _stream_handle(torch, stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def transpose_device(offsets, edges, num_vertices: int, *, t_offsets=None, t_edges=None, stream=None,
                     want_stats: bool = False):
    """Device-resident CSR -> CSC on torch CUDA tensors.

    ``offsets`` int64[V+1] (uint64 bits) and ``edges`` int32[E] (uint32 bits)
    on the same device.  Returns ``(t_offsets, t_edges, stats_or_None)``.
    Stream-ordered: without ``want_stats`` the call returns once the kernels
    are enqueued; call :func:`transpose_status` after synchronising the stream
    to learn whether an in-degree overflowed (``want_stats`` waits and raises
    :class:`CounterOverflowError` itself).
    """
    torch = _torch()
    V = int(num_vertices)
    E = int(edges.numel())
    if offsets.dtype != torch.int64 or edges.dtype != torch.int32:
        raise ValueError("offsets must be int64 (uint64 bits) and edges int32 (uint32 bits)")
    if offsets.numel() != V + 1:
        raise ValueError(f"offsets must have exactly {V + 1} entries")
    dev = offsets.device
    if t_offsets is None:
        t_offsets = torch.empty(V + 1, dtype=torch.int64, device=dev)
    if t_edges is None:
        t_edges = torch.empty(E, dtype=torch.int32, device=dev)
    st = _lib.GtStats() if want_stats else None
    with torch.cuda.device(dev):
        rc = _lib.lib.gt_transpose(
            ctypes.c_void_p(offsets.data_ptr()),
            ctypes.c_void_p(edges.data_ptr()),
            V,
            E,
            ctypes.c_void_p(t_offsets.data_ptr()),
            ctypes.c_void_p(t_edges.data_ptr()),
            None,
            0,
            _stream_handle(torch, stream),
            ctypes.byref(st) if st is not None else None,
        )
    _lib.check(rc, "gt_transpose")
    return t_offsets, t_edges, st


def _debug_check(off_d, edg_d, t_off, t_edg, nv: int, torch) -> dict:
    """The reference's debug asserts (hlh.py:400-419, 523-528, 550-558) on the
    device: write-once slots, offsets = in-degree scan, ascending lists,
    per-destination source multisets (gt_debug_check)."""
    rep = _lib.DebugReport()
    with torch.cuda.device(off_d.device):
        rc = _lib.lib.gt_debug_check(ctypes.c_void_p(off_d.data_ptr()), ctypes.c_void_p(edg_d.data_ptr()), nv,
                                     int(edg_d.numel()), ctypes.c_void_p(t_off.data_ptr()),
                                     ctypes.c_void_p(t_edg.data_ptr()), ctypes.byref(rep),
                                     _stream_handle(torch, None))
    _lib.check(rc, "gt_debug_check")
    r = {"unwritten": int(rep.unwritten), "descents": int(rep.descents), "offset_diff": int(rep.offset_diff),
         "multiset_diff": int(rep.multiset_diff)}
    if r["offset_diff"] != nv + 1:
        raise AssertionError(f"split counters do not sum to the edge count (t_offsets differ at index "
                             f"{r['offset_diff']})")
    if r["unwritten"]:
        raise AssertionError(f"a t_edges index was written more than once ({r['unwritten']} slots never written)")
    if r["multiset_diff"] != nv:
        raise AssertionError(f"the list of vertex {r['multiset_diff']} is not the multiset of its sources")
    if r["descents"]:
        raise AssertionError(f"{r['descents']} adjacent pairs out of order inside neighbour lists")
    return r


def transpose_gpu(g, devices: int = 1, *, device=None, stream=None, debug: bool = False) -> TransposeOutput:
    """Transpose a CsrGraph on the GPU; same contract as transpose_atomic +
    sort_neighbor_lists, output equal to transpose_oracle(g).

    ``devices`` plays the role of the reference's ``threads`` (must be >= 1,
    _nb.py:112-113).  The whole uint32 ID range is supported (above 2^29
    vertices the destinations are transposed in 2^29-ID slabs).  ``devices > 1`` needs an initialised torch.distributed
    process group with that many ranks (one process per GPU) and dispatches to
    :func:`paper_2501_06872_b200.multi.transpose_distributed`.  ``debug``
    runs the reference's debug asserts on the device (write-once slots,
    degree conservation, ascending lists, source multisets; ``_debug_check``)
    and raises AssertionError on a violation.
    """
    if devices < 1:
        raise ValueError(f"device count must be >= 1, got {devices}")
    if devices > 1:
        from .multi import transpose_distributed

        return transpose_distributed(g, devices=devices, device=device)
    torch = _torch()
    nv, ne = int(g.num_vertices), int(g.num_edges)
    if g.edges.dtype != np.uint32:
        raise ValueError("only 32-bit neighbour IDs (num_vertices <= 2^32) are supported")
    if g.offsets.dtype != np.uint64:
        raise ValueError("offsets must be uint64")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    t0 = time.perf_counter()
    off_d = torch.from_numpy(np.ascontiguousarray(g.offsets).view(np.int64)).to(dev, non_blocking=False)
    edg_d = torch.from_numpy(np.ascontiguousarray(g.edges).view(np.int32)).to(dev, non_blocking=False)
    t1 = time.perf_counter()
    t_edg0 = None
    if debug:  # every slot starts as the sentinel 0xFFFFFFFF (IDs are < 2^29)
        t_edg0 = torch.full((ne,), -1, dtype=torch.int32, device=dev)
    t_off, t_edg, st = transpose_device(off_d, edg_d, nv, t_edges=t_edg0, stream=stream, want_stats=True)
    dbg = _debug_check(off_d, edg_d, t_off, t_edg, nv, torch) if debug and nv > 0 else None
    t2 = time.perf_counter()
    t_offsets = t_off.cpu().numpy().view(np.uint64)
    t_edges = t_edg.cpu().numpy().view(np.uint32)
    t3 = time.perf_counter()
    out_graph = type(g)(nv, ne, t_offsets, t_edges, flip_orientation(g.orientation))
    return TransposeOutput(
        graph=out_graph,
        phase_times={
            "h2d": t1 - t0,
            "step1": st.ms_step1 / 1e3,
            "step2": st.ms_step2 / 1e3,
            "step3": st.ms_step3 / 1e3,
            "d2h": t3 - t2,
        },
        aux_footprint_bytes=int(st.workspace_bytes),
        method="gpu",
        sorted=True,
        details={
            "device_ms": st.ms_total,
            "digit_bits": tuple(st.bits),
            "rank_mode": "smem-atomic" if st.rank_mode == 0 else "or-mask",
            "big_buckets": int(st.n_big_buckets),
            "devices": 1,
            **({"debug": dbg} if dbg is not None else {}),
        },
    )


def transpose_gpu_many(graphs, device: int = 0) -> list:
    """Transpose several host graphs through ``gt_transpose_host_many``: graph
    i+1's copy-in overlaps graph i's kernels and graph i-1's copy-out (pinned
    host arrays make the copies asynchronous; pageable ones still give correct
    results).  Each result equals ``transpose_gpu(g).graph``; ``phase_times``
    holds the batch wall time per graph (the kernels overlap the copies)."""
    graphs = list(graphs)
    if not graphs:
        return []
    for g in graphs:
        if g.edges.dtype != np.uint32 or g.offsets.dtype != np.uint64:
            raise ValueError("graphs need uint64 offsets and uint32 neighbour IDs")
    _lib.load()
    k = len(graphs)
    offs = [np.ascontiguousarray(g.offsets) for g in graphs]
    edgs = [np.ascontiguousarray(g.edges) for g in graphs]
    t_offs = [np.empty(int(g.num_vertices) + 1, np.uint64) for g in graphs]
    t_edgs = [np.empty(int(g.num_edges), np.uint32) for g in graphs]
    PV, P64 = ctypes.c_void_p * k, ctypes.c_uint64 * k
    st = _lib.GtStats()
    t0 = time.perf_counter()
    rc = _lib.lib.gt_transpose_host_many(k, PV(*[a.ctypes.data for a in offs]), PV(*[a.ctypes.data for a in edgs]),
                                         P64(*[int(g.num_vertices) for g in graphs]),
                                         P64(*[int(g.num_edges) for g in graphs]),
                                         PV(*[a.ctypes.data for a in t_offs]), PV(*[a.ctypes.data for a in t_edgs]),
                                         int(device), ctypes.byref(st))
    _lib.check(rc, "gt_transpose_host_many")
    dt = (time.perf_counter() - t0) / k
    return [TransposeOutput(graph=type(g)(int(g.num_vertices), int(g.num_edges), to, te, flip_orientation(g.orientation)),
                            phase_times={"batch_per_graph": dt}, aux_footprint_bytes=int(st.workspace_bytes),
                            method="gpu", sorted=True, details={"batch": k, "devices": 1})
            for g, to, te in zip(graphs, t_offs, t_edgs)]


def transpose_host(g, device: int = 0, out=None) -> TransposeOutput:
    """Transpose one host graph through ``gt_transpose_host`` (the drop-in C-ABI
    call): large graphs take the pipelined call, whose source chunks run level
    1 while later chunks still copy in and whose bucket groups copy back while
    later groups are computed (pinned host arrays make the copies asynchronous;
    pageable ones still give correct results).  ``out`` = optional
    ``(t_offsets, t_edges)`` host arrays to fill (e.g. pinned)."""
    if g.edges.dtype != np.uint32 or g.offsets.dtype != np.uint64:
        raise ValueError("graphs need uint64 offsets and uint32 neighbour IDs")
    _lib.load()
    off = np.ascontiguousarray(g.offsets)
    edg = np.ascontiguousarray(g.edges)
    if out is None:
        out = (np.empty(int(g.num_vertices) + 1, np.uint64), np.empty(int(g.num_edges), np.uint32))
    to, te = out
    t0 = time.perf_counter()
    rc = _lib.lib.gt_transpose_host(off.ctypes.data_as(ctypes.c_void_p), edg.ctypes.data_as(ctypes.c_void_p),
                                    int(g.num_vertices), int(g.num_edges), to.ctypes.data_as(ctypes.c_void_p),
                                    te.ctypes.data_as(ctypes.c_void_p), int(device), None)
    _lib.check(rc, "gt_transpose_host")
    return TransposeOutput(graph=type(g)(int(g.num_vertices), int(g.num_edges), to, te, flip_orientation(g.orientation)),
                           phase_times={"host_call": time.perf_counter() - t0}, aux_footprint_bytes=0,
                           method="gpu", sorted=True, details={"devices": 1})


def transpose_potra(g, threads: int, budget=None, *, force_method=None, sample_fraction: float = 0.01,
                    probe_edges=None, seed: int = 0, partition_edges: int = 1 << 18,
                    debug: bool = False) -> TransposeOutput:
    """Signature of the reference's ``transpose_potra`` (hlh.py:441-452) on the GPU.

    Argument checks are the reference's (``threads >= 1``, _nb.py:112-113;
    ``force_method`` in {None, "atomic", "hlh"}, hlh.py:462-463).  The GPU
    transposition has no degree-dependent branch to choose (hubs take the
    level-3 big-bucket path by measured size; a sampled hub split at level 2
    measured slower), so step 0 is not paid on the default path:
    ``details["method_chosen"] = "gpu"`` and the step-0 fields are None.
    ``force_method="hlh"`` runs step 0 as the reference does (hlh.py:466-475:
    k from the budget by Eq. 1, ``sample_hdv`` on the GPU with the same
    ``(sample_fraction, seed, threads)`` — same HDV set and coverage estimate
    as the reference) and reports it.  ``debug=True`` runs the reference's
    debug asserts on the device (write-once slots, degree conservation,
    hlh.py:400-419, 523-528).  The output is sorted and equals
    ``transpose_oracle(g)``.
    """
    from .hdv import fit_table_budget, gpu_budget, hdv_count, sample_hdv

    if force_method not in (None, "atomic", "hlh"):
        raise ValueError(f"force_method must be 'atomic' or 'hlh', got {force_method!r}")
    if threads < 1:
        raise ValueError(f"thread count must be >= 1, got {threads}")
    t0 = time.perf_counter()
    plan = None
    if force_method == "hlh":
        if budget is None:
            budget = gpu_budget()
        k = fit_table_budget(hdv_count(budget).k, budget.load_factor, threads, budget.cache_bytes)
        plan = sample_hdv(g, k, sample_fraction=sample_fraction, seed=seed, threads=threads,
                          load_factor=budget.load_factor)
    step0 = time.perf_counter() - t0
    out = transpose_gpu(g, debug=debug)
    details = {
        "method_chosen": "gpu",
        "k": plan.k if plan else None,
        "coverage_estimate": plan.coverage_estimate if plan else None,
        "sample_size": plan.sample_size if plan else None,
        "probe": None,
        "hdv_aux_bytes": plan.aux_bytes() if plan else 0,
        "shared_aux_bytes": out.aux_footprint_bytes,
        "partitions": out.details.get("big_buckets", 0),
        "step3_imbalance": None,
        "plan": plan,
    }
    details.update(out.details)
    return TransposeOutput(graph=out.graph, phase_times={"step0": step0, **out.phase_times},
                           aux_footprint_bytes=out.aux_footprint_bytes + (plan.aux_bytes() if plan else 0),
                           method="potra-gpu", sorted=True, details=details)


def transpose_atomic(g, threads: int, partition_edges: int = 1 << 18) -> TransposeOutput:
    """Signature of the reference's ``transpose_atomic`` (baselines.py:168-170)
    on the GPU.  Unlike the reference the result is already sorted
    (``sorted=True``), so a following ``sort_neighbor_lists`` is a no-op in
    effect."""
    if threads < 1:
        raise ValueError(f"thread count must be >= 1, got {threads}")
    if partition_edges < 1:
        raise ValueError("partition_edges must be >= 1")
    return transpose_gpu(g)


def prefix_sum_gpu(counts: np.ndarray) -> np.ndarray:
    """Exclusive prefix sum with the total appended, uint64 (mirrors
    prefix_sum_parallel, baselines.py:116-127)."""
    torch = _torch()
    c = np.ascontiguousarray(counts)
    if c.size and (c.min() < 0 or c.max() >= 2**32):
        raise ValueError("counts must fit in uint32")
    c32 = torch.from_numpy(c.astype(np.uint32).view(np.int32)).cuda()
    out = torch.empty(c.size + 1, dtype=torch.int64, device=c32.device)
    rc = _lib.lib.gt_prefix_sum(ctypes.c_void_p(c32.data_ptr()), c.size, ctypes.c_void_p(out.data_ptr()),
                                _stream_handle(torch, None))
    _lib.check(rc, "gt_prefix_sum")
    return out.cpu().numpy().view(np.uint64)


def edge_balanced_vertex_bounds(offsets: np.ndarray, parts: int) -> np.ndarray:
    """Source-range sharding rule (_nb.py:118-132), computed by libgt.so."""
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    nv = off.shape[0] - 1
    parts = max(1, int(parts))
    out = np.empty(parts + 1, dtype=np.int64)
    rc = _lib.lib.gt_edge_balanced_bounds(off.ctypes.data_as(ctypes.c_void_p), nv, parts,
                                         out.ctypes.data_as(ctypes.c_void_p))
    _lib.check(rc, "gt_edge_balanced_bounds")
    return out


def selftest_rank_order(trials: int = 1 << 26) -> int:
    """Run the device self-test of lane-ordered shared-memory atomics; returns
    the number of violations (0 means the fast ranking mode is used)."""
    _torch()
    v = ctypes.c_uint64(0)
    _lib.check(_lib.lib.gt_selftest_rank_order(trials, ctypes.byref(v)), "gt_selftest_rank_order")
    return int(v.value)


def set_rank_mode(mode: int) -> None:
    """-1 auto (self-test), 0 smem-atomic ranking, 1 safe OR-mask ranking."""
    _lib.check(_lib.lib.gt_set_rank_mode(int(mode)), "gt_set_rank_mode")


def transpose_status(stream=None, device=None) -> None:
    """Raise CounterOverflowError if the last transpose enqueued on ``stream``
    (default: the current stream of ``device``) overflowed a 32-bit in-degree.
    Call after the stream has completed (gt_transpose_status)."""
    torch = _torch()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    with torch.cuda.device(dev):
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        st = ctypes.c_int(0)
        _lib.check(_lib.lib.gt_transpose_status(ctypes.c_void_p(s.cuda_stream), ctypes.byref(st)),
                   "gt_transpose_status")
        _lib.check(st.value, "gt_transpose")


def set_config(split=None, force_wide: bool = False, experiment: int = 0, host_chunks: int = 0,
               host_groups: int = 0) -> None:
    """Explicit pipeline configuration (gt_set_config): ``split`` = (a, b, c)
    digit bits (used when they cover the destination ID bits), ``force_wide``
    = the 64-bit-position form, ``experiment`` = A/B bits for measurements
    (0 = the product path), ``host_chunks`` / ``host_groups`` = the
    source chunks and bucket groups of the pipelined ``gt_transpose_host``
    (0 = by size; either set forces the pipelined call on small graphs).
    ``set_config()`` restores the defaults."""
    cfg = _lib.GtConfig()
    cfg.reserved[0] = int(experiment)
    cfg.reserved[1] = int(host_chunks)
    cfg.reserved[2] = int(host_groups)
    if split is not None:
        for i, x in enumerate(split):
            cfg.split[i] = int(x)
    cfg.force_wide = 1 if force_wide else 0
    _lib.check(_lib.lib.gt_set_config(ctypes.byref(cfg)), "gt_set_config")


class pipeline_config:
    """Context manager form of :func:`set_config` (restores the defaults)."""

    def __init__(self, split=None, force_wide: bool = False, experiment: int = 0, host_chunks: int = 0,
                 host_groups: int = 0):
        self.split, self.force_wide, self.experiment = split, force_wide, experiment
        self.host_chunks, self.host_groups = host_chunks, host_groups

    def __enter__(self):
        set_config(self.split, self.force_wide, self.experiment, self.host_chunks, self.host_groups)
        return self

    def __exit__(self, *exc):
        _lib.check(_lib.lib.gt_set_config(None), "gt_set_config")
        return False


def release_workspace() -> None:
    """Free libgt.so's cached device workspaces on the current device."""
    _torch()
    _lib.check(_lib.lib.gt_release_workspace(), "gt_release_workspace")
