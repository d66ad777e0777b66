"""Multi-GPU transposition: one process per GPU, NCCL over NVLink for the
exchange, libgt.so for every local pass.

Partitioning:
  1. Source sharding by edge count: rank r owns sources
     [src_bounds[r], src_bounds[r+1]) with src_bounds =
     edge_balanced_vertex_bounds(offsets, P) (_nb.py:118-132), i.e. a
     contiguous slice of the CSR edge stream.
  2. Sender (gt_shard_send): level 1 of the single-GPU pipeline on the slice:
     R1 = 4-byte records grouped by coarse destination bucket (bucket =
     destination >> bucket_shift), each group in CSR order, the per-bucket
     counts, and the source-high boundary rows that decode R1's sources.
  3. Counts: all_gather of the per-bucket counts -> P x D1 matrix, the one
     host read of the step.  Destination owners take contiguous bucket ranges
     balanced on the global bucket totals (gt_shard_owners) — this is the
     histogram reduce-scatter of the north_star at bucket granularity: each
     owner learns exactly the counts of its own destination range.
  4. Exchange: all_to_all of R1 (4 bytes per edge) and of the boundary rows;
     the receive buffer is ordered by sender rank = ascending source ranges,
     the order the stable transpose needs (the model is the reference's
     _mt_merge_round, baselines.py:346-375, which merges per-worker runs in
     worker order).
  5. Receiver (gt_shard_receive): levels 2-3 over the received runs (one per
     sender and bucket): the CSC slice of its destination range, offsets
     rebased to the slice's global position.
Each rank ends with its CSC slice: offsets for [dst_lo, dst_hi] and the
neighbour IDs of those lists.  The same step exists as one C-ABI call,
gt_transpose_multi (gt_multi.cu), with NCCL driven from C++.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .graph import flip_orientation

__all__ = [
    "ShardPlan",
    "plan_shards",
    "shard_geometry",
    "shard_owners",
    "GpuShardBackend",
    "exchange",
    "transpose_sharded_local",
    "transpose_distributed",
    "distributed_step",
    "MultiComm",
    "memory_plan",
]


@dataclass
class ShardPlan:
    parts: int
    src_bounds: np.ndarray  # int64[P+1] vertex bounds of source shards
    edge_bounds: np.ndarray  # int64[P+1] edge index bounds of source shards


def plan_shards(offsets: np.ndarray, parts: int) -> ShardPlan:
    from .transpose import edge_balanced_vertex_bounds

    offsets = np.asarray(offsets, dtype=np.uint64)
    if parts < 1:
        raise ValueError(f"parts must be >= 1, got {parts}")
    sb = edge_balanced_vertex_bounds(offsets, parts)
    eb = offsets[sb].astype(np.int64)
    return ShardPlan(parts, sb, eb)


def shard_geometry(num_vertices: int, num_edges: int) -> _lib.ShardGeom:
    """Bucket geometry every rank plans with (gt_shard_geometry; host only)."""
    g = _lib.ShardGeom()
    _lib.check(_lib.lib.gt_shard_geometry(int(num_vertices), int(num_edges), ctypes.byref(g)), "gt_shard_geometry")
    return g


def shard_owners(bucket_totals: np.ndarray, parts: int) -> np.ndarray:
    """Owners' bucket ranges (gt_shard_owners): uint32[parts + 1]."""
    t = np.ascontiguousarray(bucket_totals, dtype=np.uint64)
    out = np.empty(parts + 1, dtype=np.uint32)
    _lib.check(_lib.lib.gt_shard_owners(t.ctypes.data_as(ctypes.c_void_p), t.size, int(parts),
                                        out.ctypes.data_as(ctypes.c_void_p)), "gt_shard_owners")
    return out


class GpuShardBackend:
    """libgt.so kernels on torch CUDA tensors (the product path)."""

    rec_words = 1  # R1: one 32-bit word per edge

    def __init__(self, device=None):
        import torch

        if not torch.cuda.is_available():
            from .errors import GpuUnavailableError

            raise GpuUnavailableError("no CUDA device visible")
        self.torch = torch
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())

    def _stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def to_device_offsets(self, offsets: np.ndarray):
        return self.torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.uint64).view(np.int64)).to(self.device)

    def to_device_edges(self, edges: np.ndarray):
        return self.torch.from_numpy(np.ascontiguousarray(edges, dtype=np.uint32).view(np.int32)).to(self.device)

    def send(self, offsets_d, edges_slice_d, num_vertices: int, num_edges: int, e_begin: int, geom):
        """-> (r1 int32[e], bucket counts int64[D1] device, seg_hi rows int64[D1 * row] device)."""
        torch = self.torch
        n = int(edges_slice_d.numel())
        D1, row = int(geom.num_buckets), int(geom.seg_hi_row)
        r1 = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        cnt = torch.empty(D1, dtype=torch.int64, device=self.device)
        seg = torch.empty(D1 * row, dtype=torch.int64, device=self.device)
        with torch.cuda.device(self.device):
            rc = _lib.lib.gt_shard_send(ctypes.c_void_p(offsets_d.data_ptr()),
                                        ctypes.c_void_p(edges_slice_d.data_ptr()) if n else None, num_vertices,
                                        num_edges, e_begin, n, ctypes.c_void_p(r1.data_ptr()),
                                        ctypes.c_void_p(cnt.data_ptr()), ctypes.c_void_p(seg.data_ptr()),
                                        self._stream())
        _lib.check(rc, "gt_shard_send")
        return r1[:n], cnt, seg

    def receive(self, r1_recv, seg_recv, counts_all, parts: int, num_vertices: int, num_edges: int, lo: int, hi: int,
                num_records: int, global_base: int, geom, want_stats=False, check_status=True):
        """-> (t_offsets int64[n_local+1] with global positions, t_edges int32[R], stats)."""
        torch = self.torch
        shift = int(geom.bucket_shift)
        v_lo, v_hi = min(num_vertices, lo << shift), min(num_vertices, hi << shift)
        t_off = torch.empty(v_hi - v_lo + 1, dtype=torch.int64, device=self.device)
        t_edg = torch.empty(max(num_records, 1), dtype=torch.int32, device=self.device)
        st = _lib.GtStats() if want_stats else None
        with torch.cuda.device(self.device):
            rc = _lib.lib.gt_shard_receive(
                ctypes.c_void_p(r1_recv.data_ptr()) if num_records else None,
                ctypes.c_void_p(seg_recv.data_ptr()) if seg_recv.numel() else None,
                ctypes.c_void_p(counts_all.data_ptr()), parts, num_vertices, num_edges, lo, hi, num_records,
                global_base, ctypes.c_void_p(t_off.data_ptr()), ctypes.c_void_p(t_edg.data_ptr()), self._stream(),
                ctypes.byref(st) if st is not None else None)
        _lib.check(rc, "gt_shard_receive")
        if st is None and check_status:  # (callers that defer it call transpose_status after their sync)
            from .transpose import transpose_status

            torch.cuda.current_stream(self.device).synchronize()
            transpose_status(device=self.device)
        return t_off, t_edg[:num_records], st


def _owner_split(C: np.ndarray, bounds: np.ndarray, rank: int):
    """Send counts of `rank` to every owner and receive counts from every sender
    (records), from the P x D1 count matrix C and the owners' bucket bounds."""
    P = C.shape[0]
    send = np.array([int(C[rank, bounds[q]:bounds[q + 1]].sum()) for q in range(P)], dtype=np.int64)
    recv = np.array([int(C[s, bounds[rank]:bounds[rank + 1]].sum()) for s in range(P)], dtype=np.int64)
    return send, recv


def _all_to_all(out, inp, out_splits, in_splits, group=None):
    """NCCL all_to_all_single; with gloo (CPU tests) point-to-point send/recv."""
    import torch.distributed as dist

    P = dist.get_world_size(group)
    r = dist.get_rank(group)
    if dist.get_backend(group) == "nccl":
        dist.all_to_all_single(out, inp, output_split_sizes=[int(x) for x in out_splits],
                               input_split_sizes=[int(x) for x in in_splits], group=group)
        return
    so = np.concatenate([[0], np.cumsum(in_splits)])
    ro = np.concatenate([[0], np.cumsum(out_splits)])
    ops = []
    for q in range(P):
        if q == r:
            out[ro[r]:ro[r + 1]] = inp[so[r]:so[r + 1]]
            continue
        if in_splits[q]:
            ops.append(dist.P2POp(dist.isend, inp[so[q]:so[q + 1]].contiguous(), q, group))
        if out_splits[q]:
            ops.append(dist.P2POp(dist.irecv, out[ro[q]:ro[q + 1]], q, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def exchange(r1, seg, counts, geom, rec_words: int = 1, group=None):
    """All-gather of the bucket counts, owner ranges, all-to-all of R1 and of the
    boundary rows.  Returns (r1_recv, seg_recv, counts_all device, C host,
    bounds, phase seconds)."""
    import torch
    import torch.distributed as dist

    P = dist.get_world_size(group)
    r = dist.get_rank(group)
    D1, row = int(geom.num_buckets), int(geom.seg_hi_row)
    allc = [torch.empty_like(counts) for _ in range(P)]
    dist.all_gather(allc, counts, group=group)
    counts_all = torch.stack(allc).contiguous()
    C = counts_all.cpu().numpy()  # the step's one host read: sizes of the sends
    bounds = shard_owners(C.sum(axis=0), P).astype(np.int64)
    if P == 1:  # one rank owns every bucket: its R1 and rows are already where the receiver reads them
        return r1, seg, counts_all, C, bounds
    send, recv = _owner_split(C, bounds, r)
    r1_recv = torch.empty(int(recv.sum()) * rec_words, dtype=r1.dtype, device=r1.device)
    _all_to_all(r1_recv, r1, recv * rec_words, send * rec_words, group)
    nloc = int(bounds[r + 1] - bounds[r])
    seg_recv = torch.empty(P * nloc * row, dtype=seg.dtype, device=seg.device)
    seg_send = [(int(bounds[q + 1] - bounds[q])) * row for q in range(P)]
    # every owner's rows are the contiguous bucket range of this sender's table
    _all_to_all(seg_recv, seg, [nloc * row] * P, seg_send, group)
    return r1_recv, seg_recv, counts_all, C, bounds


def distributed_step(offsets_d, edges_slice_d, num_vertices: int, num_edges: int, plan: ShardPlan, rank: int,
                     backend, group=None, geom=None, timings: dict | None = None, check_status: bool = True):
    """One rank's sharded transpose on device-resident inputs (the timed step of
    bench.py at N > 1).  Returns (t_offsets slice, t_edges slice, global base,
    (dst_lo, dst_hi))."""
    P = plan.parts
    geom = geom or shard_geometry(num_vertices, num_edges)
    ev = None
    if timings is not None and hasattr(backend, "torch") and backend.torch.cuda.is_available():
        ev = [backend.torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t0 = time.perf_counter()
    if ev:
        ev[0].record()
    r1, cnt, seg = backend.send(offsets_d, edges_slice_d, num_vertices, num_edges, int(plan.edge_bounds[rank]), geom)
    if ev:
        ev[1].record()
    t1 = time.perf_counter()
    r1_recv, seg_recv, counts_all, C, bounds = exchange(r1, seg, cnt, geom, backend.rec_words, group)
    if ev:
        ev[2].record()
    t2 = time.perf_counter()
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    base = int(C[:, :lo].sum())
    nrec = int(C[:, lo:hi].sum())
    t_off, t_edg, st = backend.receive(r1_recv, seg_recv, counts_all, P, num_vertices, num_edges, lo, hi, nrec, base,
                                       geom, want_stats=timings is not None and ev is not None,
                                       check_status=check_status)
    if ev:
        ev[3].record()
    t3 = time.perf_counter()
    if timings is not None:
        if ev:  # device time of each phase (CUDA events on the launching stream)
            ev[3].synchronize()
            timings.update(send_ms=ev[0].elapsed_time(ev[1]), exchange_ms=ev[1].elapsed_time(ev[2]),
                           receive_ms=ev[2].elapsed_time(ev[3]),
                           receive_launches=int(st.n_launches) if st is not None else None,
                           records_received=nrec, buckets=(lo, hi))
        else:
            timings.update(send_ms=(t1 - t0) * 1e3, exchange_ms=(t2 - t1) * 1e3, receive_ms=(t3 - t2) * 1e3)
    shift = int(geom.bucket_shift)
    return t_off, t_edg, base, (min(num_vertices, lo << shift), min(num_vertices, hi << shift))


def transpose_sharded_local(g, plan: ShardPlan, backend):
    """Run every rank's sender and receiver steps in one process, in sequence
    (checks the sharded pipeline on a single GPU).  Returns the full
    (t_offsets uint64, t_edges uint32) on the host."""
    torch = backend.torch
    P = plan.parts
    nv, ne = int(g.num_vertices), int(g.num_edges)
    geom = shard_geometry(nv, ne)
    D1, row = int(geom.num_buckets), int(geom.seg_hi_row)
    off_d = backend.to_device_offsets(g.offsets)
    sent = []
    for r in range(P):
        e0, e1 = int(plan.edge_bounds[r]), int(plan.edge_bounds[r + 1])
        edges_d = backend.to_device_edges(g.edges[e0:e1])
        sent.append(backend.send(off_d, edges_d, nv, ne, e0, geom))
    counts_all = torch.stack([s[1] for s in sent]).contiguous()
    C = counts_all.cpu().numpy()
    bounds = shard_owners(C.sum(axis=0), P).astype(np.int64)
    t_offsets = np.zeros(nv + 1, dtype=np.uint64)
    t_edges = np.empty(ne, dtype=np.uint32)
    shift = int(geom.bucket_shift)
    w = backend.rec_words
    for q in range(P):
        lo, hi = int(bounds[q]), int(bounds[q + 1])
        pieces, segs = [], []
        for r in range(P):
            a, b = int(C[r, :lo].sum()), int(C[r, :hi].sum())
            pieces.append(sent[r][0][a * w:b * w])
            segs.append(sent[r][2][lo * row:hi * row])
        recv = torch.cat(pieces) if pieces else None
        seg_recv = torch.cat(segs).contiguous()
        base = int(C[:, :lo].sum())
        nrec = int(C[:, lo:hi].sum())
        t_off, t_edg, _ = backend.receive(recv, seg_recv, counts_all, P, nv, ne, lo, hi, nrec, base, geom)
        v_lo, v_hi = min(nv, lo << shift), min(nv, hi << shift)
        t_offsets[v_lo:v_hi + 1] = t_off.cpu().numpy().view(np.uint64)
        t_edges[base:base + nrec] = t_edg.cpu().numpy().view(np.uint32)
    return t_offsets, t_edges


def transpose_distributed(g, devices: int, device=None, backend=None, group=None, gather: bool = True):
    """Collective: every rank calls with the same host CsrGraph ``g``.  Rank 0
    receives the full transposed graph (a TransposeOutput) when ``gather``;
    other ranks receive their slice in ``details``."""
    import torch.distributed as dist

    from .transpose import TransposeOutput

    if not dist.is_available() or not dist.is_initialized():
        raise ValueError("devices > 1 requires an initialised torch.distributed process group")
    P = dist.get_world_size(group)
    if P != devices:
        raise ValueError(f"devices={devices} but the process group has {P} ranks")
    r = dist.get_rank(group)
    backend = backend or GpuShardBackend(device)
    plan = plan_shards(g.offsets, P)
    nv, ne = int(g.num_vertices), int(g.num_edges)
    off_d = backend.to_device_offsets(g.offsets)
    e0, e1 = int(plan.edge_bounds[r]), int(plan.edge_bounds[r + 1])
    edg_d = backend.to_device_edges(g.edges[e0:e1])
    t_off, t_edg, base, (lo_v, hi_v) = distributed_step(off_d, edg_d, nv, ne, plan, r, backend, group)
    details = {"rank": r, "devices": P, "dst_range": (lo_v, hi_v), "global_base": base}
    if not gather:
        return TransposeOutput(graph=None, phase_times={}, aux_footprint_bytes=0, method="gpu-sharded", sorted=True,
                               details={**details, "t_offsets": t_off, "t_edges": t_edg})
    # gather slices on rank 0 (host), for the drop-in full-graph result
    objs = [None] * P
    dist.all_gather_object(objs, (r, lo_v, hi_v, t_off.cpu().numpy(), t_edg.cpu().numpy()), group=group)
    if r != 0:
        return TransposeOutput(graph=None, phase_times={}, aux_footprint_bytes=0, method="gpu-sharded", sorted=True,
                               details=details)
    t_offsets = np.zeros(nv + 1, dtype=np.uint64)
    pieces = []
    for rr, lo, hi, o, e in sorted(objs, key=lambda t: t[0]):
        t_offsets[lo:hi + 1] = o.view(np.uint64)
        pieces.append(e.view(np.uint32))
    t_edges = np.concatenate(pieces) if pieces else np.empty(0, np.uint32)
    graph = type(g)(nv, ne, t_offsets, t_edges, flip_orientation(g.orientation))
    return TransposeOutput(graph=graph, phase_times={}, aux_footprint_bytes=0, method="gpu-sharded", sorted=True,
                           details=details)


class MultiComm:
    """A libgt NCCL communicator (gt_multi_comm_init) for gt_transpose_multi.
    Rank 0 draws the id; ``broadcast`` ships it to the other ranks (e.g.
    torch.distributed.broadcast_object_list)."""

    def __init__(self, rank: int, nranks: int, id_bytes: bytes | None = None, broadcast=None):
        buf = ctypes.create_string_buffer(128)
        if rank == 0 and id_bytes is None:
            _lib.check(_lib.lib.gt_multi_unique_id(buf), "gt_multi_unique_id")
            id_bytes = buf.raw
        if broadcast is not None:
            id_bytes = broadcast(id_bytes)
        if id_bytes is None or len(id_bytes) != 128:
            raise ValueError("a 128-byte NCCL unique id is required")
        self.rank, self.nranks = rank, nranks
        self.comm = ctypes.c_void_p()
        _lib.check(_lib.lib.gt_multi_comm_init(ctypes.create_string_buffer(id_bytes, 128), rank, nranks,
                                               ctypes.byref(self.comm)), "gt_multi_comm_init")

    def transpose(self, offsets_d, edges_slice_d, num_vertices: int, num_edges: int, src_begin: int, src_end: int,
                  capacity: int | None = None, stream=None):
        """One rank's gt_transpose_multi step -> (t_offsets slice, t_edges slice, info)."""
        import torch

        dev = offsets_d.device
        info = _lib.MultiInfo()
        cap = int(capacity) if capacity is not None else int(num_edges)
        t_off = torch.empty(int(num_vertices) + 1, dtype=torch.int64, device=dev)
        t_edg = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        with torch.cuda.device(dev):
            rc = _lib.lib.gt_transpose_multi(self.comm, self.rank, self.nranks, ctypes.c_void_p(offsets_d.data_ptr()),
                                             ctypes.c_void_p(edges_slice_d.data_ptr()) if edges_slice_d.numel() else None,
                                             int(num_vertices), int(num_edges), int(src_begin), int(src_end),
                                             ctypes.c_void_p(t_off.data_ptr()), ctypes.c_void_p(t_edg.data_ptr()), cap,
                                             ctypes.byref(info), ctypes.c_void_p(s.cuda_stream))
        _lib.check(rc, "gt_transpose_multi")
        nloc = int(info.dst_end - info.dst_begin)
        return t_off[:nloc + 1], t_edg[:int(info.num_local_edges)], info

    def close(self):
        if self.comm:
            _lib.lib.gt_multi_comm_destroy(self.comm)
            self.comm = ctypes.c_void_p()


def memory_plan(num_vertices: int, num_edges: int, parts: int, imbalance: float = 1.02) -> dict:
    """Per-rank device bytes of one sharded step (balanced shards; the receive
    side scaled by ``imbalance``): inputs (full offsets + the edge slice), the
    sender's R1 and library workspace, the exchange buffers, the receiver's
    workspace, and its CSC slice (torch-allocated buffers of multi.py included)."""
    V, E, P = int(num_vertices), int(num_edges), int(parts)
    g = shard_geometry(V, E)
    e_rank = -(-E // P)
    rec = int(e_rank * imbalance)
    nloc = -(-int(g.num_buckets) // P)
    sb, rb = ctypes.c_uint64(0), ctypes.c_uint64(0)
    _lib.check(_lib.lib.gt_shard_workspace_size(V, E, e_rank, nloc, P, rec, ctypes.byref(sb), ctypes.byref(rb)),
               "gt_shard_workspace_size")
    row = int(g.seg_hi_row) * 8
    plan = {
        "inputs (offsets + edge slice)": (V + 1) * 8 + e_rank * 4,
        "sender R1": e_rank * 4,
        "sender workspace + boundary rows": int(sb.value) + int(g.num_buckets) * row,
        "receive buffer (R1 runs + rows)": rec * 4 + P * nloc * row,
        "receiver workspace (R2 + tables)": int(rb.value),
        "CSC slice (offsets + edges)": (-(-V // P) + 1) * 8 + rec * 4,
    }
    plan["total"] = sum(plan.values())
    return plan
