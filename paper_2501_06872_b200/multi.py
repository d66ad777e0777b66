"""Multi-GPU transposition: one process per GPU, NCCL over NVLink for the
exchange, libgt.so for every local pass.

Partitioning:
  1. Source sharding by edge count: rank r owns sources
     [src_bounds[r], src_bounds[r+1]) with src_bounds =
     edge_balanced_vertex_bounds(offsets, P) (_nb.py:118-132), i.e. a
     contiguous slice of the CSR edge stream.
  2. Destination ownership: P contiguous vertex ranges dst_bounds.
  3. Sender: a stable partition of its slice by destination owner
     (gt_shard_partition, the level-1 kernel with an owner digit) -> records
     (src, dst) grouped by owner, each group in CSR order.
  4. Counts: all_gather of the P per-owner counts -> P x P matrix; receiver
     bases and the global CSC offset of every slice follow from it.  (The
     V-sized histogram reduce-scatter sketched in BASELINE/SURVEY is not
     needed: the records carry their destinations, so each receiver derives the
     in-degrees of its own range locally and only P*P counts cross NVLink.)
  5. Exchange: NCCL all_to_all_single of the records; the output is ordered by
     sender rank = ascending source ranges, so concatenation preserves the
     stable (source-ascending) order.
  6. Receiver: gt_shard_transpose — the full single-GPU pipeline over the
     received record stream for its destination range, offsets rebased to the
     global position of the slice.
Each rank ends with its CSC slice: offsets for [dst_lo, dst_hi] and the
neighbour IDs of those lists.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .graph import flip_orientation

__all__ = [
    "ShardPlan",
    "plan_shards",
    "GpuShardBackend",
    "exchange_records",
    "transpose_sharded_local",
    "transpose_distributed",
    "distributed_step",
]


@dataclass
class ShardPlan:
    parts: int
    src_bounds: np.ndarray  # int64[P+1] vertex bounds of source shards
    dst_bounds: np.ndarray  # int64[P+1] vertex bounds of destination owners
    edge_bounds: np.ndarray  # int64[P+1] edge index bounds of source shards


def plan_shards(offsets: np.ndarray, parts: int, dst_bounds=None) -> ShardPlan:
    from .transpose import edge_balanced_vertex_bounds

    offsets = np.asarray(offsets, dtype=np.uint64)
    nv = offsets.shape[0] - 1
    if parts < 1:
        raise ValueError(f"parts must be >= 1, got {parts}")
    sb = edge_balanced_vertex_bounds(offsets, parts)
    if dst_bounds is None:
        dst_bounds = (np.arange(parts + 1, dtype=np.int64) * nv) // parts
    db = np.asarray(dst_bounds, dtype=np.int64)
    if db.shape != (parts + 1,) or db[0] != 0 or db[-1] != nv or np.any(np.diff(db) < 0):
        raise ValueError("dst_bounds must be monotone with dst_bounds[0]=0, dst_bounds[-1]=num_vertices")
    eb = offsets[sb].astype(np.int64)
    return ShardPlan(parts, sb, db, eb)


class GpuShardBackend:
    """libgt.so kernels on torch CUDA tensors (the product path)."""

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

    def partition(self, offsets_d, edges_slice_d, num_vertices: int, src_lo: int, src_hi: int, dst_bounds):
        """-> (records int32[n, 2] grouped by owner, counts int64[P] numpy)."""
        torch = self.torch
        P = len(dst_bounds) - 1
        n = int(edges_slice_d.numel())
        records = torch.empty((max(n, 1), 2), dtype=torch.int32, device=self.device)
        counts = np.zeros(P, dtype=np.uint64)
        db = np.ascontiguousarray(dst_bounds, dtype=np.uint64)
        with torch.cuda.device(self.device):
            rc = _lib.lib.gt_shard_partition(
                ctypes.c_void_p(offsets_d.data_ptr()), ctypes.c_void_p(edges_slice_d.data_ptr()), num_vertices,
                src_lo, src_hi, db.ctypes.data_as(ctypes.c_void_p), P, ctypes.c_void_p(records.data_ptr()),
                counts.ctypes.data_as(ctypes.c_void_p), self._stream())
        _lib.check(rc, "gt_shard_partition")
        return records[:n], counts.astype(np.int64)

    def transpose_received(self, records, dst_lo: int, dst_hi: int, global_base: int, want_stats=False,
                           src_num_vertices: int = 1 << 32):
        """-> (t_offsets int64[n_local+1] with global positions, t_edges int32[R], stats)."""
        torch = self.torch
        R = int(records.shape[0])
        nloc = dst_hi - dst_lo
        t_off = torch.empty(nloc + 1, dtype=torch.int64, device=self.device)
        t_edg = torch.empty(max(R, 1), dtype=torch.int32, device=self.device)
        st = _lib.GtStats() if want_stats else None
        with torch.cuda.device(self.device):
            rc = _lib.lib.gt_shard_transpose(
                ctypes.c_void_p(records.data_ptr()) if R else None, R, src_num_vertices, dst_lo, dst_hi, global_base,
                ctypes.c_void_p(t_off.data_ptr()), ctypes.c_void_p(t_edg.data_ptr()), self._stream(),
                ctypes.byref(st) if st is not None else None)
        _lib.check(rc, "gt_shard_transpose")
        return t_off, t_edg[:R], st


def transpose_sharded_local(g, plan: ShardPlan, backend):
    """Run every rank's sender and receiver steps in one process, in sequence
    (used to check the sharded pipeline on a single GPU).  Returns the full
    (t_offsets uint64, t_edges uint32) on the host."""
    P = plan.parts
    nv = int(g.num_vertices)
    off_d = backend.to_device_offsets(g.offsets)
    sent = []
    counts = np.zeros((P, P), dtype=np.int64)
    for r in range(P):
        e0, e1 = int(plan.edge_bounds[r]), int(plan.edge_bounds[r + 1])
        edges_d = backend.to_device_edges(g.edges[e0:e1])
        rec, cnt = backend.partition(off_d, edges_d, nv, int(plan.src_bounds[r]), int(plan.src_bounds[r + 1]),
                                     plan.dst_bounds)
        sent.append(rec)
        counts[r] = cnt
    t_offsets = np.zeros(nv + 1, dtype=np.uint64)
    t_edges = np.empty(int(g.num_edges), dtype=np.uint32)
    base = 0
    for q in range(P):
        pieces = []
        for r in range(P):
            lo = int(counts[r, :q].sum())
            pieces.append(sent[r][lo : lo + int(counts[r, q])])
        torch = backend.torch
        recv = torch.cat(pieces, dim=0) if pieces else None
        lo_v, hi_v = int(plan.dst_bounds[q]), int(plan.dst_bounds[q + 1])
        t_off, t_edg, _ = backend.transpose_received(recv, lo_v, hi_v, base, src_num_vertices=nv)
        t_offsets[lo_v : hi_v + 1] = t_off.cpu().numpy().view(np.uint64)
        n = int(recv.shape[0])
        t_edges[base : base + n] = t_edg.cpu().numpy().view(np.uint32)
        base += n
    return t_offsets, t_edges


def exchange_records(records, send_counts: np.ndarray, group=None):
    """All-to-all of owner-grouped records.  Returns (received records ordered by
    sender rank, counts matrix P x P).  NCCL all_to_all_single on GPU tensors;
    with gloo (CPU tests) falls back to point-to-point send/recv."""
    import torch
    import torch.distributed as dist

    P = dist.get_world_size(group)
    r = dist.get_rank(group)
    send = torch.as_tensor(np.asarray(send_counts, dtype=np.int64), device=records.device)
    allc = [torch.empty_like(send) for _ in range(P)]
    dist.all_gather(allc, send, group=group)
    C = torch.stack(allc).cpu().numpy()  # C[s][q] = records from s to q
    recv_counts = C[:, r]
    out = torch.empty((int(recv_counts.sum()), 2), dtype=records.dtype, device=records.device)
    backend = dist.get_backend(group)
    if backend == "nccl":
        dist.all_to_all_single(out, records.contiguous(), output_split_sizes=recv_counts.tolist(),
                               input_split_sizes=[int(x) for x in send_counts], group=group)
    else:
        ops = []
        so = np.concatenate([[0], np.cumsum(send_counts)])
        ro = np.concatenate([[0], np.cumsum(recv_counts)])
        for q in range(P):
            if q == r:
                out[ro[r] : ro[r + 1]] = records[so[r] : so[r + 1]]
                continue
            if send_counts[q]:
                ops.append(dist.P2POp(dist.isend, records[so[q] : so[q + 1]].contiguous(), q, group))
            if recv_counts[q]:
                buf = out[ro[q] : ro[q + 1]]
                ops.append(dist.P2POp(dist.irecv, buf, q, group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
    return out, C


def distributed_step(offsets_d, edges_slice_d, num_vertices: int, plan: ShardPlan, rank: int, backend, group=None):
    """One rank's sharded transpose on device-resident inputs (the timed step
    of bench.py at N > 1).  Returns (t_offsets slice, t_edges slice, global base)."""
    rec, cnt = backend.partition(offsets_d, edges_slice_d, num_vertices, int(plan.src_bounds[rank]),
                                 int(plan.src_bounds[rank + 1]), plan.dst_bounds)
    recv, C = exchange_records(rec, cnt, group=group)
    base = int(C[:, :rank].sum())
    t_off, t_edg, _ = backend.transpose_received(recv, int(plan.dst_bounds[rank]), int(plan.dst_bounds[rank + 1]),
                                                 base, src_num_vertices=num_vertices)
    return t_off, t_edg, base


def transpose_distributed(g, devices: int, device=None, backend=None, group=None, gather: bool = True):
    """Collective: every rank calls with the same host CsrGraph ``g``.  Rank 0
    receives the full transposed graph (a TransposeOutput) when ``gather``;
    other ranks receive their slice in ``details``."""
    import torch
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
    off_d = backend.to_device_offsets(g.offsets)
    e0, e1 = int(plan.edge_bounds[r]), int(plan.edge_bounds[r + 1])
    edg_d = backend.to_device_edges(g.edges[e0:e1])
    t_off, t_edg, base = distributed_step(off_d, edg_d, int(g.num_vertices), plan, r, backend, group)
    details = {"rank": r, "devices": P, "dst_range": (int(plan.dst_bounds[r]), int(plan.dst_bounds[r + 1])),
               "global_base": base}
    if not gather:
        return TransposeOutput(graph=None, phase_times={}, aux_footprint_bytes=0, method="gpu-sharded", sorted=True,
                               details={**details, "t_offsets": t_off, "t_edges": t_edg})
    # gather slices on rank 0 (host), for the drop-in full-graph result
    off_np = t_off.cpu().numpy()
    edg_np = t_edg.cpu().numpy()
    objs = [None] * P
    dist.all_gather_object(objs, (r, off_np, edg_np), group=group)
    if r != 0:
        return TransposeOutput(graph=None, phase_times={}, aux_footprint_bytes=0, method="gpu-sharded", sorted=True,
                               details=details)
    nv = int(g.num_vertices)
    t_offsets = np.zeros(nv + 1, dtype=np.uint64)
    pieces = []
    for rr, o, e in sorted(objs, key=lambda t: t[0]):
        lo, hi = int(plan.dst_bounds[rr]), int(plan.dst_bounds[rr + 1])
        t_offsets[lo : hi + 1] = o.view(np.uint64)
        pieces.append(e.view(np.uint32))
    t_edges = np.concatenate(pieces) if pieces else np.empty(0, np.uint32)
    graph = type(g)(nv, int(g.num_edges), t_offsets, t_edges, flip_orientation(g.orientation))
    return TransposeOutput(graph=graph, phase_times={}, aux_footprint_bytes=0, method="gpu-sharded", sorted=True,
                           details=details)
