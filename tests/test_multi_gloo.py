"""World-size-2 (and 3) gloo tests of the multi-GPU host logic on CPU: source
sharding, owner counts all_gather, record exchange, global bases, slice
assembly.  The per-rank kernels are replaced by a CPU stand-in built on the
oracle's stable order (test infrastructure); the exchange/orchestration code is
the product's own (paper_2501_06872_b200.multi)."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

sys.path.insert(0, str(ROOT))


class CpuShardBackend:
    """CPU stand-in for GpuShardBackend (same interface)."""

    torch = torch

    def to_device_offsets(self, offsets):
        return torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.uint64).view(np.int64))

    def to_device_edges(self, edges):
        return torch.from_numpy(np.ascontiguousarray(edges, dtype=np.uint32).view(np.int32))

    def partition(self, offsets_d, edges_slice_d, num_vertices, src_lo, src_hi, dst_bounds):
        off = offsets_d.numpy().view(np.uint64)
        edges = edges_slice_d.numpy().view(np.uint32)
        deg = np.diff(off[src_lo : src_hi + 1].astype(np.int64))
        owners = np.repeat(np.arange(src_lo, src_hi, dtype=np.uint32), deg)
        owner_rank = np.searchsorted(np.asarray(dst_bounds)[1:-1], edges, side="right")
        order = np.argsort(owner_rank, kind="stable")
        rec = np.stack([owners[order], edges[order]], axis=1).astype(np.uint32)
        counts = np.bincount(owner_rank, minlength=len(dst_bounds) - 1).astype(np.int64)
        return torch.from_numpy(rec.view(np.int32)), counts

    def transpose_received(self, records, dst_lo, dst_hi, global_base, want_stats=False, src_num_vertices=None):
        rec = records.numpy().view(np.uint32).reshape(-1, 2)
        d = rec[:, 1].astype(np.int64) - dst_lo
        order = np.argsort(d, kind="stable")
        t_edges = rec[order, 0].copy()
        cnt = np.bincount(d, minlength=dst_hi - dst_lo)
        t_off = np.zeros(dst_hi - dst_lo + 1, dtype=np.uint64)
        np.cumsum(cnt, out=t_off[1:])
        t_off += np.uint64(global_base)
        return torch.from_numpy(t_off.view(np.int64)), torch.from_numpy(t_edges.view(np.int32)), None


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, seed, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2501_06872_b200.graph import CsrGraph
        from paper_2501_06872_b200.multi import transpose_distributed

        rng = np.random.default_rng(seed)
        nv, ne = 5003, 60_000
        src = rng.integers(0, nv, ne)
        dst = np.minimum((nv * rng.random(ne) ** 2).astype(np.int64), nv - 1)
        g = CsrGraph.from_edge_pairs(src, dst, nv)
        out = transpose_distributed(g, devices=world, backend=CpuShardBackend())
        if rank == 0:
            np.savez(result_path, off=out.graph.offsets, edg=out.graph.edges, ioff=g.offsets, iedg=g.edges, nv=nv)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_exchange_gloo(tmp_path, world):
    from oracle import oracle

    path = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(world, _free_port(), 17 + world, path), nprocs=world, join=True)
    z = np.load(path)
    o, e = oracle.transpose_c(z["ioff"], z["iedg"], int(z["nv"]))
    assert np.array_equal(z["off"], o)
    assert np.array_equal(z["edg"], e)


def test_plan_shards_contract():
    from paper_2501_06872_b200.multi import plan_shards

    off = np.array([0, 5, 5, 6, 20, 21, 30], dtype=np.uint64)
    p = plan_shards(off, 3)
    assert p.src_bounds.tolist() == [0, 4, 4, 6]  # edge_balanced_vertex_bounds probe
    assert p.edge_bounds.tolist() == [0, 20, 20, 30]
    assert p.dst_bounds.tolist() == [0, 2, 4, 6]
    with pytest.raises(ValueError):
        plan_shards(off, 0)
    with pytest.raises(ValueError):
        plan_shards(off, 2, dst_bounds=[0, 7, 6])
