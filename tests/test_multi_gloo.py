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
    """CPU stand-in for GpuShardBackend (same interface and bucket geometry;
    records travel as (src, dst) pairs, rec_words = 2)."""

    torch = torch
    rec_words = 2

    def to_device_offsets(self, offsets):
        return torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.uint64).view(np.int64))

    def to_device_edges(self, edges):
        return torch.from_numpy(np.ascontiguousarray(edges, dtype=np.uint32).view(np.int32))

    def send(self, offsets_d, edges_slice_d, num_vertices, num_edges, e_begin, geom):
        off = offsets_d.numpy().view(np.uint64).astype(np.int64)
        edges = edges_slice_d.numpy().view(np.uint32)
        pos = e_begin + np.arange(edges.size, dtype=np.int64)
        owners = (np.searchsorted(off, pos, side="right") - 1).astype(np.uint32)
        bucket = (edges.astype(np.int64) >> int(geom.bucket_shift))
        order = np.argsort(bucket, kind="stable")
        rec = np.stack([owners[order], edges[order]], axis=1).astype(np.uint32).reshape(-1)
        counts = np.bincount(bucket, minlength=int(geom.num_buckets)).astype(np.int64)
        seg = np.zeros(int(geom.num_buckets) * int(geom.seg_hi_row), dtype=np.int64)
        return torch.from_numpy(rec.view(np.int32)), torch.from_numpy(counts), torch.from_numpy(seg)

    def receive(self, r1_recv, seg_recv, counts_all, parts, num_vertices, num_edges, lo, hi, num_records,
                global_base, geom, want_stats=False, check_status=True):
        shift = int(geom.bucket_shift)
        v_lo, v_hi = min(num_vertices, lo << shift), min(num_vertices, hi << shift)
        rec = r1_recv.numpy().view(np.uint32).reshape(-1, 2)
        assert rec.shape[0] == num_records
        d = rec[:, 1].astype(np.int64) - v_lo
        order = np.argsort(d, kind="stable")
        t_edges = rec[order, 0].copy()
        cnt = np.bincount(d, minlength=v_hi - v_lo)
        t_off = np.zeros(v_hi - v_lo + 1, dtype=np.uint64)
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


@pytest.mark.parametrize("world", [2, 3, 4])
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
    with pytest.raises(ValueError):
        plan_shards(off, 0)


def test_c5_memory_plan_fits():
    """Per-rank device memory of the sharded C5 step (8.6e9 edges): it fits a
    180 GB B200 from P = 2 on and shrinks ~1/P; at P = 1 the
    single-GPU path (R1 inside t_edges, no exchange buffers) is the one used."""
    from paper_2501_06872_b200.multi import memory_plan

    V, E = 1 << 29, 16 << 29
    tot = {P: memory_plan(V, E, P)["total"] for P in (1, 2, 4, 8)}
    assert tot[2] < 120e9 and tot[4] < 60e9 and tot[8] < 35e9
    assert tot[8] < tot[4] < tot[2] < tot[1]
