"""Seeded synthetic graphs for the BASELINE.json configs.

The reference ships no RMAT / Erdos-Renyi / web generator (its
``generate_skewed``, graph.py:187-222, is a Zipf-destination model that is not
one of the five configs), so these are this package's own.  Every draw is a
counter-based hash (splitmix64 finalizer) of (seed, stream, index), so the
numpy implementation here and the CUDA kernels in csrc/gt_gen.cu produce the
same edge multiset bit for bit; tests/test_gen.py checks that on the GPU.

Configs (BASELINE.json ``configs``):
  C1  RMAT scale 16, edge factor 16, a/b/c/d = .57/.19/.19/.05
  C2  Erdos-Renyi, |V| = 2^24, |E| = 2^28
  C3  RMAT scale 24, edge factor 32, IDs permuted (seeded Feistel bijection)
  C4  web-like, |V| = 2^26, |E| ~ 2^30         (generator: next round)
  C5  RMAT scale 29, edge factor 16, IDs permuted
Self-loops and duplicate edges are kept; CSR lists are sorted ascending.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

__all__ = [
    "CONFIGS",
    "GraphConfig",
    "rmat_pairs_np",
    "er_pairs_np",
    "csr_from_pairs_np",
    "generate_np",
    "generate_device",
]

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
SEED_MUL = 0xD1B54A32D192ED03
STREAM_RMAT, STREAM_PERM, STREAM_ER = 1, 2, 3
# floor(p * 2^32) for the R-MAT quadrant CDF (a, a+b, a+b+c) = (.57, .76, .95)
RMAT_A, RMAT_AB, RMAT_ABC = 2448131358, 3264175144, 4080218931


@dataclass(frozen=True)
class GraphConfig:
    name: str
    kind: str  # "rmat" | "er" | "web"
    num_vertices: int
    num_edges: int
    scale: int = 0
    permute: bool = False
    seed: int = 1

    @property
    def workload(self) -> str:
        return self.name


CONFIGS = {
    "C1": GraphConfig("C1-rmat-s16-ef16", "rmat", 1 << 16, 1 << 20, scale=16, permute=False, seed=1),
    "C2": GraphConfig("C2-er-v2^24-e2^28", "er", 1 << 24, 1 << 28, seed=2),
    "C3": GraphConfig("C3-rmat-s24-ef32-permuted", "rmat", 1 << 24, 1 << 29, scale=24, permute=True, seed=3),
    "C4": GraphConfig("C4-web-v2^26-e~2^30", "web", 1 << 26, 1 << 30, seed=4),
    "C5": GraphConfig("C5-rmat-s29-ef16-permuted", "rmat", 1 << 29, 1 << 33, scale=29, permute=True, seed=5),
}


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * np.uint64(0xBF58476D1CE4E5B9)
    z = z ^ (z >> np.uint64(27))
    z = z * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _mix64_int(z: int) -> int:
    z &= M64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & M64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _stream_key(seed: int, stream: int) -> int:
    return _mix64_int((seed * SEED_MUL + stream * GOLDEN + 1) & M64)


def _hash_at(key: int, idx: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        return _mix64(np.uint64(key) + (idx.astype(np.uint64) + np.uint64(1)) * np.uint64(GOLDEN))


def _feistel(x: np.ndarray, keys, half: int, mask: int) -> np.ndarray:
    L = x >> np.uint64(half)
    R = x & np.uint64(mask)
    with np.errstate(over="ignore"):
        for k in keys:
            t = L ^ (_mix64(R ^ np.uint64(k)) & np.uint64(mask))
            L, R = R, t
    return (L << np.uint64(half)) | R


def _permute(x: np.ndarray, scale: int, seed: int) -> np.ndarray:
    width = scale + (scale & 1)
    half = width // 2
    mask = (1 << half) - 1
    pk = _stream_key(seed, STREAM_PERM)
    keys = [int(_hash_at(pk, np.array([r]))[0]) for r in range(4)]
    n = np.uint64(1 << scale)
    y = _feistel(x.astype(np.uint64), keys, half, mask)
    bad = y >= n
    while bad.any():  # cycle walking (odd scales)
        y[bad] = _feistel(y[bad], keys, half, mask)
        bad = y >= n
    return y


def rmat_pairs_np(scale: int, num_edges: int, seed: int, permute: bool, chunk: int = 1 << 22):
    """R-MAT (a,b,c,d) = (.57,.19,.19,.05) edge pairs, as uint32 src/dst arrays."""
    key = _stream_key(seed, STREAM_RMAT)
    src = np.empty(num_edges, dtype=np.uint32)
    dst = np.empty(num_edges, dtype=np.uint32)
    for lo in range(0, num_edges, chunk):
        hi = min(num_edges, lo + chunk)
        e = np.arange(lo, hi, dtype=np.uint64)
        s = np.zeros(hi - lo, dtype=np.uint64)
        d = np.zeros(hi - lo, dtype=np.uint64)
        for l in range(0, scale, 2):
            h = _hash_at(key, e * np.uint64(16) + np.uint64(l >> 1))
            for q in range(2):
                if l + q >= scale:
                    break
                u = (h >> np.uint64(32 * q)) & np.uint64(0xFFFFFFFF)
                bit = np.uint64(1 << (scale - 1 - (l + q)))
                in_b = (u >= RMAT_A) & (u < RMAT_AB)
                in_c = (u >= RMAT_AB) & (u < RMAT_ABC)
                in_d = u >= RMAT_ABC
                d |= np.where(in_b | in_d, bit, np.uint64(0))
                s |= np.where(in_c | in_d, bit, np.uint64(0))
        if permute:
            s = _permute(s, scale, seed)
            d = _permute(d, scale, seed)
        src[lo:hi] = s
        dst[lo:hi] = d
    return src, dst


def er_pairs_np(num_vertices: int, num_edges: int, seed: int):
    """Uniform directed Erdos-Renyi pairs (multiply-high of 32-bit draws)."""
    key = _stream_key(seed, STREAM_ER)
    e = np.arange(num_edges, dtype=np.uint64)
    v = np.uint64(num_vertices)
    with np.errstate(over="ignore"):
        src = (((_hash_at(key, e * np.uint64(2)) >> np.uint64(32)) * v) >> np.uint64(32)).astype(np.uint32)
        dst = (((_hash_at(key, e * np.uint64(2) + np.uint64(1)) >> np.uint64(32)) * v) >> np.uint64(32)).astype(
            np.uint32
        )
    return src, dst


def csr_from_pairs_np(src, dst, num_vertices: int):
    """CSR with lists ascending by destination (graph.py:104-122 semantics)."""
    order = np.lexsort((dst, src))
    edges = np.ascontiguousarray(dst[order].astype(np.uint32))
    counts = np.bincount(src.astype(np.int64), minlength=num_vertices)
    offsets = np.zeros(num_vertices + 1, dtype=np.uint64)
    np.cumsum(counts, out=offsets[1:])
    return offsets, edges


def generate_np(cfg: GraphConfig):
    """(offsets uint64[V+1], edges uint32[E]) on the host (small configs)."""
    if cfg.kind == "rmat":
        s, d = rmat_pairs_np(cfg.scale, cfg.num_edges, cfg.seed, cfg.permute)
    elif cfg.kind == "er":
        s, d = er_pairs_np(cfg.num_vertices, cfg.num_edges, cfg.seed)
    else:
        raise NotImplementedError(f"{cfg.kind} generator lands next round")
    return csr_from_pairs_np(s, d, cfg.num_vertices)


def generate_device(cfg: GraphConfig, device="cuda", num_edges: int | None = None):
    """Generate the config's CSR directly in HBM with libgt.so.  Returns torch
    tensors (offsets int64[V+1], edges int32[E]) holding uint64/uint32 bits."""
    import torch

    from . import _lib

    E = cfg.num_edges if num_edges is None else int(num_edges)
    V = cfg.num_vertices
    dev = torch.device(device)
    stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    src = torch.empty(E, dtype=torch.int32, device=dev)
    dst = torch.empty(E, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        if cfg.kind == "rmat":
            rc = _lib.lib.gt_gen_rmat(cfg.scale, E, cfg.seed, int(cfg.permute), ctypes.c_void_p(src.data_ptr()),
                                      ctypes.c_void_p(dst.data_ptr()), stream)
        elif cfg.kind == "er":
            rc = _lib.lib.gt_gen_er(V, E, cfg.seed, ctypes.c_void_p(src.data_ptr()),
                                    ctypes.c_void_p(dst.data_ptr()), stream)
        else:
            raise NotImplementedError(f"{cfg.kind} generator lands next round")
        _lib.check(rc, "generator")
        offsets = torch.empty(V + 1, dtype=torch.int64, device=dev)
        edges = torch.empty(E, dtype=torch.int32, device=dev)
        rc = _lib.lib.gt_build_csr(ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()), V, E,
                                   ctypes.c_void_p(offsets.data_ptr()), ctypes.c_void_p(edges.data_ptr()), stream)
        _lib.check(rc, "gt_build_csr")
    del src, dst
    return offsets, edges
