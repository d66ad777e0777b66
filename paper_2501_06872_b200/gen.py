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
  C4  web-like, |V| = 2^26, |E| ~ 2^30: out-degrees Zipf(2.1) on [1, 2^16]
      rescaled to |E| ~ 2^30; each edge lands uniformly within +-4096 of its
      source with probability 0.85, else on one of 2^16 seeded hubs drawn
      Zipf(1.2).  The two Zipf laws are inverse-CDF threshold tables built
      once here (float64) and shared with the CUDA kernels, so both sides
      draw identical integers.
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
    "WebParams",
    "web_tables",
    "web_pairs_np",
    "csr_from_pairs_np",
    "generate_np",
    "generate_device",
]

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
SEED_MUL = 0xD1B54A32D192ED03
STREAM_RMAT, STREAM_PERM, STREAM_ER, STREAM_WDEG, STREAM_WEDGE, STREAM_HUB = 1, 2, 3, 4, 5, 6
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
    web: "WebParams | None" = None

    @property
    def workload(self) -> str:
        return self.name


CONFIGS = {
    "C1": GraphConfig("C1-rmat-s16-ef16", "rmat", 1 << 16, 1 << 20, scale=16, permute=False, seed=1),
    "C2": GraphConfig("C2-er-v2^24-e2^28", "er", 1 << 24, 1 << 28, seed=2),
    "C3": GraphConfig("C3-rmat-s24-ef32-permuted", "rmat", 1 << 24, 1 << 29, scale=24, permute=True, seed=3),
    "C4": GraphConfig("C4-web-v2^26-e~2^30", "web", 1 << 26, 1 << 30, scale=26, seed=4),
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


# ---------------------------------------------------------------- web-like (C4)
@dataclass(frozen=True)
class WebParams:
    """Web-like generator parameters (BASELINE.json config 4 at the defaults)."""

    deg_alpha: float = 2.1      # out-degree Zipf exponent
    deg_max: int = 1 << 16      # truncation [1, deg_max]
    hubs: int = 1 << 16         # hub set size
    hub_alpha: float = 1.2      # hub popularity Zipf exponent
    window: int = 4096          # local destinations uniform in [v - window, v + window] (mod |V|)
    p_local: float = 0.85


P_LOCAL_Q32 = 3650722201  # floor(0.85 * 2^32)


def _zipf_thresholds(n: int, alpha: float) -> np.ndarray:
    """uint64 inverse-CDF thresholds of P(k) ~ k^-alpha, k = 1..n: a 64-bit draw
    u maps to index searchsorted(T, u, 'right') (0-based rank)."""
    w = np.arange(1, n + 1, dtype=np.float64) ** (-alpha)
    c = np.cumsum(w)
    c /= c[-1]
    # largest float64 below 2^64 is 2^64 - 2048: keeps every entry representable
    t = np.minimum(np.floor(c * 18446744073709551616.0), 18446744073709549568.0)
    out = np.empty(n, dtype=np.uint64)
    # exact conversion of float64 values < 2^64 to uint64
    hi = np.floor(t / 4294967296.0)
    lo = t - hi * 4294967296.0
    out[:] = (hi.astype(np.uint64) << np.uint64(32)) | lo.astype(np.uint64)
    out[-1] = np.uint64(M64)
    return out


def web_tables(num_vertices: int, target_edges: int, wp: WebParams = WebParams()):
    """(degree thresholds, hub thresholds, degree scale in Q16) for a web-like graph."""
    dt = _zipf_thresholds(wp.deg_max, wp.deg_alpha)
    ht = _zipf_thresholds(wp.hubs, wp.hub_alpha)
    k = np.arange(1, wp.deg_max + 1, dtype=np.float64)
    w = k ** (-wp.deg_alpha)
    mean = float((k * w).sum() / w.sum())
    scale_q16 = int(round(65536.0 * target_edges / (num_vertices * mean)))
    return dt, ht, max(scale_q16, 1)


def web_degrees_np(num_vertices: int, seed: int, dt: np.ndarray, scale_q16: int) -> np.ndarray:
    key = _stream_key(seed, STREAM_WDEG)
    u = _hash_at(key, np.arange(num_vertices, dtype=np.uint64))
    k = np.searchsorted(dt, u, side="right").astype(np.uint64) + np.uint64(1)  # 1..deg_max
    d = (k * np.uint64(scale_q16) + np.uint64(32768)) >> np.uint64(16)
    return np.maximum(d, np.uint64(1))


def web_hub_ids(num_vertices: int, hubs: int, seed: int) -> np.ndarray:
    """Seeded hub set: a Feistel bijection of [0, |V|) applied to hub ranks."""
    scale = int(num_vertices).bit_length() - 1
    assert 1 << scale == num_vertices, "web-like graphs use |V| = 2^scale"
    return _permute(np.arange(hubs, dtype=np.uint64), scale, seed ^ 0x5A5A)


def web_pairs_np(num_vertices: int, target_edges: int, seed: int, wp: WebParams = WebParams()):
    """Web-like edge pairs (uint32 src, dst) in generation order."""
    dt, ht, sq = web_tables(num_vertices, target_edges, wp)
    deg = web_degrees_np(num_vertices, seed, dt, sq)
    E = int(deg.sum())
    src = np.repeat(np.arange(num_vertices, dtype=np.uint32), deg.astype(np.int64))
    e = np.arange(E, dtype=np.uint64)
    key = _stream_key(seed, STREAM_WEDGE)
    ha = _hash_at(key, e * np.uint64(2))
    hb = _hash_at(key, e * np.uint64(2) + np.uint64(1))
    local = (ha & np.uint64(0xFFFFFFFF)) < np.uint64(P_LOCAL_Q32)
    span = np.uint64(2 * wp.window + 1)
    off = ((ha >> np.uint64(32)) * span) >> np.uint64(32)  # 0..2*window
    V = np.uint64(num_vertices)
    ldst = (src.astype(np.uint64) + V - np.uint64(wp.window) + off) % V
    hubs = web_hub_ids(num_vertices, wp.hubs, seed)
    r = np.searchsorted(ht, hb, side="right")
    hdst = hubs[r]
    dst = np.where(local, ldst, hdst).astype(np.uint32)
    return src, dst


def generate_np(cfg: GraphConfig):
    """(offsets uint64[V+1], edges uint32[E]) on the host (small configs)."""
    if cfg.kind == "rmat":
        s, d = rmat_pairs_np(cfg.scale, cfg.num_edges, cfg.seed, cfg.permute)
    elif cfg.kind == "er":
        s, d = er_pairs_np(cfg.num_vertices, cfg.num_edges, cfg.seed)
    elif cfg.kind == "web":
        s, d = web_pairs_np(cfg.num_vertices, cfg.num_edges, cfg.seed, cfg.web or WebParams())
    else:
        raise ValueError(f"unknown generator kind {cfg.kind!r}")
    return csr_from_pairs_np(s, d, cfg.num_vertices)


def generate_device(cfg: GraphConfig, device="cuda", num_edges: int | None = None, lean: bool | None = None):
    """Generate the config's CSR directly in HBM with libgt.so.  Returns torch
    tensors (offsets int64[V+1], edges int32[E]) holding uint64/uint32 bits.

    ``lean`` (default: R-MAT with more than 2^31 edges, i.e. config C5) never
    materialises the edge pairs: gt_gen_rmat_csr writes the CSR with lists in
    generation order and two transposes sort the lists (T(T(g)) has g's
    offsets and every list ascending), so the peak is input + output + the
    transpose workspace."""
    import torch

    from . import _lib

    E = cfg.num_edges if num_edges is None else int(num_edges)
    if lean is None:
        lean = cfg.kind == "rmat" and E > (1 << 31)
    if lean and cfg.kind == "rmat":
        return _rmat_lean_device(cfg, E, torch.device(device))
    V = cfg.num_vertices
    dev = torch.device(device)
    stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    if cfg.kind == "web":
        src, dst = web_pairs_device(cfg, dev)
        E = int(src.numel())
    else:
        src = torch.empty(E, dtype=torch.int32, device=dev)
        dst = torch.empty(E, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        if cfg.kind == "web":
            rc = 0
        elif cfg.kind == "rmat":
            rc = _lib.lib.gt_gen_rmat(cfg.scale, E, cfg.seed, int(cfg.permute), ctypes.c_void_p(src.data_ptr()),
                                      ctypes.c_void_p(dst.data_ptr()), stream)
        elif cfg.kind == "er":
            rc = _lib.lib.gt_gen_er(V, E, cfg.seed, ctypes.c_void_p(src.data_ptr()),
                                    ctypes.c_void_p(dst.data_ptr()), stream)
        else:
            raise ValueError(f"unknown generator kind {cfg.kind!r}")
        _lib.check(rc, "generator")
        offsets = torch.empty(V + 1, dtype=torch.int64, device=dev)
        edges = torch.empty(E, dtype=torch.int32, device=dev)
        rc = _lib.lib.gt_build_csr(ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()), V, E,
                                   ctypes.c_void_p(offsets.data_ptr()), ctypes.c_void_p(edges.data_ptr()), stream)
        _lib.check(rc, "gt_build_csr")
    del src, dst
    return offsets, edges


def web_pairs_device(cfg: GraphConfig, device="cuda"):
    """Web-like pairs generated in HBM by libgt.so (identical to web_pairs_np).
    Returns torch int32 tensors (src, dst) holding uint32 bits."""
    import torch

    from . import _lib

    wp = cfg.web or WebParams()
    V = cfg.num_vertices
    dt, ht, sq = web_tables(V, cfg.num_edges, wp)
    hubs = web_hub_ids(V, wp.hubs, cfg.seed).astype(np.uint32)
    dev = torch.device(device)
    with torch.cuda.device(dev):
        stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        d_dt = torch.from_numpy(dt.view(np.int64)).to(dev)
        d_ht = torch.from_numpy(ht.view(np.int64)).to(dev)
        d_hubs = torch.from_numpy(hubs.view(np.int32)).to(dev)
        offs = torch.empty(V + 1, dtype=torch.int64, device=dev)
        n_edges = ctypes.c_uint64(0)
        rc = _lib.lib.gt_gen_web_degrees(V, cfg.seed, ctypes.c_void_p(d_dt.data_ptr()), dt.shape[0], sq,
                                         ctypes.c_void_p(offs.data_ptr()), ctypes.byref(n_edges), stream)
        _lib.check(rc, "gt_gen_web_degrees")
        E = int(n_edges.value)
        src = torch.empty(E, dtype=torch.int32, device=dev)
        dst = torch.empty(E, dtype=torch.int32, device=dev)
        rc = _lib.lib.gt_gen_web_edges(V, cfg.seed, ctypes.c_void_p(offs.data_ptr()), ctypes.c_void_p(d_ht.data_ptr()),
                                       ht.shape[0], ctypes.c_void_p(d_hubs.data_ptr()), wp.window, P_LOCAL_Q32,
                                       ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()), stream)
        _lib.check(rc, "gt_gen_web_edges")
    return src, dst


def _rmat_lean_device(cfg: GraphConfig, E: int, dev):
    import torch

    from . import _lib
    from .transpose import transpose_device

    V = cfg.num_vertices
    with torch.cuda.device(dev):
        stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        offsets = torch.empty(V + 1, dtype=torch.int64, device=dev)
        raw = torch.empty(E, dtype=torch.int32, device=dev)
        rc = _lib.lib.gt_gen_rmat_csr(cfg.scale, E, cfg.seed, int(cfg.permute), ctypes.c_void_p(offsets.data_ptr()),
                                      ctypes.c_void_p(raw.data_ptr()), stream)
        _lib.check(rc, "gt_gen_rmat_csr")
        t_off, t_edg, _ = transpose_device(offsets, raw, V)  # lists of T(g): ascending sources
        del raw
        torch.cuda.empty_cache()
        edges = torch.empty(E, dtype=torch.int32, device=dev)
        transpose_device(t_off, t_edg, V, t_offsets=offsets, t_edges=edges)  # T(T(g)): g with sorted lists
        del t_off, t_edg
        torch.cuda.empty_cache()
    return offsets, edges
