"""TEST INFRASTRUCTURE ONLY — CPU oracle for the transposition path.

Imported by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg;
never by the product package.  Two restatements of the reference algorithm:

* ``transpose_np`` — numpy restatement of ``transpose_oracle``
  (pkg/src/potra/graph.py:136-148, via from_edge_pairs graph.py:104-122 and
  _owners graph.py:125-129): owners = repeat(arange(V), degrees); a *stable*
  argsort by endpoint of the CSR-ordered stream equals the reference's
  lexsort((owner, endpoint)) because owners are non-decreasing in CSR order;
  offsets = bincount + cumsum.
* ``libgt_oracle.so`` (gt_oracle.c, built by oracle/Makefile): serial stable
  counting sort (same order, 64-bit cursors) plus OpenMP ports of the
  reference's parallel CPU algorithms used as the CPU baseline:
  transpose_scantrans (baselines.py:265-312), transpose_atomic
  (baselines.py:168-209) and sort_neighbor_lists (baselines.py:457-475).

* ``sample_hdv_np`` — numpy restatement of step 0's ``sample_hdv``
  (hlh.py:153-218) with the reference's generators (worker_seeds /
  xoshiro_seed_scalar / xoshiro_step, _nb.py:47-93), vectorised over the
  worker streams; pinned by tests/golden/hdv_cases.npz (make_hdv_golden.py).

Pinned against the reference: tests/golden/ holds outputs of the real
``potra.transpose_oracle`` (made by tests/golden/make_golden.py, which imports
/root/reference); tests/test_oracle.py checks both restatements against them.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "libgt_oracle.so"

GTO_OK, GTO_EINVAL, GTO_EOVERFLOW, GTO_ENOMEM = 0, -1, -2, -3


def transpose_np(offsets: np.ndarray, edges: np.ndarray, num_vertices: int):
    """numpy restatement of transpose_oracle -> (t_offsets uint64, t_edges uint32)."""
    offsets = np.asarray(offsets, dtype=np.uint64)
    edges = np.asarray(edges)
    deg = np.diff(offsets.view(np.int64))
    owners = np.repeat(np.arange(num_vertices, dtype=np.uint32), deg)
    order = np.argsort(edges, kind="stable")
    t_edges = np.ascontiguousarray(owners[order].astype(np.uint32))
    counts = np.bincount(edges.astype(np.int64), minlength=num_vertices)
    t_offsets = np.zeros(num_vertices + 1, dtype=np.uint64)
    np.cumsum(counts, out=t_offsets[1:])
    return t_offsets, t_edges


_lib = None


def build():
    """Compile gt_oracle.c into oracle/libgt_oracle.so (gcc, OpenMP)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        lib = ctypes.CDLL(str(LIB))
        vp, u64, i = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int
        lib.gto_transpose_serial.argtypes = [vp, vp, u64, u64, vp, vp]
        lib.gto_transpose_scantrans.argtypes = [vp, vp, u64, u64, vp, vp, i]
        lib.gto_transpose_atomic.argtypes = [vp, vp, u64, u64, vp, vp, i, u64]
        lib.gto_sort_lists.argtypes = [vp, u64, vp, i]
        lib.gto_scan_exclusive.argtypes = [vp, u64, vp, i]
        lib.gto_edge_balanced_bounds.argtypes = [vp, u64, ctypes.c_int64, vp]
        lib.gto_edge_balanced_bounds.restype = None
        lib.gto_generate.argtypes = [i, i, i, u64, u64, u64, vp, vp, i]
        d, i64 = ctypes.c_double, ctypes.c_int64
        lib.gto_transpose_potra.argtypes = [vp, vp, u64, u64, vp, vp, i, i64, d, u64, u64, i, vp, vp, vp]
        for f in ("gto_transpose_serial", "gto_transpose_scantrans", "gto_transpose_atomic", "gto_sort_lists",
                  "gto_scan_exclusive", "gto_max_threads", "gto_generate", "gto_transpose_potra"):
            getattr(lib, f).restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(rc: int, what: str):
    if rc == GTO_OK:
        return
    if rc == GTO_EOVERFLOW:
        raise OverflowError(f"{what}: 32-bit counter overflow")
    if rc == GTO_EINVAL:
        raise ValueError(what)
    raise MemoryError(what)


def transpose_c(offsets, edges, num_vertices: int):
    """Serial stable counting sort in C (the checker for large sizes)."""
    lib = load()
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    e = np.ascontiguousarray(edges, dtype=np.uint32)
    t_off = np.empty(num_vertices + 1, dtype=np.uint64)
    t_e = np.empty(e.shape[0], dtype=np.uint32)
    _check(lib.gto_transpose_serial(_p(off), _p(e), num_vertices, e.shape[0], _p(t_off), _p(t_e)),
           "gto_transpose_serial")
    return t_off, t_e


def transpose_scantrans_c(offsets, edges, num_vertices: int, threads: int):
    """OpenMP port of transpose_scantrans (sorted by construction)."""
    lib = load()
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    e = np.ascontiguousarray(edges, dtype=np.uint32)
    t_off = np.empty(num_vertices + 1, dtype=np.uint64)
    t_e = np.empty(e.shape[0], dtype=np.uint32)
    _check(lib.gto_transpose_scantrans(_p(off), _p(e), num_vertices, e.shape[0], _p(t_off), _p(t_e), threads),
           "gto_transpose_scantrans")
    return t_off, t_e


def transpose_atomic_sorted_c(offsets, edges, num_vertices: int, threads: int, partition_edges: int = 1 << 18):
    """OpenMP port of transpose_atomic followed by sort_neighbor_lists."""
    lib = load()
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    e = np.ascontiguousarray(edges, dtype=np.uint32)
    t_off = np.empty(num_vertices + 1, dtype=np.uint64)
    t_e = np.empty(e.shape[0], dtype=np.uint32)
    _check(lib.gto_transpose_atomic(_p(off), _p(e), num_vertices, e.shape[0], _p(t_off), _p(t_e), threads,
                                    partition_edges), "gto_transpose_atomic")
    _check(lib.gto_sort_lists(_p(t_off), num_vertices, _p(t_e), threads), "gto_sort_lists")
    return t_off, t_e


def generate_c(cfg, threads: int):
    """Seeded R-MAT / Erdos-Renyi CSR (gen.generate_np's draws) on host cores.
    Used where the product library must not be loaded (bench.py's reference arm)."""
    if cfg.kind not in ("rmat", "er"):
        raise ValueError(f"generate_c covers rmat and er, not {cfg.kind!r}")
    lib = load()
    off = np.empty(cfg.num_vertices + 1, dtype=np.uint64)
    e = np.empty(cfg.num_edges, dtype=np.uint32)
    _check(lib.gto_generate(0 if cfg.kind == "rmat" else 1, cfg.scale, int(cfg.permute), cfg.num_vertices,
                            cfg.num_edges, cfg.seed, _p(off), _p(e), threads), "gto_generate")
    return off, e


def detect_cache_budget():
    """hw.detect_cache_budget (hw.py:19-63): L2 + L3 bytes from sysfs, or None."""
    import glob

    units = {"K": 1024, "M": 1024 ** 2, "G": 1024 ** 3}
    seen, tot = set(), {}
    for d in glob.glob("/sys/devices/system/cpu/cpu*/cache/index*"):
        try:
            lvl = int(open(os.path.join(d, "level")).read())
            typ = open(os.path.join(d, "type")).read().strip()
            sz = open(os.path.join(d, "size")).read().strip()
            sh = open(os.path.join(d, "shared_cpu_list")).read().strip()
        except (OSError, ValueError):
            continue
        if typ == "Instruction" or (lvl, sh) in seen:
            continue
        seen.add((lvl, sh))
        b = int(sz[:-1]) * units[sz[-1].upper()] if sz and sz[-1].upper() in units else int(sz)
        tot[lvl] = tot.get(lvl, 0) + b
    return (tot.get(2, 0) + tot.get(3, 0)) or None


def potra_k(threads: int, cache_bytes=None, load_factor: float = 0.5) -> int:
    """k of transpose_potra's default budget: hdv_count (model.py:65-75) then
    _fit_table_budget (hlh.py:422-433), 12-byte slots, 13 B per HDV per thread."""
    import math

    cache = cache_bytes or detect_cache_budget() or 32 * 1024 * 1024
    k_raw = max(0, math.floor(cache / (12 / load_factor + 13 * threads)))
    if k_raw <= 0:
        return 0
    cap = max(2, 1 << max(1, (math.ceil(k_raw / load_factor) - 1).bit_length()))
    while cap >= 2:
        k = min(k_raw, math.floor(load_factor * cap))
        if 12 * cap + 13 * threads * k <= cache:
            return k
        cap //= 2
    return 0


def transpose_potra_c(offsets, edges, num_vertices: int, threads: int, k=None, sample_fraction: float = 0.01,
                      seed: int = 0, partition_edges: int = 1 << 18, force_method=None, sort: bool = False):
    """OpenMP port of transpose_potra (hlh.py:441-588), optionally followed by
    sort_neighbor_lists.  Returns (t_offsets, t_edges, info dict with the
    reference's phase names)."""
    import time

    lib = load()
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    e = np.ascontiguousarray(edges, dtype=np.uint32)
    t_off = np.empty(num_vertices + 1, dtype=np.uint64)
    t_e = np.empty(e.shape[0], dtype=np.uint32)
    if k is None:
        k = potra_k(threads)
    phase = np.zeros(4, np.float64)
    info = np.zeros(3, np.int64)
    est = np.zeros(1, np.float64)
    fm = {None: -1, "atomic": 0, "hlh": 1}[force_method]
    _check(lib.gto_transpose_potra(_p(off), _p(e), num_vertices, e.shape[0], _p(t_off), _p(t_e), threads, int(k),
                                   float(sample_fraction), seed, partition_edges, fm, _p(phase), _p(info), _p(est)),
           "gto_transpose_potra")
    out = {"method_chosen": "hlh" if info[0] else "atomic", "k": int(info[1]), "sample_size": int(info[2]),
           "coverage_estimate": float(est[0]),
           "phase_times": {"step0": phase[0], "step1": phase[1], "step2": phase[2], "step3": phase[3]}}
    if sort:
        t0 = time.perf_counter()
        _check(lib.gto_sort_lists(_p(t_off), num_vertices, _p(t_e), threads), "gto_sort_lists")
        out["phase_times"]["sort"] = time.perf_counter() - t0
    return t_off, t_e, out


def edge_balanced_bounds_c(offsets, parts: int):
    lib = load()
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    parts = max(1, int(parts))
    out = np.empty(parts + 1, dtype=np.int64)
    lib.gto_edge_balanced_bounds(_p(off), off.shape[0] - 1, parts, _p(out))
    return out


def edge_balanced_bounds_np(offsets, parts: int):
    """Restates edge_balanced_vertex_bounds (_nb.py:118-132)."""
    offsets = np.asarray(offsets, dtype=np.uint64)
    nv = offsets.shape[0] - 1
    ne = int(offsets[-1])
    parts = max(1, parts)
    targets = (np.arange(parts + 1, dtype=np.int64) * ne) // parts
    bounds = np.searchsorted(offsets, targets.astype(np.uint64), side="left").astype(np.int64)
    bounds[0] = 0
    bounds[-1] = nv
    return bounds


_M64 = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15


def _mix64(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _rotl(x, k):
    return (x << np.uint64(k)) | (x >> np.uint64(64 - k))


def _tally_np(edges, nv, num_samples, seeds):
    """_sample_tally (hlh.py:153-164): stream w draws samples
    [w*N/W, (w+1)*N/W) as edges[r % E]; all streams advance together."""
    W = len(seeds)
    freq = np.zeros(nv, np.int64)
    st = np.zeros((4, W), np.uint64)
    for w, sd in enumerate(seeds):  # xoshiro_seed_scalar (_nb.py:62-69)
        x = sd
        for j in range(4):
            x = (x + _GAMMA) & _M64
            st[j, w] = _mix64(x)
    lo = np.array([w * num_samples // W for w in range(W)], np.int64)
    cnt = np.array([(w + 1) * num_samples // W for w in range(W)], np.int64) - lo
    n = np.uint64(edges.shape[0])
    s0, s1, s2, s3 = st
    with np.errstate(over="ignore"):
        for i in range(int(cnt.max()) if W else 0):
            r = _rotl(s1 * np.uint64(5), 7) * np.uint64(9)  # xoshiro_step (_nb.py:72-83)
            t = s1 << np.uint64(17)
            s2 ^= s0
            s3 ^= s1
            s1 ^= s2
            s0 ^= s3
            s2 ^= t
            s3 = _rotl(s3, 45)
            live = cnt > i
            np.add.at(freq, edges[(r[live] % n).astype(np.int64)].astype(np.int64), 1)
    return freq


def sample_hdv_np(edges, nv: int, k: int, sample_fraction: float, seed: int, threads: int):
    """Restates sample_hdv (hlh.py:167-218): returns (hdv_ids uint64, coverage_estimate, sample_size)."""
    import math

    edges = np.asarray(edges).view(np.uint32)
    ne = edges.shape[0]
    k = min(k, nv)
    if sample_fraction >= 1.0 or ne == 0:
        freq = np.bincount(edges.astype(np.int64), minlength=nv) if ne else np.zeros(nv, np.int64)
        est = freq
        size = ne
    else:
        size = math.ceil(sample_fraction * nv)
        seeds, x = [], seed & _M64
        for _ in range(2 * threads):  # worker_seeds (_nb.py:86-93)
            x = (x + _GAMMA) & _M64
            seeds.append(_mix64(x))
        freq = _tally_np(edges, nv, size, seeds[:threads]) if size else np.zeros(nv, np.int64)
        est = _tally_np(edges, nv, size, seeds[threads:]) if size else np.zeros(nv, np.int64)
    ids = np.lexsort((np.arange(nv, dtype=np.int64), -freq))[:k].astype(np.uint64) if k else np.empty(0, np.uint64)
    hits = int(est[ids.astype(np.int64)].sum()) if k else 0
    return ids, (hits / size if size else 0.0), size


def max_threads() -> int:
    return int(load().gto_max_threads())


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
