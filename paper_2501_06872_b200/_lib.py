"""ctypes binding of libgt.so (the C ABI declared in include/gt.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2501_06872_b200/csrc``).  There is no fallback: if the library
cannot be loaded every GPU entry point raises :class:`GpuUnavailableError`.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import CounterOverflowError, FootprintError, GpuUnavailableError

__all__ = ["lib", "GtStats", "GtConfig", "ShardGeom", "MultiInfo", "PotgHeader", "check", "LIB_PATH", "SYMBOLS", "load"]

LIB_PATH = Path(__file__).resolve().parent / "libgt.so"

GT_OK, GT_EINVAL, GT_EOVERFLOW, GT_ENOMEM, GT_ECUDA, GT_ENODEV = 0, -1, -2, -3, -4, -5
GT_EFORMAT, GT_EIO = -6, -7


class GtStats(ctypes.Structure):
    _fields_ = [
        ("ms_total", ctypes.c_double),
        ("ms_step1", ctypes.c_double),
        ("ms_step2", ctypes.c_double),
        ("ms_step3", ctypes.c_double),
        ("workspace_bytes", ctypes.c_uint64),
        ("bits", ctypes.c_int32 * 3),
        ("rank_mode", ctypes.c_int32),
        ("n_big_buckets", ctypes.c_uint64),
        ("n_launches", ctypes.c_uint64),
        ("ms_kernel", ctypes.c_double * 4),
    ]


class GtConfig(ctypes.Structure):
    _fields_ = [("split", ctypes.c_int32 * 3), ("force_wide", ctypes.c_int32), ("reserved", ctypes.c_int32 * 4)]


class ShardGeom(ctypes.Structure):
    _fields_ = [
        ("num_buckets", ctypes.c_uint32),
        ("bucket_shift", ctypes.c_uint32),
        ("seg_hi_row", ctypes.c_uint32),
        ("wide", ctypes.c_uint32),
        ("bits", ctypes.c_int32 * 3),
        ("pad", ctypes.c_uint32),
    ]


class MultiInfo(ctypes.Structure):
    _fields_ = [
        ("dst_begin", ctypes.c_uint64),
        ("dst_end", ctypes.c_uint64),
        ("global_base", ctypes.c_uint64),
        ("num_local_edges", ctypes.c_uint64),
        ("bucket_lo", ctypes.c_uint32),
        ("bucket_hi", ctypes.c_uint32),
        ("ms_send", ctypes.c_double),
        ("ms_exchange", ctypes.c_double),
        ("ms_receive", ctypes.c_double),
    ]


class DebugReport(ctypes.Structure):
    _fields_ = [("unwritten", ctypes.c_uint64), ("descents", ctypes.c_uint64), ("offset_diff", ctypes.c_uint64),
                ("multiset_diff", ctypes.c_uint64)]


class PotgHeader(ctypes.Structure):
    _fields_ = [
        ("version", ctypes.c_uint32),
        ("id_width", ctypes.c_uint32),
        ("orientation", ctypes.c_uint32),
        ("pad", ctypes.c_uint32),
        ("num_vertices", ctypes.c_uint64),
        ("num_edges", ctypes.c_uint64),
    ]


ABI_VERSION = 4  # include/gt.h GT_ABI_VERSION
_u64, _i64, _int, _vp = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
_stats_p = ctypes.POINTER(GtStats)
_hdr_p = ctypes.POINTER(PotgHeader)
_u64p = ctypes.POINTER(_u64)

# name -> (restype, argtypes); must match include/gt.h exactly
SYMBOLS = {
    "gt_abi_version": (_int, []),
    "gt_last_error": (ctypes.c_char_p, []),
    "gt_workspace_size": (_int, [_u64, _u64, ctypes.POINTER(_u64)]),
    "gt_transpose": (_int, [_vp, _vp, _u64, _u64, _vp, _vp, _vp, _u64, _vp, _stats_p]),
    "gt_transpose_host": (_int, [_vp, _vp, _u64, _u64, _vp, _vp, _int, _stats_p]),
    "gt_transpose_host_many": (_int, [_int, _vp, _vp, _vp, _vp, _vp, _vp, _int, _stats_p]),
    "gt_prefix_sum": (_int, [_vp, _u64, _vp, _vp]),
    "gt_edge_balanced_bounds": (_int, [_vp, _u64, _i64, _vp]),
    "gt_selftest_rank_order": (_int, [_u64, ctypes.POINTER(_u64)]),
    "gt_set_rank_mode": (_int, [_int]),
    "gt_set_config": (_int, [ctypes.POINTER(GtConfig)]),
    "gt_get_config": (_int, [ctypes.POINTER(GtConfig)]),
    "gt_transpose_status": (_int, [_vp, ctypes.POINTER(_int)]),
    "gt_release_workspace": (_int, []),
    "gt_shard_geometry": (_int, [_u64, _u64, ctypes.POINTER(ShardGeom)]),
    "gt_shard_send": (_int, [_vp, _vp, _u64, _u64, _u64, _u64, _vp, _vp, _vp, _vp]),
    "gt_shard_receive": (_int, [_vp, _vp, _vp, _int, _u64, _u64, ctypes.c_uint32, ctypes.c_uint32, _u64, _u64, _vp,
                                _vp, _vp, _stats_p]),
    "gt_shard_owners": (_int, [_vp, ctypes.c_uint32, _int, _vp]),
    "gt_shard_workspace_size": (_int, [_u64, _u64, _u64, ctypes.c_uint32, _int, _u64, _u64p, _u64p]),
    "gt_multi_unique_id": (_int, [_vp]),
    "gt_multi_comm_init": (_int, [_vp, _int, _int, ctypes.POINTER(_vp)]),
    "gt_multi_comm_destroy": (_int, [_vp]),
    "gt_transpose_multi": (_int, [_vp, _int, _int, _vp, _vp, _u64, _u64, _u64, _u64, _vp, _vp, _u64,
                                  ctypes.POINTER(MultiInfo), _vp]),
    "gt_gen_rmat": (_int, [_u64, _u64, _u64, _int, _vp, _vp, _vp]),
    "gt_gen_er": (_int, [_u64, _u64, _u64, _vp, _vp, _vp]),
    "gt_gen_rmat_csr": (_int, [_u64, _u64, _u64, _int, _vp, _vp, _vp]),
    "gt_gen_web_degrees": (_int, [_u64, _u64, _vp, ctypes.c_uint32, ctypes.c_uint32, _vp, _u64p, _vp]),
    "gt_gen_web_edges": (_int, [_u64, _u64, _vp, _vp, ctypes.c_uint32, _vp, ctypes.c_uint32, ctypes.c_uint32, _vp, _vp,
                                _vp]),
    "gt_build_csr": (_int, [_vp, _vp, _u64, _u64, _vp, _vp, _vp]),
    "gt_sort_lists": (_int, [_vp, _vp, _u64, _u64, _vp, _vp]),
    "gt_verify_transpose": (_int, [_vp, _vp, _u64, _u64, _vp, _vp, _vp]),
    "gt_debug_check": (_int, [_vp, _vp, _u64, _u64, _vp, _vp, ctypes.POINTER(DebugReport), _vp]),
    "gt_first_diff_u64": (_int, [_vp, _vp, _u64, _u64p, _vp]),
    "gt_first_diff_u32": (_int, [_vp, _vp, _u64, _u64p, _vp]),
    "gt_in_degree_offsets": (_int, [_vp, _u64, _u64, _vp, _vp]),
    "gt_first_diff_lists": (_int, [_vp, _vp, _vp, _vp, _vp, _u64, _u64p, _vp]),
    "gt_sample_hdv": (_int, [_vp, _u64, _u64, _u64, _u64, _u64, _int, _vp, _u64p, _vp]),
    "gt_hdv_table_build": (_int, [_vp, _u64, _u64, _int, _vp, _vp, _vp]),
    "gt_hdv_lookup": (_int, [_vp, _vp, _u64, _int, _vp, _u64, _vp, _vp]),
    "gt_coverage_exact": (_int, [_vp, _vp, _u64, _int, _vp, _u64, _u64p, _vp]),
    "gt_potg_read_header": (_int, [ctypes.c_char_p, _hdr_p, _u64p]),
    "gt_potg_read": (_int, [ctypes.c_char_p, _hdr_p, _vp, _vp, _vp, _u64p]),
    "gt_potg_write": (_int, [ctypes.c_char_p, _vp, _vp, _u64, _u64, _int, _int, _vp]),
}

_lock = threading.Lock()
_lib = None
_load_error: str | None = None


def load():
    """Load libgt.so once; raise GpuUnavailableError when it is missing."""
    global _lib, _load_error
    with _lock:
        if _lib is not None:
            return _lib
        path = os.environ.get("GT_LIBRARY", str(LIB_PATH))
        try:
            handle = ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
        except OSError as exc:
            _load_error = f"cannot load {path}: {exc} (run __graft_entry__.build())"
            raise GpuUnavailableError(_load_error) from None
        for name, (res, args) in SYMBOLS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.gt_abi_version() != ABI_VERSION:
            raise GpuUnavailableError("libgt.so ABI version mismatch")
        _lib = handle
        return _lib


class _LazyLib:
    def __getattr__(self, name):
        return getattr(load(), name)


lib = _LazyLib()


def check(rc: int, what: str) -> None:
    """Map a GT_* return code to the reference's exception types."""
    if rc == GT_OK:
        return
    msg = lib.gt_last_error().decode(errors="replace")
    text = f"{what}: {msg}"
    if rc == GT_EINVAL:
        raise ValueError(text)
    if rc == GT_EOVERFLOW:
        raise CounterOverflowError(msg)
    if rc == GT_ENOMEM:
        raise MemoryError(text)
    if rc == GT_ENODEV:
        raise GpuUnavailableError(text)
    if rc == GT_EIO:
        raise OSError(msg)
    raise RuntimeError(text)


def footprint_error(required: int, limit: int) -> FootprintError:
    return FootprintError(required, limit)
