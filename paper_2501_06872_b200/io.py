"""POTG graph files straight to / from device memory, with the reference's API.

Mirrors ``potra.io`` (pkg/src/potra/io.py): ``load_graph(path, format)``,
``store_graph(g, path)``, ``MAGIC``, ``HEADER_SIZE``, and the same
``GraphFormatError`` messages and byte offsets.  The binary format is read and
written by libgt.so (``gt_potg_read_header`` / ``gt_potg_read`` /
``gt_potg_write``): the file is streamed through pinned buffers into HBM and
its checks (offsets[0] == 0, monotone offsets, offsets[-1] == E, IDs < V) run
on the device.  ``load_graph_device`` / ``store_graph_device`` keep the graph
on the GPU; ``transpose_file`` is the ``potra transpose --algo gpu`` seam
(cli.py:272-325): file -> HBM -> transpose -> file.

The edge-list text format is host-side parsing (io.py:117-143) and is
restated with numpy.
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import GraphFormatError
from .graph import CsrGraph, edge_id_dtype

__all__ = [
    "MAGIC",
    "HEADER_SIZE",
    "DeviceGraph",
    "read_header",
    "load_graph",
    "load_graph_device",
    "store_graph",
    "store_graph_device",
    "transpose_file",
]

MAGIC = b"POTG"
HEADER_SIZE = 24
_ORIENT_CODE = {"CSR": 0, "CSC": 1}
_ORIENT_NAME = {0: "CSR", 1: "CSC"}


@dataclass
class DeviceGraph:
    """A graph resident in device memory: ``offsets`` int64[V+1] (uint64 bits),
    ``edges`` int32[E] (uint32 bits) or int64[E] when V > 2^32."""

    num_vertices: int
    num_edges: int
    offsets: object
    edges: object
    orientation: str = "CSR"

    def to_host(self) -> CsrGraph:
        off = self.offsets.cpu().numpy().view(np.uint64)
        e = self.edges.cpu().numpy()
        e = e.view(np.uint32) if e.dtype == np.int32 else e.view(np.uint64)
        return CsrGraph(self.num_vertices, self.num_edges, off, e, self.orientation)


def _path_bytes(path) -> bytes:
    return os.fsencode(os.fspath(path))


def _raise_format(rc: int, err_off: ctypes.c_uint64, what: str):
    if rc == _lib.GT_EFORMAT:
        raise GraphFormatError(_lib.lib.gt_last_error().decode(errors="replace"), byte_offset=int(err_off.value))
    _lib.check(rc, what)


def read_header(path) -> _lib.PotgHeader:
    """Parse and check the 24-byte header and the file length (io.py:54-84).
    Host only; no GPU needed."""
    h = _lib.PotgHeader()
    err = ctypes.c_uint64(0)
    rc = _lib.load().gt_potg_read_header(_path_bytes(path), ctypes.byref(h), ctypes.byref(err))
    if rc:
        _raise_format(rc, err, "gt_potg_read_header")
    return h


def load_graph_device(path, device=None, stream=None) -> DeviceGraph:
    """Read a POTG file into device memory, checked on the device."""
    from .transpose import _stream_handle, _torch

    torch = _torch()
    h = read_header(path)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    V, E, w = int(h.num_vertices), int(h.num_edges), int(h.id_width)
    off = torch.empty(V + 1, dtype=torch.int64, device=dev)
    edg = torch.empty(E, dtype=torch.int32 if w == 4 else torch.int64, device=dev)
    err = ctypes.c_uint64(0)
    with torch.cuda.device(dev):
        rc = _lib.lib.gt_potg_read(_path_bytes(path), ctypes.byref(h), ctypes.c_void_p(off.data_ptr()),
                                   ctypes.c_void_p(edg.data_ptr() if E else 0), _stream_handle(torch, stream),
                                   ctypes.byref(err))
    if rc:
        _raise_format(rc, err, "gt_potg_read")
    return DeviceGraph(V, E, off, edg, _ORIENT_NAME[int(h.orientation)])


def store_graph_device(g: DeviceGraph, path, stream=None) -> None:
    """Write a device-resident graph in the binary format (store_graph, io.py:28-38)."""
    from .transpose import _stream_handle, _torch

    torch = _torch()
    V, E = int(g.num_vertices), int(g.num_edges)
    w = edge_id_dtype(V).itemsize
    if g.edges.element_size() != w:
        raise ValueError(f"edges must be {w}-byte IDs for {V} vertices")
    with torch.cuda.device(g.offsets.device):
        rc = _lib.lib.gt_potg_write(_path_bytes(path), ctypes.c_void_p(g.offsets.data_ptr()),
                                    ctypes.c_void_p(g.edges.data_ptr() if E else 0), V, E,
                                    _ORIENT_CODE[g.orientation], w, _stream_handle(torch, stream))
    _lib.check(rc, "gt_potg_write")


def load_graph(path, format: str = "binary") -> CsrGraph:
    """Read a graph file; format is "binary" or "edge-list-text" (io.py:41-47).
    The binary path goes through device memory (GPU required)."""
    if format == "binary":
        return load_graph_device(path).to_host()
    if format == "edge-list-text":
        return _load_text(path)
    raise ValueError(f"unknown format {format!r}")


def store_graph(g, path) -> None:
    """Write g in the binary format; load_graph round-trips bit-for-bit.
    Host CsrGraph -> file via device memory (GPU required); a DeviceGraph is
    written directly."""
    if isinstance(g, DeviceGraph):
        store_graph_device(g, path)
        return
    from .transpose import _torch

    torch = _torch()
    dt = edge_id_dtype(g.num_vertices)
    off = torch.from_numpy(np.ascontiguousarray(g.offsets, dtype=np.uint64).view(np.int64)).cuda()
    e = np.ascontiguousarray(g.edges, dtype=dt)
    edg = torch.from_numpy(e.view(np.int32 if dt.itemsize == 4 else np.int64)).cuda()
    store_graph_device(DeviceGraph(int(g.num_vertices), int(g.num_edges), off, edg, g.orientation), path)


def _load_text(path) -> CsrGraph:
    """Edge-list text is host-side parsing outside this package's scope (the
    GPU path starts at a CSR in memory or a POTG file).  It is delegated to the
    reference's own reader (potra.io.load_graph, io.py:117-143) when potra is
    importable."""
    try:
        from potra import io as _potra_io  # the reference package, when installed
    except ImportError:
        raise NotImplementedError(
            "edge-list-text input is read by the reference's potra.io.load_graph; "
            "potra is not importable here (convert to the binary POTG format first)") from None
    g = _potra_io.load_graph(path, format="edge-list-text")
    return CsrGraph(int(g.num_vertices), int(g.num_edges), np.asarray(g.offsets, dtype=np.uint64),
                    np.asarray(g.edges, dtype=np.uint32))


def transpose_file(in_path, out_path, *, sort: bool = False, device=None) -> dict:
    """The ``potra transpose --algo gpu`` seam: POTG file -> HBM -> transpose ->
    POTG file, never materialising the graph on the host.  Returns phase
    times in seconds ({"read", "step1", "step2", "step3", "write"});
    ``sort`` is accepted for CLI parity (the output is already sorted)."""
    from .transpose import _torch, transpose_device

    torch = _torch()
    t0 = time.perf_counter()
    g = load_graph_device(in_path, device=device)
    if g.edges.dtype != torch.int32:
        raise ValueError("only 32-bit neighbour IDs (num_vertices <= 2^32) are supported")
    torch.cuda.synchronize(g.offsets.device)
    t1 = time.perf_counter()
    t_off, t_edg, st = transpose_device(g.offsets, g.edges, g.num_vertices, want_stats=True)
    flip = {"CSR": "CSC", "CSC": "CSR"}[g.orientation]
    t2 = time.perf_counter()
    store_graph_device(DeviceGraph(g.num_vertices, g.num_edges, t_off, t_edg, flip), out_path)
    t3 = time.perf_counter()
    return {
        "read": t1 - t0,
        "step1": st.ms_step1 / 1e3,
        "step2": st.ms_step2 / 1e3,
        "step3": st.ms_step3 / 1e3,
        "write": t3 - t2,
        "aux_footprint_bytes": int(st.workspace_bytes),
    }
