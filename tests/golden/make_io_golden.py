"""Generate the POTG / text-format / verify_output golden fixtures from the
reference implementation (run in the build container, where /root/reference
is importable):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_io_golden.py

Writes tests/golden/io_cases.json and tests/golden/verify_cases.npz (+ .json).
The GPU tests compare this package's readers/writers/verifier with these
recorded reference results; nothing here is imported at test time.
"""

from __future__ import annotations

import json
import os
import struct
import tempfile
from pathlib import Path

import numpy as np

from potra import bench, graph, io
from potra.baselines import TransposeOutput
from potra.errors import GraphFormatError

HERE = Path(__file__).resolve().parent
HDR = struct.Struct("<4sBBBBQQ")


def potg_bytes(magic=b"POTG", version=1, width=4, orient=0, pad=0, nv=0, ne=0, offsets=(), edges=(), edge_dtype=None):
    b = HDR.pack(magic, version, width, orient, pad, nv, ne)
    b += np.asarray(offsets, dtype="<u8").tobytes()
    edt = edge_dtype or ("<u4" if width == 4 else "<u8")
    b += np.asarray(edges, dtype=edt).tobytes()
    return b


def run_reference(data: bytes, fmt="binary"):
    with tempfile.NamedTemporaryFile(delete=False, suffix=".potg" if fmt == "binary" else ".txt") as f:
        f.write(data)
        path = f.name
    try:
        g = io.load_graph(path, format=fmt)
        return {"ok": True, "nv": g.num_vertices, "ne": g.num_edges, "offsets": g.offsets.tolist(),
                "edges": g.edges.tolist(), "edges_dtype": str(g.edges.dtype), "orientation": g.orientation}
    except GraphFormatError as exc:
        return {"ok": False, "message": str(exc), "byte_offset": exc.byte_offset}
    finally:
        os.unlink(path)


def main():
    rng = np.random.default_rng(11)
    cases = []

    def add(name, data, fmt="binary"):
        cases.append({"name": name, "format": fmt, "hex": data.hex(), **run_reference(data, fmt)})

    # valid files
    add("empty_v0", potg_bytes(nv=0, ne=0, offsets=[0]))
    add("v17_e0", potg_bytes(nv=17, ne=0, offsets=[0] * 18))
    add("fig_csc", potg_bytes(orient=1, nv=4, ne=5, offsets=[0, 2, 3, 5, 5], edges=[1, 3, 0, 0, 2]))
    add("width8", potg_bytes(width=8, nv=3, ne=2, offsets=[0, 1, 1, 2], edges=[2, 0]))
    # header errors
    add("short_header", b"POTG\x01\x04")
    add("bad_magic", potg_bytes(magic=b"PQTG", nv=0, offsets=[0]))
    add("bad_magic_bin", potg_bytes(magic=b"\x00'\xff\n", nv=0, offsets=[0]))
    add("bad_version", potg_bytes(version=2, nv=0, offsets=[0]))
    add("bad_width", potg_bytes(width=3, nv=0, offsets=[0]))
    add("bad_orient", potg_bytes(orient=2, nv=0, offsets=[0]))
    add("width4_too_many_vertices", potg_bytes(nv=2**32 + 1, ne=0))
    add("truncated_offsets", potg_bytes(nv=5, ne=0, offsets=[0, 0, 0]))
    add("truncated_edges", potg_bytes(nv=2, ne=4, offsets=[0, 2, 4], edges=[1, 0, 1]))
    # data errors (checked on the device)
    add("offsets0_nonzero", potg_bytes(nv=2, ne=2, offsets=[1, 1, 2], edges=[0, 1]))
    add("nonmonotone", potg_bytes(nv=4, ne=3, offsets=[0, 2, 1, 3, 3], edges=[0, 1, 2]))
    add("nonmonotone_later", potg_bytes(nv=5, ne=4, offsets=[0, 1, 2, 4, 3, 4], edges=[0, 1, 2, 3]))
    add("last_mismatch", potg_bytes(nv=2, ne=3, offsets=[0, 1, 2], edges=[0, 1, 1]))
    add("edge_out_of_range", potg_bytes(nv=3, ne=4, offsets=[0, 2, 3, 4], edges=[0, 2, 3, 7]))
    add("edge_out_of_range_w8", potg_bytes(width=8, nv=3, ne=2, offsets=[0, 1, 2, 2], edges=[1, 5]))
    # a random valid graph
    nv, ne = 300, 2000
    src = rng.integers(0, nv, ne)
    dst = rng.integers(0, nv, ne)
    g = graph.CsrGraph.from_edge_pairs(src, dst, nv)
    with tempfile.NamedTemporaryFile(delete=False, suffix=".potg") as f:
        path = f.name
    io.store_graph(g, path)
    data = Path(path).read_bytes()
    io.store_graph(graph.transpose_oracle(g), path)
    data_t = Path(path).read_bytes()
    os.unlink(path)
    add("random_300", data)
    cases.append({"name": "random_300_transposed", "format": "binary", "hex": data_t.hex(), "ok": True,
                  "is_transpose_of": "random_300"})
    # text format
    add("text_ok", b"# comment\n0 1\n\n2 0\n1 1\n2 0\n", "edge-list-text")
    add("text_empty", b"# nothing\n\n", "edge-list-text")
    add("text_bad_fields", b"0 1\n1 2 3\n", "edge-list-text")
    add("text_non_integer", b"0 x\n", "edge-list-text")
    add("text_negative", b"0 1\n-1 2\n", "edge-list-text")
    (HERE / "io_cases.json").write_text(json.dumps(cases, indent=1))

    # verify_output reports of the reference on corrupted outputs
    nv, ne = 500, 6000
    src = rng.integers(0, nv, ne)
    dst = np.minimum((nv * rng.random(ne) ** 2).astype(np.int64), nv - 1)
    g = graph.CsrGraph.from_edge_pairs(src, dst, nv)
    t = graph.transpose_oracle(g)
    variants = {"exact": (t.offsets.copy(), t.edges.copy(), True)}
    e = t.edges.copy()
    e[4000] = (e[4000] + 1) % nv
    variants["edge_changed"] = (t.offsets.copy(), e, True)
    o = t.offsets.copy()
    o[200] += 1
    variants["offset_changed"] = (o, t.edges.copy(), True)
    e = t.edges.copy()  # scramble every list: same multisets, unsorted
    off = t.offsets.astype(np.int64)
    for v in range(nv):
        seg = e[off[v]:off[v + 1]]
        e[off[v]:off[v + 1]] = seg[rng.permutation(seg.size)]
    variants["scrambled_unsorted"] = (t.offsets.copy(), e, False)
    variants["scrambled_claimed_sorted"] = (t.offsets.copy(), e, True)
    arrays = {"in_offsets": g.offsets, "in_edges": g.edges}
    reports = {}
    for name, (vo, ve, srt) in variants.items():
        arrays[f"{name}_offsets"] = vo
        arrays[f"{name}_edges"] = ve
        out = TransposeOutput(graph=graph.CsrGraph(nv, ne, vo, ve, "CSC"), phase_times={}, aux_footprint_bytes=0,
                              method="x", sorted=srt, details={})
        rep = {}
        for mode in ("full-oracle", "multiset-sample"):
            for sv in (100_000, 37):
                r = bench.verify_output(g, out, mode=mode, seed=5, sample_vertices=sv)
                rep[f"{mode}/{sv}"] = {"passed": r.passed, "mismatch_vertex": r.mismatch_vertex, "message": r.message}
        reports[name] = {"sorted": srt, "reports": rep}
    np.savez_compressed(HERE / "verify_cases.npz", **arrays)
    (HERE / "verify_cases.json").write_text(json.dumps(reports, indent=1))
    print(f"{len(cases)} io cases, {len(reports)} verify variants")


if __name__ == "__main__":
    main()
