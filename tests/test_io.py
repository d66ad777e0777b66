"""POTG file format, edge-list text, and the CLI seam — against results the
reference produced for the same bytes (tests/golden/make_io_golden.py).

CPU tests: header parsing/validation (host-only C entry point); edge-list text
is delegated to the reference's reader.  GPU tests: device reads (data checks run on the device), writes,
round trips, and file -> HBM -> transpose -> file through the CLI."""

import json

import numpy as np
import pytest

from conftest import GOLDEN

CASES = json.loads((GOLDEN / "io_cases.json").read_text())
BY_NAME = {c["name"]: c for c in CASES}
HEADER_ERRORS = [c for c in CASES if c["format"] == "binary" and not c["ok"] and
                 c["message"].startswith(("malformed header", "truncated"))]
DATA_ERRORS = [c for c in CASES if c["format"] == "binary" and not c["ok"] and c not in HEADER_ERRORS]
VALID = [c for c in CASES if c["format"] == "binary" and c["ok"] and "offsets" in c]
TEXT = [c for c in CASES if c["format"] == "edge-list-text"]


def write(tmp_path, case):
    p = tmp_path / f"{case['name']}.bin"
    p.write_bytes(bytes.fromhex(case["hex"]))
    return p


def test_fixture_coverage():
    assert len(HEADER_ERRORS) >= 9 and len(DATA_ERRORS) >= 6 and len(VALID) >= 5 and len(TEXT) >= 5


@pytest.mark.parametrize("case", HEADER_ERRORS, ids=lambda c: c["name"])
def test_header_errors_match_reference(tmp_path, case):
    from paper_2501_06872_b200.errors import GraphFormatError
    from paper_2501_06872_b200.io import read_header

    with pytest.raises(GraphFormatError) as ei:
        read_header(write(tmp_path, case))
    assert str(ei.value) == case["message"]
    assert ei.value.byte_offset == case["byte_offset"]


@pytest.mark.parametrize("case", VALID + DATA_ERRORS, ids=lambda c: c["name"])
def test_header_of_files_with_valid_headers(tmp_path, case):
    from paper_2501_06872_b200.io import read_header

    data = bytes.fromhex(case["hex"])
    h = read_header(write(tmp_path, case))
    assert h.version == data[4] and h.id_width == data[5] and h.orientation == data[6]
    assert h.num_vertices == int.from_bytes(data[8:16], "little")
    assert h.num_edges == int.from_bytes(data[16:24], "little")


def test_missing_file_is_oserror(tmp_path):
    from paper_2501_06872_b200.io import read_header

    with pytest.raises(OSError):
        read_header(tmp_path / "does_not_exist.potg")


def test_edge_list_text_is_delegated(tmp_path):
    """Text parsing is the reference's own (potra.io); without potra it is refused."""
    import importlib.util

    from paper_2501_06872_b200.io import load_graph

    p = write(tmp_path, TEXT[0])
    if importlib.util.find_spec("potra") is None:
        with pytest.raises(NotImplementedError):
            load_graph(p, format="edge-list-text")


def test_unknown_format_is_valueerror(tmp_path):
    from paper_2501_06872_b200.io import load_graph

    with pytest.raises(ValueError):
        load_graph(tmp_path / "x", format="xml")


def test_cli_rejects_bad_threads(tmp_path, capsys):
    from paper_2501_06872_b200.cli import main

    assert main(["transpose", "--algo", "gpu", "--threads", "0", "--in", "a", "--out", "b"]) == 2
    with pytest.raises(SystemExit):
        main(["transpose", "--algo", "atomic", "--in", "a", "--out", "b"])


# ----------------------------------------------------------------- GPU


@pytest.mark.gpu
@pytest.mark.parametrize("case", VALID, ids=lambda c: c["name"])
def test_device_read_matches_reference(tmp_path, case):
    from paper_2501_06872_b200.io import load_graph

    g = load_graph(write(tmp_path, case))
    assert g.num_vertices == case["nv"] and g.num_edges == case["ne"]
    assert g.offsets.dtype == np.uint64 and g.offsets.tolist() == case["offsets"]
    assert str(g.edges.dtype) == case["edges_dtype"] and g.edges.tolist() == case["edges"]
    assert g.orientation == case["orientation"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", DATA_ERRORS, ids=lambda c: c["name"])
def test_device_data_checks_match_reference(tmp_path, case):
    from paper_2501_06872_b200.errors import GraphFormatError
    from paper_2501_06872_b200.io import load_graph

    with pytest.raises(GraphFormatError) as ei:
        load_graph(write(tmp_path, case))
    assert str(ei.value) == case["message"]
    assert ei.value.byte_offset == case["byte_offset"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", VALID, ids=lambda c: c["name"])
def test_store_is_byte_identical(tmp_path, case):
    from paper_2501_06872_b200.io import load_graph, store_graph

    src = write(tmp_path, case)
    out = tmp_path / "out.potg"
    g = load_graph(src)
    store_graph(g, out)
    data = src.read_bytes()
    if data[5] == (4 if case["nv"] <= 2**32 else 8):
        assert out.read_bytes() == data
    else:  # store_graph writes the width forced by V (io.py:31-33), as the reference does
        assert out.read_bytes()[5] == 4
        h = load_graph(out)
        assert h.offsets.tolist() == case["offsets"] and h.edges.tolist() == case["edges"]


@pytest.mark.gpu
def test_transpose_file_and_cli_equal_reference_bytes(tmp_path):
    from paper_2501_06872_b200.cli import main
    from paper_2501_06872_b200.io import transpose_file

    src = write(tmp_path, BY_NAME["random_300"])
    want = bytes.fromhex(BY_NAME["random_300_transposed"]["hex"])
    out = tmp_path / "t.potg"
    phases = transpose_file(src, out)
    assert out.read_bytes() == want and phases["step1"] >= 0
    out2, rep = tmp_path / "t2.potg", tmp_path / "r.json"
    assert main(["transpose", "--algo", "gpu", "--in", str(src), "--out", str(out2), "--report", str(rep)]) == 0
    assert out2.read_bytes() == want
    r = json.loads(rep.read_text())
    assert r["schema_version"] == 1 and r["sorted"] is True and set(r["phase_times"]) >= {"step1", "step2", "step3"}


@pytest.mark.gpu
def test_large_roundtrip_through_staging(tmp_path):
    """More than one pinned staging buffer (64 MiB) in each direction."""
    import torch

    from paper_2501_06872_b200 import gen
    from paper_2501_06872_b200.io import DeviceGraph, load_graph_device, store_graph_device

    off, edg = gen.generate_device(gen.CONFIGS["C1"], torch.device("cuda"))
    # C1 repeated to exceed 64 MiB of edges: 20 disjoint copies side by side
    V, E = off.numel() - 1, edg.numel()
    reps = 20
    offs = torch.cat([off[:-1] + i * E for i in range(reps)] + [off[-1:] + (reps - 1) * E])
    edges = torch.cat([edg + i * V for i in range(reps)])
    g = DeviceGraph(V * reps, E * reps, offs, edges.to(torch.int32))
    p = tmp_path / "big.potg"
    store_graph_device(g, p)
    assert p.stat().st_size == 24 + (V * reps + 1) * 8 + E * reps * 4
    h = load_graph_device(p)
    assert torch.equal(h.offsets, offs) and torch.equal(h.edges, g.edges)
