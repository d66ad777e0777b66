"""Single-call gt_transpose_host on C3 (pinned host buffers) for several
source-chunk / bucket-group counts of the pipelined call, plus the serial call
(stats requested).  Prints ms per call; the PCIe floor is H2D + D2H."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import ctypes  # noqa: E402

from paper_2501_06872_b200 import _lib, gen, pipeline_config  # noqa: E402

cfg = gen.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
off_d, edg_d = gen.generate_device(cfg)
V, E = cfg.num_vertices, cfg.num_edges
h_off = off_d.cpu().pin_memory()
h_edg = edg_d.cpu().pin_memory()
del off_d, edg_d
torch.cuda.empty_cache()
h_toff = torch.empty(V + 1, dtype=torch.int64).pin_memory()
h_tedg = torch.empty(E, dtype=torch.int32).pin_memory()
out = (h_toff.numpy().view(np.uint64), h_tedg.numpy().view(np.uint32))
ref = None


def call(stats=None):
    rc = _lib.lib.gt_transpose_host(ctypes.c_void_p(h_off.data_ptr()), ctypes.c_void_p(h_edg.data_ptr()), V, E,
                                    ctypes.c_void_p(h_toff.data_ptr()), ctypes.c_void_p(h_tedg.data_ptr()), 0, stats)
    _lib.check(rc, "gt_transpose_host")


for chunks, groups in [(-1, 0), (0, 0), (8, 16), (16, 16)]:
    with pipeline_config(host_chunks=chunks, host_groups=groups, experiment=256):
        call()
        if ref is None:
            ref = (out[0].copy(), out[1].copy())
        else:
            assert np.array_equal(out[0], ref[0]) and np.array_equal(out[1], ref[1])
        ts = []
        for _ in range(4):
            t = time.perf_counter()
            call()
            ts.append(time.perf_counter() - t)
    print(f"chunks {chunks} groups {groups}: {min(ts) * 1e3:.1f} ms (median {sorted(ts)[2] * 1e3:.1f})", flush=True)
st = _lib.GtStats()
call(ctypes.byref(st))
assert np.array_equal(out[0], ref[0]) and np.array_equal(out[1], ref[1])
print(f"stats: total {st.ms_total:.2f} step1 {st.ms_step1:.2f} step2 {st.ms_step2:.2f} step3 {st.ms_step3:.2f} ms")
