"""PCIe copy rates on the GPU box (pinned host buffers): H2D, D2H, both at once,
and chunked — the floor of the single-call end-to-end leg."""
import time

import torch

n = 2_281_701_384 // 4
h_in = torch.empty(n, dtype=torch.int32).pin_memory()
h_out = torch.empty(n, dtype=torch.int32).pin_memory()
d_a = torch.empty(n, dtype=torch.int32, device="cuda")
d_b = torch.empty(n, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best * 1e3


gb = n * 4 / 1e9
t = timed(lambda: d_a.copy_(h_in, non_blocking=True))
print(f"H2D {gb:.2f} GB: {t:.1f} ms = {gb / t * 1e3:.1f} GB/s")
t = timed(lambda: h_out.copy_(d_b, non_blocking=True))
print(f"D2H {gb:.2f} GB: {t:.1f} ms = {gb / t * 1e3:.1f} GB/s")


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


t = timed(both)
print(f"H2D || D2H {gb:.2f} GB each: {t:.1f} ms")
for chunks in (4, 16):
    c = n // chunks

    def chunked():
        for i in range(chunks):
            d_a[i * c:(i + 1) * c].copy_(h_in[i * c:(i + 1) * c], non_blocking=True)

    t = timed(chunked)
    print(f"H2D in {chunks} chunks: {t:.1f} ms = {gb / t * 1e3:.1f} GB/s")
