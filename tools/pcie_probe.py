"""Pinned host<->device copy bandwidth with 1..4 concurrent streams per direction (diagnostics)."""
import time

import torch

n = 737_280_000 // 4
h_in = torch.empty(n, dtype=torch.float32, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
d_in = torch.empty(n, dtype=torch.float32, device="cuda")
d_out = torch.empty(n, dtype=torch.float32, device="cuda")


def run(k, mode):
    st_in = [torch.cuda.Stream() for _ in range(k)]
    st_out = [torch.cuda.Stream() for _ in range(k)]
    chunks = 32
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for c in range(chunks):
        a, b = c * n // chunks, (c + 1) * n // chunks
        if mode in ("h2d", "bidir"):
            with torch.cuda.stream(st_in[c % k]):
                d_in[a:b].copy_(h_in[a:b], non_blocking=True)
        if mode in ("d2h", "bidir"):
            with torch.cuda.stream(st_out[c % k]):
                h_out[a:b].copy_(d_out[a:b], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    gb = n * 4 / 1e9
    print(f"{mode:6s} streams/dir={k}: {dt * 1e3:7.2f} ms, {gb / dt:6.1f} GB/s per direction")


for mode in ("h2d", "d2h", "bidir"):
    for k in (1, 2, 4):
        run(k, mode)
        run(k, mode)
