"""End-to-end (pinned host -> device -> host) throughput of cfg3 by channel-block count,
next to the raw PCIe copy rates on the box: python tools/e2e_blocks_probe.py"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402
import paper_2504_08624_b200 as wp  # noqa: E402
from paper_2504_08624_b200 import engine  # noqa: E402

cfg = bench.CONFIGS["cfg3"]
C, fs = cfg["C"], cfg["fs"]
N = int(cfg["dur"] * fs)
hin = wp.white_noise(cfg["dur"], C, fs, seed=42).tensor().cpu().pin_memory()
hout = torch.empty_like(hin).pin_memory()
d = torch.empty_like(hin, device="cuda")
nb = hin.numel() * 4
for name, fn in [("h2d", lambda: d.copy_(hin, non_blocking=True)), ("d2h", lambda: hout.copy_(d, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    print(f"{name}: {5 * nb / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
s2 = torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    d.copy_(hin, non_blocking=True)
    with torch.cuda.stream(s2):
        hout.copy_(d, non_blocking=True)
torch.cuda.synchronize()
print(f"h2d || d2h: {5 * nb / (time.perf_counter() - t0) / 1e9:.1f} GB/s each way (both at once)")
lazy = wp.Wave.from_tensor(hin, fs) | wp.Chain(bench.stages_for("cfg3", wp))
ent = lazy._entries
for blocks in (4, 8, 16, 32):
    times = []
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        engine.stream_host_entries(ent, hin, hout, blocks=blocks)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    t = min(times[1:])
    print(f"blocks={blocks}: {C * N / t / 1e9:.2f} G ch-samples/s ({t * 1e3:.1f} ms)")
