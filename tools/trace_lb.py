"""Per-tile role timeline of chain_lb (diagnostics): python tools/trace_lb.py [cfg3|cfg5] [seconds]
Needs a -DLB_TRACE build of the library (the product build compiles the stamps out):
    python tools/lb_variants.py build traced=-DLB_TRACE
    WP_LIB=tools/variants/traced/libwpb200.so python tools/trace_lb.py cfg3
Without one only the untraced time per pass is printed.
Events (ns, %globaltimer): 0 converter start, 1 operands ready, 2 MMA start, 3 MMAs issued,
4 look-back start, 5 look-back done, 6 scan done (aggregate published, prefixes in the ring),
7 epilogue done, 8 scan start (MMAs complete), 9 epilogue has the carry, 10 epilogue has the prefixes,
11 epilogue state s_m ready, 12 scan work done (before the ring wait), 13 first TMEM chunk loaded."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402
import paper_2504_08624_b200 as wp  # noqa: E402
from paper_2504_08624_b200 import _native, engine  # noqa: E402

EV = 16
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
cfg = bench.CONFIGS[name]
C, fs = cfg["C"], cfg["fs"]
dur = float(sys.argv[2]) if len(sys.argv) > 2 else (cfg["dur"] if name != "cfg5" else 20.0)
N = int(round(dur * fs))
stages = wp.Chain(bench.stages_for(name, wp)).bind(fs).stages
x = wp.white_noise(dur, C, fs, seed=42).tensor()
y = torch.empty_like(x)
plan = engine.plan_for(stages, device=0)
print(plan.describe_for(C, N))
nb = plan.workspace_bytes(C, N)
ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
tiles = C * ((N + 8191) // 8192)
tr = torch.zeros(tiles * EV, dtype=torch.int64, device="cuda")
for _ in range(3):
    plan.execute(x.data_ptr(), y.data_ptr(), C, N, N, N, ws.data_ptr(), nb, st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    plan.execute(x.data_ptr(), y.data_ptr(), C, N, N, N, ws.data_ptr(), nb, st)
e1.record()
torch.cuda.synchronize()
print("ms per pass (untraced): %.4f" % (e0.elapsed_time(e1) / 10))
_native.set_trace(tr.data_ptr(), tr.numel())
plan.execute(x.data_ptr(), y.data_ptr(), C, N, N, N, ws.data_ptr(), nb, st)
torch.cuda.synchronize()
_native.set_trace(0, 0)
t = tr.cpu().numpy().astype(np.float64).reshape(tiles, EV)
if not (t > 0).any():
    print("(no stamps: not a -DLB_TRACE build)")
    sys.exit(0)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, np.nan)
names = ["conv0", "opfull", "mma0", "mma1", "lb0", "lbdone", "scan1", "epi1", "scan0", "carry", "ring", "s_m",
         "scanw", "tm0", "-", "-"]
print("span us: %.1f" % (np.nanmax(t[:, 7]) / 1e3))
for a, b in [(0, 1), (1, 2), (2, 3), (3, 8), (8, 12), (12, 6), (6, 10), (4, 5), (6, 9), (5, 9), (9, 11),
             (11, 13), (13, 7), (2, 7), (0, 7)]:
    d = (t[:, b] - t[:, a]) / 1e3
    print(f"{names[a]:>6} -> {names[b]:<6} median {np.nanmedian(d):7.2f} us  p90 {np.nanpercentile(d, 90):7.2f}")
G = min(tiles, 148)
# gaps inside one role between consecutive local tiles of a CTA
for a, b, nm in [(7, 10, "epilogue: epi1(i) -> ring(i+1)"), (6, 8, "scan: scan1(i) -> scan0(i+1)"),
                 (1, 0, "conv: opfull(i) -> conv0(i+1)"), (3, 2, "mma: mma1(i) -> mma0(i+1)")]:
    g = []
    for bb in range(G):
        col_a, col_b = t[bb::G, a], t[bb::G, b]
        g.append(col_b[1:] - col_a[:-1])
    g = np.concatenate(g) / 1e3
    print(f"{nm:34s} median {np.nanmedian(g):6.2f} us  p90 {np.nanpercentile(g, 90):6.2f}")
for ev in range(EV):
    per = []
    for b in range(G):
        col = t[b::G, ev]
        col = col[~np.isnan(col)]
        if col.size > 2:
            per.append(np.median(np.diff(col)))
    print(f"per-CTA period of {names[ev]:>6}: median {np.median(per) / 1e3:.2f} us")
