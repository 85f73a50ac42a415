"""Per-tile stage timeline of fir_tc (diagnostics): python tools/trace_fir.py [cfg2] [seconds]
Needs a -DFT_TRACE build of the library (the product build compiles the stamps out):
    python tools/lb_variants.py build "ftrace%wp_fir_tc.cu=-DFT_TRACE"
    WP_LIB=tools/variants/ftrace/libwpb200.so python tools/trace_fir.py cfg2
Events (ns, %globaltimer): 0 window copy issued, 1 converters see the window, 2 window in registers
(buffer freed), 3 operand buffer free, 4 operands written, 5 MMA start, 6 MMAs issued (commit),
7 epilogue has the accumulator, 8 accumulator read (TMEM freed), 9 stores issued."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402
import paper_2504_08624_b200 as wp  # noqa: E402
from paper_2504_08624_b200 import _native, engine  # noqa: E402

EV = 16
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = bench.CONFIGS[name]
C, fs = cfg["C"], cfg["fs"]
dur = float(sys.argv[2]) if len(sys.argv) > 2 else cfg["dur"]
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
if len(stages) == 1 and hasattr(stages[0], "taps"):
    # output check: fp64 direct convolution of every channel (torch conv1d on the device)
    h = torch.tensor(np.asarray(stages[0].taps, dtype=np.float64), device="cuda")
    xd = torch.nn.functional.pad(x.double(), (len(h) - 1, 0)).unsqueeze(1)
    ref = torch.nn.functional.conv1d(xd, h.flip(0).view(1, 1, -1)).squeeze(1)
    err = ((y.double() - ref).abs().max() / ref.abs().max()).item()
    print("max err / peak vs fp64 conv: %.2e %s" % (err, "OK" if err < 1e-5 else "FAIL"))
_native.set_trace(tr.data_ptr(), tr.numel())
plan.execute(x.data_ptr(), y.data_ptr(), C, N, N, N, ws.data_ptr(), nb, st)
torch.cuda.synchronize()
_native.set_trace(0, 0)
t = tr.cpu().numpy().astype(np.float64).reshape(tiles, EV)
if not (t > 0).any():
    print("(no stamps: not a -DFT_TRACE build)")
    sys.exit(0)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, np.nan)
names = ["copy", "inful", "inreg", "opfree", "opful", "mma0", "mma1", "accful", "accrd", "stored"]
print("span us: %.1f   first tile copy issued at %.2f us, last store issued at %.2f us"
      % (np.nanmax(t[:, 9]) / 1e3, np.nanmin(t[:, 0]) / 1e3, np.nanmax(t[:, 9]) / 1e3))
for a, b in [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (6, 7), (7, 8), (8, 9), (0, 9)]:
    d = (t[:, b] - t[:, a]) / 1e3
    print(f"{names[a]:>6} -> {names[b]:<6} median {np.nanmedian(d):7.2f} us  p90 {np.nanpercentile(d, 90):7.2f}")
G = min(tiles, 148)
for ev in range(10):
    per = []
    for b in range(G):
        col = t[b::G, ev]
        col = col[~np.isnan(col)]
        if col.size > 2:
            per.append(np.median(np.diff(col)))
    print(f"per-CTA period of {names[ev]:>6}: median {np.median(per) / 1e3:.2f} us")
# ramp: when does each CTA's first tile finish, and the last
first_done = np.array([np.nanmin(t[b::G, 9]) for b in range(G)]) / 1e3
last_done = np.array([np.nanmax(t[b::G, 9]) for b in range(G)]) / 1e3
print("first tile stored: median %.2f us; CTA finish: min %.2f median %.2f max %.2f us"
      % (np.median(first_done), last_done.min(), np.median(last_done), last_done.max()))
