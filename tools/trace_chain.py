"""Per-tile stage timeline of the tensor-core chain kernel (diagnostics).

python tools/trace_chain.py [cfg3|cfg5|cfg1] -> prints median stage latencies
and the per-CTA tile period. Events (ns, %globaltimer) per tile:
 0 converter start     1 operands ready (OP_FULL)   2 MMA issue start
 3 scan start (e ready) 4 scan done (aggregate)     5 look-back start
 6 look-back done       7 epilogue start            8 epilogue done
"""

from __future__ import annotations

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import bench  # noqa: E402
import paper_2504_08624_b200 as wp  # noqa: E402
from paper_2504_08624_b200 import _native, engine  # noqa: E402

EV = 12


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    cfg = bench.CONFIGS[name]
    C, fs = cfg["C"], cfg["fs"]
    dur = float(sys.argv[2]) if len(sys.argv) > 2 else cfg["dur"]
    N = int(round(dur * fs))
    stages = wp.Chain(bench.stages_for(name, wp)).bind(fs).stages
    w = wp.white_noise(dur, C, fs, seed=42)
    x = w.tensor()
    y = torch.empty_like(x)
    plan = engine.plan_for(stages, device=0)
    print(plan.describe())
    nb = plan.workspace_bytes(C, N)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    tiles = C * ((N + 8191) // 8192)
    tr = torch.zeros(tiles * EV, dtype=torch.int64, device="cuda")
    for _ in range(3):
        plan.execute(x.data_ptr(), y.data_ptr(), C, N, N, N, ws.data_ptr(), nb, st)
    torch.cuda.synchronize()
    _native.set_trace(tr.data_ptr(), tr.numel())
    plan.execute(x.data_ptr(), y.data_ptr(), C, N, N, N, ws.data_ptr(), nb, st)
    torch.cuda.synchronize()
    _native.set_trace(0, 0)
    t = tr.view(tiles, EV).cpu().numpy().astype(np.float64)
    t0 = t[t > 0].min()
    t = np.where(t > 0, t - t0, np.nan)
    names = ["conv", "opfull", "mma", "scan0", "scan1", "lb0", "lb1", "epi0", "epi1", "scanSB", "epiCV", "lbspin"]
    print("kernel span us: %.1f" % (np.nanmax(t[:, 8]) / 1e3))
    for a, b in [(0, 1), (1, 2), (2, 3), (3, 9), (9, 4), (4, 5), (5, 11), (11, 6), (6, 7), (7, 10), (6, 10),
                 (10, 8), (0, 8)]:
        d = (t[:, b] - t[:, a]) / 1e3
        print(f"{names[a]:>6} -> {names[b]:<6} median {np.nanmedian(d):7.2f} us  p90 {np.nanpercentile(d, 90):7.2f}")
    G = min(tiles, 148)
    for ev in (0, 2, 3, 5, 7, 8):
        per = []
        for b in range(G):
            col = t[b::G, ev]
            col = col[~np.isnan(col)]
            if col.size > 2:
                per.append(np.median(np.diff(col)))
        print(f"per-CTA period of {names[ev]:>6}: median {np.median(per) / 1e3:.2f} us")


if __name__ == "__main__":
    main()
