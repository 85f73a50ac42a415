"""Replay a tools/stress_random.py failure (gpurun_out/stress_fail_*.npz) through the
device path (all channels, one call) and channel by channel, printing each pass's
kernel and the error vs the float64 oracle: python tools/stress_replay.py <npz>"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import oracle  # noqa: E402
import paper_2504_08624_b200 as wp  # noqa: E402
from paper_2504_08624_b200 import engine  # noqa: E402

d = np.load(sys.argv[1])
x = d["x"].astype(np.float32)
fs = 48000
stages = []
for k in sorted((k for k in d.keys() if k.startswith("s")), key=lambda k: int(k[1:].split("_")[0])):
    v = d[k]
    if k.endswith("IirFilter"):
        stages.append(wp.IirFilter.from_sections([tuple(r) for r in v], fs))
    elif k.endswith("FirFilter"):
        stages.append(wp.FirFilter.from_taps(v, fs))
    elif k.endswith("Gain"):
        stages.append(wp.Gain(float(v[0])))
bound = wp.Chain(stages).bind(fs).stages
ref = oracle.pipe(x.astype(np.float64), bound, oracle.default_threads())
C, N = x.shape
plan = engine.plan_for(bound, device=0)
for label, chans in [("all channels", list(range(C))), ("one channel", [0]), ("two channels", [0, 1])]:
    print(label, plan.describe_for(len(chans), N))
    y = wp.pipe(wp.Wave.from_tensor(torch.from_numpy(x[chans]).cuda(), fs), wp.Chain(stages)).tensor().cpu().numpy()
    print("   err", oracle.parity_error(y.astype(np.float64), ref[chans]))
# per stage alone and per section alone (same input): which part carries the error
xt = torch.from_numpy(x).cuda()
for i, st in enumerate(stages):
    b1 = wp.Chain([st]).bind(fs).stages
    y1 = wp.pipe(wp.Wave.from_tensor(xt, fs), wp.Chain([st])).tensor().cpu().numpy()
    r1 = oracle.pipe(x.astype(np.float64), b1, oracle.default_threads())
    print(f"stage {i} alone: err {oracle.parity_error(y1.astype(np.float64), r1):.2e}", engine.plan_for(b1, device=0).describe_for(C, N)[0][:40])
    if hasattr(st, "sections"):
        for k, row in enumerate(st.sos_rows()):
            f = wp.IirFilter.from_sections([tuple(row)], fs)
            y2 = wp.pipe(wp.Wave.from_tensor(xt, fs), wp.Chain([f])).tensor().cpu().numpy()
            r2 = oracle.iir_cascade(row[None, :], x.astype(np.float64))
            print(f"   section {k} {np.round(row, 4)}: err {oracle.parity_error(y2.astype(np.float64), r2):.2e}")
