"""Re-run one random 6-section case of tools/six_section_probe.py several times:
determinism and the error around its worst sample (diagnostics)."""
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
sys.path.insert(0, os.path.join(HERE, "..", "tests"))
import oracle  # noqa: E402
import paper_2504_08624_b200 as wp  # noqa: E402
from conftest import random_stable_section  # noqa: E402
from paper_2504_08624_b200 import engine  # noqa: E402

target, seed = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(seed)
for i in range(target + 1):
    f = wp.IirFilter.from_sections([random_stable_section(rng) for _ in range(6)], 44100,
                                   overall_gain=float(rng.uniform(0.25, 2.0)))
    C, N = int(rng.integers(1, 13)), int(10 ** rng.uniform(4, 5.5))
    x = rng.standard_normal((C, N)).astype(np.float32)
ref = oracle.iir_cascade(f.sos_rows(), x.astype(np.float64))
print(engine.plan_for(wp.Chain([f]).bind(44100).stages, device=0).describe_for(C, N))
outs = []
for r in range(5):
    y = wp.pipe(wp.Wave.from_tensor(torch.from_numpy(x).cuda(), 44100), wp.Chain([f])).tensor().cpu().numpy()
    outs.append(y)
    err = np.abs(y - ref) / np.abs(ref).max()
    c, n = np.unravel_index(np.argmax(err), err.shape)
    print(f"run {r}: max err {err.max():.2e} at ch {c} n {n}; identical to run 0: {np.array_equal(y, outs[0])}")
c, n = np.unravel_index(np.argmax(np.abs(outs[0] - ref)), ref.shape)
np.set_printoptions(precision=6, suppress=False, linewidth=150)
print("ref   ", ref[c, n - 3:n + 4])
print("gpu   ", outs[0][c, n - 3:n + 4])
print("err/pk", ((outs[0][c, n - 3:n + 4] - ref[c, n - 3:n + 4]) / np.abs(ref).max()))
print("peak", np.abs(ref).max(), "this channel's peak", np.abs(ref[c]).max())
