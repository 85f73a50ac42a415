"""Randomized GPU-vs-oracle stress (diagnostics; not part of the pytest suite):
python tools/stress_random.py [seconds] [seed] [max IIR sections per chain, default 5]
Random chains (IIR cascades, FIRs of 3-600 taps, gains, Normalize, in random order),
random channel counts and lengths (often several 8192-sample tiles plus a tail),
device or pinned-host sources, compared with the oracle at the tests' tolerances."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import oracle  # noqa: E402
import paper_2504_08624_b200 as wp  # noqa: E402
from conftest import random_cascade  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
# total IIR sections per chain: <= 5 keeps every LTI run in one pass; more sections run
# as several passes whose fp32 intermediates can limit adversarial chains
MAX_SECTIONS = int(sys.argv[3]) if len(sys.argv) > 3 else 5
fs = 48000
t0 = time.time()
n = worst_iir = worst_fir = 0.0
cases = 0
while time.time() - t0 < budget:
    stages, has_iir, nsec = [], False, 0
    for _ in range(int(rng.integers(1, 5))):
        kind = rng.choice(["iir", "fir", "gain", "norm"], p=[0.4, 0.4, 0.15, 0.05])
        if kind == "iir":
            if nsec >= MAX_SECTIONS:
                continue
            f = random_cascade(rng, max_sections=min(4, MAX_SECTIONS - nsec), fs=fs)
            nsec += len(f.sections)
            stages.append(f)
            has_iir = True
        elif kind == "fir":
            T = int(rng.choice([int(rng.integers(3, 300)), int(rng.integers(300, 600))]))
            stages.append(wp.FirFilter.from_taps(rng.uniform(-1, 1, T) / np.sqrt(T), fs))
        elif kind == "gain":
            stages.append(wp.Gain(float(rng.uniform(0.2, 2.0))))
        else:
            stages.append(wp.Normalize(float(rng.uniform(0.3, 1.0))))
    C = int(rng.integers(1, 12))
    N = 8192 * int(rng.integers(0, 9)) + int(rng.integers(1, 8192))
    x = rng.standard_normal((C, N)).astype(np.float32)
    import torch

    def desc(st):
        out = []
        for s in st:
            if hasattr(s, "taps"):
                out.append(f"FIR{len(s.taps)}")
            elif hasattr(s, "sos_rows"):
                out.append(f"IIR{len(s.bind(fs).sos_rows()) if hasattr(s, 'bind') else '?'}")
            else:
                out.append(type(s).__name__)
        return out

    try:
        _ = wp.Chain(stages).bind(fs).stages
    except Exception as e:  # noqa: BLE001
        print("bind failed", desc(stages), e)
        continue
    host = rng.random() < 0.3 and not any(isinstance(s, wp.Normalize) for s in stages)
    try:
        if host:
            w = wp.Wave.from_tensor(torch.from_numpy(x).pin_memory(), fs)  # streamed host path
            y = wp.pipe(w, wp.Chain(stages)).numpy32().astype(np.float64)
        else:
            w = wp.Wave.from_tensor(torch.from_numpy(x).cuda(), fs)
            y = wp.pipe(w, wp.Chain(stages)).tensor().cpu().numpy().astype(np.float64)
    except Exception as e:  # noqa: BLE001
        print(f"ERROR case {cases}: C={C} N={N} host={host} stages={desc(stages)}: {e}")
        sys.exit(2)
    ref = oracle.pipe(x.astype(np.float64), wp.Chain(stages).bind(fs).stages, oracle.default_threads())
    err = oracle.parity_error(y, ref)
    tol = 1e-4 if has_iir else 1e-5
    if has_iir:
        worst_iir = max(worst_iir, err)
    else:
        worst_fir = max(worst_fir, err)
    cases += 1
    if not err <= tol:
        print(f"FAIL case {cases}: C={C} N={N} err={err:.3e} tol={tol} stages={desc(stages)} host={host}")
        bound = wp.Chain(stages).bind(fs).stages
        os.makedirs("gpurun_out", exist_ok=True)
        np.savez(f"gpurun_out/stress_fail_{cases}.npz", x=x, y=y, ref=ref,
                 **{f"s{i}_{type(b).__name__}": (b.sos_rows() if hasattr(b, "sos_rows") else
                                                  np.asarray(getattr(b, "taps", [getattr(b, "factor", 0.0)])))
                    for i, b in enumerate(bound)})
        if os.environ.get("STRESS_KEEP_GOING") is None:
            sys.exit(1)
print(f"{cases} random chains in {time.time() - t0:.0f} s: worst IIR {worst_iir:.2e} (bar 1e-4), "
      f"worst FIR-only {worst_fir:.2e} (bar 1e-5)")
