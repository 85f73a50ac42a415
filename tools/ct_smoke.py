"""Quick parity sweep of the tensor-core chain path vs the oracle (diagnostics).

python tools/ct_smoke.py  -> error/peak for several chains x inputs.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import oracle  # noqa: E402
import paper_2504_08624_b200 as wp  # noqa: E402


def chains(fs):
    return {
        "cfg3": [wp.design_butterworth("hp", 4, 100), wp.design_chebyshev1("lp", 4, 1.0, 8000),
                 wp.design_fir("lp", 101, 15000), wp.Gain(0.5)],
        "cfg1": [wp.design_butterworth("lp", 4, 1000)],
        "cfg5": [wp.design_butterworth("lp", 8, 2000)],
        "hp2|fir31": [wp.design_butterworth("hp", 2, 300), wp.design_fir("lp", 31, 5000)],
    }


def main():
    fs = 48000
    C, N = 3, 200_000
    n = np.arange(N)
    inputs = {
        "noise": oracle.white_noise(N / fs, C, fs, 7),
        "sine_bank": oracle.sine_bank(C, N, fs),
        "0.9sin30": np.tile(0.9 * np.sin(2 * np.pi * 30 * n / fs), (C, 1)),
        "sin50+440": np.tile(0.5 * np.sin(2 * np.pi * 50 * n / fs) + 0.3 * np.sin(2 * np.pi * 440 * n / fs), (C, 1)),
    }
    worst = 0.0
    for cname, st in chains(fs).items():
        chain = wp.Chain(st)
        bound = chain.bind(fs).stages
        for iname, x in inputs.items():
            x32 = x.astype(np.float32)
            w = wp.Wave(x32.astype(np.float64), fs)
            y = (w | chain).samples
            ref = oracle.pipe(x32.astype(np.float64), bound)
            err = oracle.parity_error(y, ref)
            worst = max(worst, err)
            print(f"{cname:10s} {iname:10s} err/peak {err:.2e}")
    print("worst", worst)


if __name__ == "__main__":
    torch.cuda.init()
    main()
