"""Generate the golden fixtures in this directory from the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

It imports the unmodified reference package ``wavepipe`` read-only and writes

* design.json   - coefficients of every pinned design plus the
                  catalog designs used by the reference tests;
* vectors.npz   - small input/output pairs: inputs are fp32-rounded (the B200
                  path's input dtype) and widened to float64 before being fed to
                  the reference, outputs are the reference's float64 results;
* noise.json    - white_noise heads (wave.py:141-168);
* golden_hashes.json - the reference's own end-to-end sha256
                  (pkg/tests/golden/golden_hashes.json, recomputed here by
                  running the reference CLI and checked equal).

The fixtures pin the oracle (tests/test_oracle.py) and are the ground truth of
the GPU parity tests; nothing reads /root/reference at test time.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

import wavepipe as wp
from wavepipe.cli import main as ref_cli

HERE = os.path.dirname(os.path.abspath(__file__))


class RefGain:
    """The reference's duck-typed gain stage (pkg/tests/test_chain.py:177-187)."""

    def __init__(self, factor):
        self.factor = factor

    def bind(self, fs):
        return self

    def apply(self, wave, backend="auto"):
        return wp.Wave(wave.samples * self.factor, fs=wave.fs)


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32)


def iir_entry(f):
    return {
        "type": "iir",
        "overall_gain": f.overall_gain,
        "sections": [[s.b0, s.b1, s.b2, s.a1, s.a2] for s in f.sections],
    }


def main():
    designs = {}
    pinned = {
        "cfg1_butter_lp4_1000_44100": wp.design_butterworth("lp", 4, 1000, 44100),
        "cfg3_butter_hp4_100_48000": wp.design_butterworth("hp", 4, 100, 48000),
        "cfg3_cheby1_lp4_1db_8000_48000": wp.design_chebyshev1("lp", 4, 1.0, 8000, 48000),
        "cfg5_butter_lp8_2000_48000": wp.design_butterworth("lp", 8, 2000, 48000),
        "butter_lp4_1000_44100": wp.design_butterworth("lowpass", 4, 1000, 44100),
        "cheby1_lp4_1db_2000_44100": wp.design_chebyshev1("lowpass", 4, 1.0, 2000, 44100),
        "butter_hp3_1000_44100": wp.design_butterworth("hp", 3, 1000, 44100),
        "cheby1_hp5_0.5db_3000_44100": wp.design_chebyshev1("hp", 5, 0.5, 3000, 44100),
        "lo_shelf_2000_-6_0.707_44100": wp.design_shelf("lo_shelf", 2000, -6.0, 0.707, 44100),
        "hi_shelf_1000_6_0.707_44100": wp.design_shelf("hi_shelf", 1000, 6.0, 0.707, 44100),
        "peaking_1000_12_1_44100": wp.design_peaking(1000, 12.0, 1.0, 44100),
    }
    for name, f in pinned.items():
        designs[name] = iir_entry(f)
    firs = {
        "cfg2_fir_lp101_1000_hamming_48000": wp.design_fir("lp", 101, 1000, "hamming", 48000),
        "cfg3_fir_lp101_15000_hamming_48000": wp.design_fir("lp", 101, 15000, "hamming", 48000),
        "cfg4_fir_lp4096_2000_hamming_48000": wp.design_fir("lp", 4096, 2000, "hamming", 48000),
        "fir_hp65_3000_blackman_44100": wp.design_fir("hp", 65, 3000, "blackman", 44100),
        "fir_bp129_500_4000_rect_44100": wp.design_fir("bp", 129, (500, 4000), "rect", 44100),
    }
    for name, f in firs.items():
        designs[name] = {"type": "fir", "taps": f.taps.tolist()}
    with open(os.path.join(HERE, "design.json"), "w") as fh:
        json.dump(designs, fh, indent=1)

    vec = {}

    def case(name, x, stages, fs, strategy=None):
        x32 = f32(x)
        w = wp.Wave(x32.astype(np.float64), fs)
        if strategy is not None:
            assert len(stages) == 1
            y = wp.apply_fir(stages[0].bind(fs), w, strategy=strategy).samples
        else:
            y = wp.pipe(w, wp.Chain(stages) if len(stages) > 1 else stages[0]).samples
        vec[f"{name}__x"] = x32
        vec[f"{name}__y"] = y
        print(f"{name}: x{x32.shape} peak {np.max(np.abs(y)):.3g}")

    noise = lambda c, n, fs, seed=42: wp.white_noise(n / fs, c, fs, seed).samples  # noqa: E731
    n = np.arange(16000)
    case("cfg1", noise(2, 6000, 44100), [wp.design_butterworth("lp", 4, 1000)], 44100)
    case("cfg2", noise(2, 6000, 48000), [wp.design_fir("lp", 101, 1000, "hamming")], 48000)
    cfg3 = [
        wp.design_butterworth("hp", 4, 100),
        wp.design_chebyshev1("lp", 4, 1.0, 8000),
        wp.design_fir("lp", 101, 15000),
        RefGain(0.5),
    ]
    case("cfg3_noise", noise(2, 12000, 48000), cfg3, 48000)
    sines = np.stack(
        [
            0.5 * np.sin(2 * np.pi * 50 * n / 48000) + 0.3 * np.sin(2 * np.pi * 440 * n / 48000),
            0.9 * np.sin(2 * np.pi * 30 * n / 48000),
        ]
    )
    case("cfg3_sine", sines, cfg3, 48000)
    case("cfg4", noise(1, 20000, 48000), [wp.design_fir("lp", 4096, 2000, "hamming")], 48000)
    case("cfg5", noise(3, 6000, 48000), [wp.design_butterworth("lp", 8, 2000)], 48000)
    bench_chain = [
        wp.design_butterworth("lowpass", 4, 1000.0),
        wp.design_butterworth("lowpass", 4, 1200.0),
        wp.design_chebyshev1("lowpass", 4, 1.0, 2000.0),
        wp.design_chebyshev1("lowpass", 4, 1.0, 2400.0),
    ]
    case("bench_chain", noise(2, 4000, 44100, seed=5), bench_chain, 44100)
    case(
        "mixed_fir_peak",
        noise(2, 2048, 44100, seed=11),
        [wp.design_fir("lowpass", 33, 4000), wp.design_peaking(1000, gain_db=2.0)],
        44100,
    )
    case(
        "shelves",
        noise(2, 4096, 44100, seed=3),
        [wp.design_shelf("hi_shelf", 1000, gain_db=3.0), wp.design_shelf("lo_shelf", 2000, gain_db=3.0)],
        44100,
    )

    # random cascades, drawn like conftest.random_cascade (pkg/tests/conftest.py:29-49)
    rng = np.random.default_rng(0xB200)
    for i in range(6):
        n_sec = int(rng.integers(1, 7))
        secs = []
        for _ in range(n_sec):
            if rng.random() < 0.7:
                r = rng.uniform(0.0, 0.95)
                th = rng.uniform(0.0, np.pi)
                a1, a2 = -2.0 * r * np.cos(th), r * r
            else:
                p1, p2 = rng.uniform(-0.95, 0.95, size=2)
                a1, a2 = -(p1 + p2), p1 * p2
            b = rng.uniform(-2.0, 2.0, size=3)
            secs.append(wp.BiquadSection(b[0], b[1], b[2], a1, a2))
        filt = wp.IirFilter.from_sections(secs, fs=44100, overall_gain=float(rng.uniform(0.25, 2.0)))
        designs[f"random_cascade_{i}"] = iir_entry(filt)
        case(f"random_cascade_{i}", rng.standard_normal((2, 3000)), [filt], 44100)
    # random FIR taps (test_acceptance.py:60-83): both strategies
    for i, n_taps in enumerate((3, 129, 700, 1025)):
        taps = rng.standard_normal(n_taps) / np.sqrt(n_taps)
        filt = wp.FirFilter.from_taps(taps, fs=44100)
        designs[f"random_fir_{i}"] = {"type": "fir", "taps": taps.tolist()}
        x = rng.standard_normal((2, 5000))
        case(f"random_fir_{i}_direct", x, [filt], 44100, strategy="direct")
        case(f"random_fir_{i}_fft", x, [filt], 44100, strategy="fft")
    with open(os.path.join(HERE, "design.json"), "w") as fh:
        json.dump(designs, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "vectors.npz"), **vec)

    noise_fix = {
        "seed7_head": wp.white_noise(5, 1, 8000, seed=7).samples[0, :5].tolist(),
        "seed42_3ch_480": wp.white_noise(0.01, 3, 48000, seed=42).samples.tolist(),
        "seed20260809_tail": wp.white_noise(2, 2, 44100, seed=20260809).samples[:, -8:].tolist(),
    }
    with open(os.path.join(HERE, "noise.json"), "w") as fh:
        json.dump(noise_fix, fh)

    # end-to-end golden: the reference's own CLI on its pinned chain
    chain = (
        "butter(lp, order=4, fc=1000) | butter(lp, order=4, fc=1200) | "
        "cheby1(lp, order=4, fc=2000, ripple_db=1) | cheby1(lp, order=4, fc=2400, ripple_db=1)"
    )
    with tempfile.TemporaryDirectory() as tmp:
        noise_path = os.path.join(tmp, "n.wav")
        out_path = os.path.join(tmp, "o.wav")
        assert ref_cli(["noise", "--duration", "2", "--channels", "2", "--fs", "44100",
                        "--seed", "20260809", "--out", noise_path]) == 0
        assert ref_cli(["apply", noise_path, out_path, "--chain", chain]) == 0
        digest = hashlib.sha256(open(out_path, "rb").read()).hexdigest()
    stored = json.load(open("/root/reference/pkg/tests/golden/golden_hashes.json"))["cmd_apply_pinned_chain"]
    assert digest == stored, (digest, stored)
    with open(os.path.join(HERE, "golden_hashes.json"), "w") as fh:
        json.dump({"cmd_apply_pinned_chain": digest, "noise_encoding": "float32",
                   "chain": chain}, fh, indent=2)
    print("golden sha256", digest)


if __name__ == "__main__":
    sys.exit(main())
