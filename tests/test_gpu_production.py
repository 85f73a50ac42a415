"""GPU parity at production lengths and the acceptance-scale randomized sweep.

Whole output rows are compared with the CPU oracle (restatement of the
reference's numba kernels, bit-identical to them) on the kernels the
BASELINE shapes actually use: the cross-tile state carry of the single-pass
chain (look-back over hundreds of tiles per channel, block-end inclusive
states every 32 tiles) is exercised where it matters, including poles near
z = 1 where a wrong carry would not decay away within a tile.

Bars (north star): IIR / chains <= 1e-4, FIR <= 1e-5 of the output peak.
"""

import numpy as np
import pytest

import oracle
import paper_2504_08624_b200 as wp
from paper_2504_08624_b200 import engine

from conftest import random_cascade

pytestmark = pytest.mark.gpu

FIR_TOL = 1e-5
IIR_TOL = 1e-4


def _run(stages, x, fs):
    """GPU result and oracle result of a bound chain on the same fp32 input."""
    import torch

    x32 = np.ascontiguousarray(x, dtype=np.float32)
    w = wp.Wave.from_tensor(torch.from_numpy(x32).cuda(), fs)
    y = wp.pipe(w, wp.Chain(stages)).tensor().cpu().numpy().astype(np.float64)
    ref = oracle.pipe(x32.astype(np.float64), wp.Chain(stages).bind(fs).stages, oracle.default_threads())
    return y, ref


def _cfg3():
    return [wp.design_butterworth("hp", 4, 100), wp.design_chebyshev1("lp", 4, 1.0, 8000),
            wp.design_fir("lp", 101, 15000), wp.Gain(0.5)]


def _describe(stages, fs, C, N):
    return engine.plan_for(wp.Chain(stages).bind(fs).stages, device=0).describe_for(C, N)


def test_cfg3_full_length_rows():
    """cfg3 at the full 5.76 M samples per channel (704 tiles, 22 look-back
    blocks): two whole rows against the oracle."""
    fs, N = 48000, 5_760_000
    x = oracle.white_noise(N / fs, 2, fs, 42)
    assert "chain_lb" in _describe(_cfg3(), fs, 32, N)[0]
    y, ref = _run(_cfg3(), x, fs)
    assert oracle.parity_error(y, ref) <= IIR_TOL
    # the tail as strictly as the whole: the carry must not drift over the row
    assert oracle.parity_error(y[:, -48000:], ref[:, -48000:]) <= IIR_TOL


def test_cfg5_default_route_full_length_rows():
    """cfg5's filter (Butterworth LP8 2 kHz) at the full 14.4 M samples per
    channel on the default large-call route (chain_lb, 1758 tiles/channel)."""
    fs, N = 48000, 14_400_000
    stages = [wp.design_butterworth("lp", 8, 2000)]
    d = _describe(stages, fs, 2, N)[0]
    assert "chain_lb" in d, d
    x = oracle.white_noise(N / fs, 2, fs, 5)
    y, ref = _run(stages, x, fs)
    assert oracle.parity_error(y, ref) <= IIR_TOL
    assert oracle.parity_error(y[:, -48000:], ref[:, -48000:]) <= IIR_TOL


@pytest.mark.parametrize("kind", ["hp2_3hz_fir", "one_pole_0p9999", "hp4_20hz_sine"])
def test_near_unit_pole_long_channels(kind):
    """Poles within 1e-3 of z = 1 over >= 300 tiles per channel: a state carried
    wrongly across a tile would persist for thousands of samples."""
    fs = 48000
    N = 310 * 8192 + 123
    n = np.arange(N)
    if kind == "hp2_3hz_fir":
        stages = [wp.design_butterworth("hp", 2, 3), wp.design_fir("lp", 31, 15000)]
        x = np.stack([0.9 * np.sin(2 * np.pi * 40 * n / fs), oracle.white_noise(N / fs, 1, fs, 3)[0]])
    elif kind == "one_pole_0p9999":
        stages = [wp.IirFilter.from_sections([wp.BiquadSection(1e-4, 0.0, 0.0, -0.9999, 0.0)], fs=fs)]
        x = np.stack([np.ones(N), oracle.white_noise(N / fs, 1, fs, 4)[0]])
    else:
        stages = [wp.design_butterworth("hp", 4, 20), wp.Gain(2.0)]
        x = np.stack([0.9 * np.sin(2 * np.pi * 30 * n / fs), 0.5 * np.sin(2 * np.pi * 300 * n / fs)])
    y, ref = _run(stages, x, fs)
    assert oracle.parity_error(y, ref) <= IIR_TOL, kind
    assert oracle.parity_error(y[:, -8192:], ref[:, -8192:]) <= IIR_TOL, kind


def test_cfg4_full_length_channel_pair():
    """cfg4's 4096-tap FIR over one channel pair at the full 28.8 M samples (the
    FFT overlap-save path), against the reference's overlap-add restatement."""
    fs, N = 48000, 28_800_000
    stages = [wp.design_fir("lp", 4096, 2000, "hamming")]
    assert _describe(stages, fs, 2, N)[0].startswith("fft_ols")
    x = oracle.white_noise(N / fs, 2, fs, 6)
    y, ref = _run(stages, x, fs)
    assert oracle.parity_error(y, ref) <= FIR_TOL


def test_silence_after_loud_passage():
    """A tile of silence after a loud one: the state term dominates the output
    (state operand rows that would overflow fp16 take the CUDA-core path)."""
    fs = 48000
    N = 64 * 8192
    rng = np.random.default_rng(8)
    x = np.zeros((2, N))
    x[:, : 20 * 8192] = 1e3 * rng.standard_normal((2, 20 * 8192))
    x[1, 40 * 8192:] = 1e-3 * rng.standard_normal(N - 40 * 8192)
    stages = [wp.design_butterworth("lp", 8, 300), wp.design_fir("lp", 41, 9000)]
    y, ref = _run(stages, x, fs)
    assert oracle.parity_error(y, ref) <= IIR_TOL
    # the decaying tail itself, relative to its own peak
    tail = slice(20 * 8192, 22 * 8192)
    assert oracle.parity_error(y[:, tail], ref[:, tail]) <= IIR_TOL


# ---- acceptance-scale randomized sweep (pkg/tests/test_acceptance.py:39-83) ----


def test_acceptance_random_cascades():
    """200 random cascades x 1-12 channels x 10^3-10^5 frames
    (test_acceptance.py:39-57, seed 0xACCE01 of the reference's sweep)."""
    rng = np.random.default_rng(0xACCE01)
    worst = 0.0
    for case in range(200):
        filt = random_cascade(rng, max_sections=6, fs=44100)
        C = int(rng.integers(1, 13))
        N = int(10 ** rng.uniform(3, 5))
        x = rng.standard_normal((C, N))
        y, ref = _run([filt], x, 44100)
        err = oracle.parity_error(y, ref)
        worst = max(worst, err)
        assert err <= IIR_TOL, (case, C, N, err)
    print(f"worst of 200 cascades: {worst:.2e}")


@pytest.mark.parametrize("strategy", ["direct", "fft"])
def test_acceptance_random_firs(strategy):
    """100 random FIRs of 3-1025 taps through both strategies
    (test_acceptance.py:60-83, seed 0xACCE02)."""
    rng = np.random.default_rng(0xACCE02)
    for case in range(100):
        T = int(rng.integers(3, 1026))
        taps = rng.uniform(-1, 1, T) / np.sqrt(T)
        C = int(rng.integers(1, 5))
        N = int(rng.integers(T, 60000))
        x = rng.standard_normal((C, N))
        f = wp.FirFilter.from_taps(taps, 48000)
        w = wp.Wave(x.astype(np.float32).astype(np.float64), 48000)
        y = wp.apply_fir(f, w, strategy=strategy).samples
        ref = oracle.fir_direct(taps, w.samples)
        assert oracle.parity_error(y, ref) <= FIR_TOL, (case, T, C, N)


def test_multitile_random_chains():
    """Random IIR (1-5 sections) | FIR (8-257 taps) | gain chains and FIR-only
    chains over 2-12 tiles of 8192 plus a random tail: one chain_lb / fir_tc pass
    each, full tiles through the TMA output path, the last partial tile through
    the guarded stores."""
    rng = np.random.default_rng(0xB200)
    fs = 48000
    for case in range(36):
        C = int(rng.integers(1, 10))
        N = 8192 * int(rng.integers(2, 13)) + int(rng.integers(0, 8192))
        T = int(rng.integers(8, 258))
        taps = rng.uniform(-1, 1, T) / np.sqrt(T)
        fir = wp.FirFilter.from_taps(taps, fs)
        if case % 3 == 2:
            stages = [fir, wp.Gain(0.7)]
            kind = "fir_tc"
        else:
            stages = [random_cascade(rng, max_sections=5, fs=fs), fir, wp.Gain(1.3)]
            kind = "chain_lb"
        desc = wp.Chain(stages).bind(fs).stages
        assert any(kind in d for d in engine.plan_for(desc, device=0).describe_for(C, N)), (case, kind)
        x = rng.standard_normal((C, N))
        y, ref = _run(stages, x, fs)
        tol = FIR_TOL if kind == "fir_tc" else IIR_TOL
        assert oracle.parity_error(y, ref) <= tol, (case, kind, C, N, T)


def test_ill_conditioned_random_cascade_dense_basis():
    """The worst of 1500 random 6-section cascades (the reference's generator,
    tools/six_section_probe.py seed 5, case 1407): its per-section balanced basis
    has an fp32 roundoff gain of ~1700, so the plan keeps the run in one pass and
    switches to the globally balanced (dense) basis - 1.4e-4 of the peak before,
    under 1e-5 after."""
    from conftest import random_stable_section

    rng = np.random.default_rng(5)
    for _ in range(1408):
        f = wp.IirFilter.from_sections([random_stable_section(rng) for _ in range(6)], 44100,
                                       overall_gain=float(rng.uniform(0.25, 2.0)))
        C, N = int(rng.integers(1, 13)), int(10 ** rng.uniform(4, 5.5))
        x = rng.standard_normal((C, N))
    desc = engine.plan_for(wp.Chain([f]).bind(44100).stages, device=0).describe_for(C, N)
    assert len(desc) == 1 and "globally balanced dense" in desc[0], desc
    y, ref = _run([f], x, 44100)
    assert oracle.parity_error(y, ref) <= 1e-5
