"""GPU parity: the sm_100a path (through the public API -> C ABI) against the
reference's own outputs (golden fixtures) and the CPU oracle.

Bars (SURVEY.md §8c / BASELINE.md §4), metric max|y - y_ref| / max|y_ref|:
FIR <= 1e-5, IIR cascades and chains <= 1e-4 (the scan re-associates the
recurrence into 64-sample chunks; IIR blocks with pole radius > 0.98 run in
float64). Known-answer tests of the reference are exact.
"""

import numpy as np
import pytest

import oracle
import paper_2504_08624_b200 as wp
from paper_2504_08624_b200 import _native

from conftest import iir_from_entry, random_cascade, random_unbound_stage

pytestmark = pytest.mark.gpu

FIR_TOL = 1e-5
IIR_TOL = 1e-4


def _cfg3():
    return [
        wp.design_butterworth("hp", 4, 100),
        wp.design_chebyshev1("lp", 4, 1.0, 8000),
        wp.design_fir("lp", 101, 15000),
        wp.Gain(0.5),
    ]


def _bench_chain():
    return [
        wp.design_butterworth("lowpass", 4, 1000.0),
        wp.design_butterworth("lowpass", 4, 1200.0),
        wp.design_chebyshev1("lowpass", 4, 1.0, 2000.0),
        wp.design_chebyshev1("lowpass", 4, 1.0, 2400.0),
    ]


GOLDEN_CASES = {
    "cfg1": (44100, lambda D: [wp.design_butterworth("lp", 4, 1000)], IIR_TOL),
    "cfg2": (48000, lambda D: [wp.design_fir("lp", 101, 1000, "hamming")], FIR_TOL),
    "cfg3_noise": (48000, lambda D: _cfg3(), IIR_TOL),
    "cfg3_sine": (48000, lambda D: _cfg3(), IIR_TOL),
    "cfg4": (48000, lambda D: [wp.design_fir("lp", 4096, 2000, "hamming")], FIR_TOL),
    "cfg5": (48000, lambda D: [wp.design_butterworth("lp", 8, 2000)], IIR_TOL),
    "bench_chain": (44100, lambda D: _bench_chain(), IIR_TOL),
    "mixed_fir_peak": (44100, lambda D: [wp.design_fir("lowpass", 33, 4000), wp.design_peaking(1000, gain_db=2.0)], IIR_TOL),
    "shelves": (44100, lambda D: [wp.design_shelf("hi_shelf", 1000, gain_db=3.0), wp.design_shelf("lo_shelf", 2000, gain_db=3.0)], IIR_TOL),
}
for _i in range(6):
    GOLDEN_CASES[f"random_cascade_{_i}"] = (44100, (lambda i: lambda D: [iir_from_entry(D[f"random_cascade_{i}"], 44100)])(_i), IIR_TOL)


@pytest.mark.parametrize("name", sorted(GOLDEN_CASES))
def test_golden_reference_outputs(name, golden_vectors, golden_designs):
    """Reference (wavepipe, float64) output on the same fp32-rounded input."""
    fs, build, tol = GOLDEN_CASES[name]
    x = golden_vectors[f"{name}__x"]
    y_ref = golden_vectors[f"{name}__y"]
    w = wp.Wave(x, fs)
    y = wp.pipe(w, wp.Chain(build(golden_designs)))
    err = oracle.parity_error(y.samples, y_ref)
    assert err <= tol, f"{name}: parity {err:.3e} > {tol:g}"


@pytest.mark.parametrize("i", range(4))
@pytest.mark.parametrize("strategy", ["direct", "fft"])
def test_golden_random_fir(i, strategy, golden_vectors, golden_designs):
    taps = golden_designs[f"random_fir_{i}"]["taps"]
    x = golden_vectors[f"random_fir_{i}_{strategy}__x"]
    y_ref = golden_vectors[f"random_fir_{i}_{strategy}__y"]
    filt = wp.FirFilter.from_taps(taps, fs=44100)
    y = wp.apply_fir(filt, wp.Wave(x, 44100), strategy=strategy)
    assert oracle.parity_error(y.samples, y_ref) <= FIR_TOL


# ---- known-answer tests of the reference (test_engine.py) -------------------


def test_iir_identity_bit_exact(rng):
    w = wp.Wave(rng.standard_normal((3, 1000)), 44100)
    ident = wp.IirFilter.from_sections([wp.BiquadSection(1.0, 0.0, 0.0, 0.0, 0.0)], fs=44100)
    assert np.array_equal(wp.apply_iir(ident, w).samples, w.samples)


def test_one_pole_impulse_exact():
    impulse = np.zeros(8)
    impulse[0] = 1.0
    one_pole = wp.IirFilter.from_sections([wp.BiquadSection(1.0, 0.0, 0.0, -0.5, 0.0)], fs=44100)
    out = wp.apply_iir(one_pole, wp.Wave([impulse], 44100))
    np.testing.assert_array_equal(out.samples[0], 0.5 ** np.arange(8))


def test_one_pole_long_impulse_crosses_tiles():
    n = 50000  # spans several tiles, exercises the look-back
    x = np.zeros(n)
    x[0] = 1.0
    f = wp.IirFilter.from_sections([wp.BiquadSection(1.0, 0.0, 0.0, -0.9995, 0.0)], fs=44100)
    out = wp.apply_iir(f, wp.Wave([x], 44100)).samples[0]
    expect = 0.9995 ** np.arange(n)
    assert np.max(np.abs(out - expect)) <= 1e-4


@pytest.mark.parametrize(
    "taps,x,expect",
    [
        ([1.0], None, None),
        ([0.0, 1.0], [1.0, 2.0, 3.0], [0.0, 1.0, 2.0]),
        ([0.5, 0.5], [1.0, 0.0, 0.0, 0.0], [0.5, 0.5, 0.0, 0.0]),
        ([0.25, 0.25, 0.25, 0.25], [1.0, 1.0], [0.25, 0.5]),
    ],
)
def test_fir_known_answers(taps, x, expect, rng):
    if x is None:
        w = wp.Wave(rng.standard_normal((2, 1000)), 44100)
        out = wp.apply_fir(wp.FirFilter.from_taps(taps, fs=44100), w, strategy="direct")
        assert np.array_equal(out.samples, w.samples)
    else:
        out = wp.apply_fir(wp.FirFilter.from_taps(taps, fs=44100), wp.Wave([x], 44100), strategy="direct")
        np.testing.assert_array_equal(out.samples[0], expect)


def test_fir_fft_tiny_signal():
    w = wp.Wave([[1.0, 2.0]], 44100)
    f = wp.FirFilter.from_taps([0.5, 0.25, 0.125], fs=44100)
    d = wp.apply_fir(f, w, strategy="direct").samples
    ff = wp.apply_fir(f, w, strategy="fft").samples
    np.testing.assert_allclose(ff, d, atol=1e-6)


# ---- oracle parity on fresh seeded inputs ---------------------------------


@pytest.mark.parametrize("seed", range(8))
def test_random_cascades_vs_oracle(seed):
    rng = np.random.default_rng(0xACCE01 + seed)
    filt = random_cascade(rng, max_sections=6)
    frames = int(10 ** rng.uniform(3, 5))
    channels = int(rng.integers(1, 13))
    w = wp.Wave(rng.standard_normal((channels, frames)), 44100)
    y = wp.apply_iir(filt, w).samples
    ref = oracle.iir_cascade(filt.sos_rows(), w.samples)
    assert oracle.parity_error(y, ref) <= IIR_TOL


@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_forced_precision_paths(precision):
    rng = np.random.default_rng(7)
    filt = wp.design_butterworth("lp", 8, 2000, 48000)
    w = wp.Wave(rng.standard_normal((3, 70000)), 48000)
    wp.set_iir_precision(precision)
    try:
        y = wp.apply_iir(filt, w).samples
    finally:
        wp.set_iir_precision("auto")
    assert oracle.parity_error(y, oracle.iir_cascade(filt.sos_rows(), w.samples)) <= IIR_TOL


@pytest.mark.parametrize("n_taps", [3, 31, 101, 257, 1025])
def test_fir_direct_vs_oracle(n_taps):
    rng = np.random.default_rng(n_taps)
    taps = rng.standard_normal(n_taps) / np.sqrt(n_taps)
    w = wp.Wave(rng.standard_normal((3, 40000 + n_taps)), 44100)
    y = wp.apply_fir(wp.FirFilter.from_taps(taps, 44100), w, strategy="direct").samples
    assert oracle.parity_error(y, oracle.fir_direct(taps, w.samples)) <= FIR_TOL


def test_ragged_shapes_and_unaligned_rows():
    rng = np.random.default_rng(3)
    chain = [wp.design_butterworth("hp", 2, 300, 44100), wp.design_fir("lp", 17, 5000, fs=44100), wp.Gain(2.0)]
    for frames in (1, 2, 3, 5, 63, 64, 65, 8063, 8064, 8065, 8191, 8192, 8193, 20001):
        w = wp.Wave(rng.standard_normal((2, frames)), 44100)
        y = wp.pipe(w, wp.Chain(chain)).samples
        ref = oracle.pipe(w.samples, chain)
        assert oracle.parity_error(y, ref) <= IIR_TOL, frames


def test_normalize_stage():
    rng = np.random.default_rng(5)
    w = wp.Wave(rng.standard_normal((4, 5000)) * 3.0, 44100)
    y = (w | wp.design_butterworth("lp", 2, 1000) | wp.Normalize(0.5)).samples
    ref = oracle.pipe(w.samples, [wp.design_butterworth("lp", 2, 1000, 44100), wp.Normalize(0.5)])
    assert oracle.parity_error(y, ref) <= IIR_TOL
    assert abs(np.max(np.abs(y)) - 0.5) < 1e-6


# ---- determinism and algebra (bit-exact) -----------------------------------


def test_channel_independence_bit_exact():
    rng = np.random.default_rng(11)
    filt = random_cascade(rng)
    w = wp.Wave(rng.standard_normal((4, 30000)), 44100)
    full = wp.apply_iir(filt, w)
    for c in range(4):
        assert np.array_equal(full.samples[c], wp.apply_iir(filt, w.channel(c)).samples[0])


def test_repeat_runs_bit_identical():
    w = wp.white_noise(3.0, 8, 48000, seed=9)
    chain = wp.Chain(_cfg3())
    a = wp.pipe(w, chain).samples
    for _ in range(3):
        assert np.array_equal(wp.pipe(w, chain).samples, a)


def test_pipe_compose_coherence_bit_exact():
    for seed in range(10):
        rng = np.random.default_rng(seed)
        w = wp.Wave(rng.standard_normal((2, 257)), 44100)
        left = wp.Chain([random_unbound_stage(rng) for _ in range(int(rng.integers(0, 3)))])
        right = wp.Chain([random_unbound_stage(rng) for _ in range(int(rng.integers(1, 3)))])
        composed = wp.compose(left, right)
        assert wp.pipe(wp.pipe(w, left), right) == wp.pipe(w, composed)
        assert wp.pipe(w, composed) == wp.pipe(w, composed.bind(w.fs))


def test_wave_or_operator_and_custom_stage():
    w = wp.white_noise(0.05, 2, 44100, seed=11)
    hi, lo = wp.design_shelf("hi_shelf", 1000, gain_db=3.0), wp.design_shelf("lo_shelf", 2000, gain_db=3.0)
    assert (w | hi | lo) == wp.pipe(wp.pipe(w, hi), lo)

    class Half:
        def bind(self, fs):
            return self

        def apply(self, wave, backend="auto"):
            return wp.Wave(wave.samples * 0.5, fs=wave.fs)

    out = wp.pipe(w, wp.compose(Half(), wp.design_peaking(1000, gain_db=0.0)))
    np.testing.assert_array_equal(out.samples, w.samples * 0.5)


# ---- device noise generator ---------------------------------------------------


def test_white_noise_matches_reference_stream(golden_noise):
    w = wp.white_noise(5, 1, 8000, seed=7)
    head = np.array(golden_noise["seed7_head"])
    np.testing.assert_allclose(w.samples[0, :5], head, rtol=0, atol=1e-6)
    multi = wp.white_noise(0.01, 3, 48000, seed=42).samples
    ref = np.array(golden_noise["seed42_3ch_480"]).astype(np.float32).astype(np.float64)
    assert np.max(np.abs(multi - ref)) <= 1e-6


def test_white_noise_large_prefix_stable():
    a = wp.white_noise(2.0, 1, 48000, seed=3).samples
    b = wp.white_noise(2.0, 4, 48000, seed=3).samples
    assert np.array_equal(a[0], b[0])
    ref = oracle.white_noise(2.0, 4, 48000, 3).astype(np.float32).astype(np.float64)
    assert np.max(np.abs(b - ref)) <= 1e-6


# ---- full-size properties (BASELINE configs) -------------------------------


def test_cfg3_full_size_prefix_parity():
    """cfg3 at full size (32 x 5.76 M); the oracle checks a 4-channel, 1 s
    prefix (all filters are causal: the output prefix depends only on the
    input prefix)."""
    fs = 48000
    w = wp.white_noise(120.0, 32, fs, seed=42)
    y = wp.pipe(w, wp.Chain(_cfg3()))
    t = y.tensor()
    assert t.shape == (32, 5_760_000)
    sub = [0, 13, 31]
    x = w.tensor()[sub, :48000].cpu().numpy().astype(np.float64)
    ref = oracle.pipe(x, wp.Chain(_cfg3()).bind(fs).stages)
    got = t[sub, :48000].cpu().numpy().astype(np.float64)
    assert oracle.parity_error(got, ref) <= IIR_TOL
    # linearity across the whole buffer: chain(2x) == 2 chain(x) within fp32 rounding
    import torch

    y2 = wp.pipe(wp.Wave.from_tensor(w.tensor() * 2.0, fs), wp.Chain(_cfg3())).tensor()
    rel = (torch.max(torch.abs(y2 - 2.0 * t)) / torch.max(torch.abs(2.0 * t))).item()
    assert rel <= 1e-4


def test_plan_launch_accounting():
    plan = _native.Plan(tuple(wp.engine._entry(s) for s in wp.Chain(_cfg3()).bind(48000).stages))
    assert plan.num_passes == 1  # IIR(4 sections) -> FIR -> gain fused into one pass
    # one pass = one chain_lb launch (no intermediate signal in HBM)
    assert plan.launches == 1
    before = _native.launch_count()
    wp.pipe(wp.white_noise(1.0, 2, 48000, seed=1), wp.Chain(_cfg3())).tensor()
    assert _native.launch_count() - before == 2  # noise + the pass's kernel


@pytest.mark.parametrize("scale", [1e-6, 1.0, 3e4, 1e9])
def test_fir_tensor_core_dynamic_range(scale):
    """The tcgen05 split-fp16 FIR rescales each tile by a power of two, so the
    result is independent of the signal's absolute magnitude."""
    rng = np.random.default_rng(17)
    taps = wp.design_fir("lp", 101, 1000, "hamming", 48000).taps
    x = rng.standard_normal((3, 30000)) * scale
    x[1, 5000:12000] = 0.0  # silent stretch inside a channel
    w = wp.Wave(x, 48000)
    plan = wp.engine.plan_for([wp.FirFilter.from_taps(taps, 48000)])
    assert "fir_tc" in plan.describe()[0]
    y = wp.apply_fir(wp.FirFilter.from_taps(taps, 48000), w).samples
    assert oracle.parity_error(y, oracle.fir_direct(taps, w.samples)) <= FIR_TOL


def test_fir_tensor_core_zeros_and_tail():
    w = wp.Wave(np.zeros((2, 9000)), 48000)
    f = wp.design_fir("lp", 101, 1000, fs=48000)
    assert np.array_equal(wp.apply_fir(f, w).samples, np.zeros((2, 9000)))
    rng = np.random.default_rng(2)
    for frames in (1, 7, 4095, 4096, 4097, 12289):
        w = wp.Wave(rng.standard_normal((2, frames)), 48000)
        y = wp.apply_fir(f, w).samples
        assert oracle.parity_error(y, oracle.fir_direct(f.taps, w.samples)) <= FIR_TOL, frames


# ---- kernel selection: the headline configs run on the intended kernels -----


@pytest.mark.gpu
@pytest.mark.parametrize(
    "stages, fs, shape, kernel",
    [
        (lambda: [wp.design_butterworth("hp", 4, 100), wp.design_chebyshev1("lp", 4, 1.0, 8000),
                  wp.design_fir("lp", 101, 15000), wp.Gain(0.5)], 48000, (32, 5760000), "chain_lb"),  # cfg3
        (lambda: [wp.design_butterworth("lp", 8, 2000)], 48000, (1024, 14400000), "chain_lb"),      # cfg5
        (lambda: _bench_chain()[:2] + [wp.design_peaking(1000, gain_db=2.0)], 44100, (2, 88200),
         "chain_lb"),                                                                                # 5 SOS: one pass
        (lambda: [wp.design_butterworth("lp", 8, 2000)], 48000, (1, 16384), "fused"),                 # tiny IIR
        (lambda: [wp.design_butterworth("lp", 4, 1000)], 48000, (2, 96000), "fused"),                 # small, 2 SOS
        (lambda: [wp.design_butterworth("lp", 8, 2000)], 48000, (4, 48000), "chain_lb"),              # small, 4 SOS
        (lambda: [wp.design_butterworth("lp", 4, 1000)], 44100, (2, 441000), "chain_lb"),             # cfg1
        (lambda: [wp.design_fir("lp", 101, 1000, "hamming")], 48000, (8, 2880000), "fir_tc"),          # cfg2
        (lambda: [wp.design_fir("lp", 4096, 2000, "hamming")], 48000, (128, 28800000), "fft_ols"),     # cfg4
    ],
)
def test_plan_uses_intended_kernel(stages, fs, shape, kernel):
    from paper_2504_08624_b200 import engine

    plan = engine.plan_for(wp.Chain(stages()).bind(fs).stages, device=0)
    desc = plan.describe_for(*shape)
    assert len(desc) == 1 and kernel in desc[0].split("[")[0], desc
    assert plan.launches_for(*shape) == 1


# ---- host -> device -> host streaming (pinned sources, channel blocks) -------


@pytest.mark.gpu
@pytest.mark.parametrize("C", [1, 5, 32])
@pytest.mark.parametrize("fir_taps", [101, 2048])
def test_streamed_host_path_bit_exact(C, fir_taps):
    import torch

    fs = 48000
    w = wp.white_noise(0.25, C, fs, seed=21)
    chain = wp.Chain([wp.design_butterworth("hp", 4, 100), wp.design_fir("lp", fir_taps, 4000), wp.Gain(0.5)]) \
        if fir_taps <= 129 else wp.Chain([wp.design_fir("lp", fir_taps, 4000)])
    ref = (w | chain).numpy32().copy()
    pinned = torch.empty((C, w.frames), dtype=torch.float32, pin_memory=True)
    pinned.copy_(w.tensor())
    src = wp.Wave.from_tensor(pinned, fs)
    out = torch.empty_like(pinned).pin_memory()
    lazy = src | chain
    assert lazy._host_streamable()
    lazy.numpy32(out=out)
    assert np.array_equal(out.numpy(), ref)
    assert np.array_equal((src | chain).numpy32(), ref)  # pinned result allocated internally


@pytest.mark.gpu
@pytest.mark.parametrize("C", [1, 7])
@pytest.mark.parametrize("blocks", [0, 1, 3, 64])
@pytest.mark.parametrize("fft", [False, True])
def test_plan_execute_host_blocks_strides(C, blocks, fft):
    """wp_plan_execute_host (pinned and pageable host buffers, padded host row
    strides, any block count, pair-aligned blocks on the FFT path) is
    bit-identical to one device-resident wp_plan_execute; Normalize is refused."""
    import torch

    from paper_2504_08624_b200 import _native, engine

    fs, N, ld = 48000, 20001, 20011
    w = wp.white_noise(N / fs, C, fs, seed=5)
    stages = [wp.design_fir("lp", 1500, 4000)] if fft else \
        [wp.design_butterworth("hp", 4, 100), wp.design_fir("lp", 101, 4000), wp.Gain(0.5)]
    chain = wp.Chain(stages)
    ref = (w | chain).numpy32().copy()
    bound = chain.bind(fs).stages
    plan = engine.plan_for(bound)
    assert any(d.startswith("fft_ols") for d in plan.describe()) == fft
    for pin in (True, False):
        hx = torch.full((C, ld), float("nan"), dtype=torch.float32, pin_memory=pin)
        hx[:, :N].copy_(w.tensor())
        hy = torch.full((C, ld), 7.0, dtype=torch.float32, pin_memory=pin)
        dx = torch.empty((C, N), dtype=torch.float32, device="cuda")
        dy = torch.empty_like(dx)
        ws = torch.empty(plan.workspace_bytes(C, N), dtype=torch.uint8, device="cuda")
        stream = torch.cuda.current_stream().cuda_stream
        plan.execute_host(hx.data_ptr(), hy.data_ptr(), C, N, ld, ld, dx.data_ptr(), dy.data_ptr(),
                          ws.data_ptr(), ws.numel(), blocks, stream)
        torch.cuda.current_stream().synchronize()
        assert np.array_equal(hy[:, :N].numpy(), ref)
        assert np.all(hy[:, N:].numpy() == 7.0)  # padding untouched
    with pytest.raises(wp.WavepipeError):
        plan.execute_host(hx.data_ptr(), hy.data_ptr(), C, N, ld, ld, dx.data_ptr(), dx.data_ptr(),
                          ws.data_ptr(), ws.numel(), blocks, stream)  # dx == dy
    norm = engine.plan_for(list(bound) + [wp.Normalize()])
    with pytest.raises(wp.WavepipeError, match="Normalize"):
        norm.execute_host(hx.data_ptr(), hy.data_ptr(), C, N, ld, ld, dx.data_ptr(), dy.data_ptr(),
                          ws.data_ptr(), ws.numel(), blocks, stream)
    assert _native.EXPORTED.count("wp_plan_execute_host") == 1


@pytest.mark.gpu
def test_plan_execute_host_blocks_take_the_whole_call_route():
    """cfg1's shape (2 x 441000, LP4): the whole call runs chain_lb (108 tiles),
    a one-channel block alone would take the CUDA-core scan (54 tiles); the
    streamed blocks keep the whole call's route, so the e2e output is
    bit-identical to the device-resident pass."""
    import torch

    fs = 44100
    w = wp.white_noise(10.0, 2, fs, seed=42)
    chain = wp.Chain([wp.design_butterworth("lp", 4, 1000)])
    plan = __import__("paper_2504_08624_b200.engine", fromlist=["plan_for"]).plan_for(chain.bind(fs).stages)
    assert plan.describe_for(2, w.frames)[0].startswith("chain_lb")
    assert not plan.describe_for(1, w.frames)[0].startswith("chain_lb")
    ref = (w | chain).numpy32().copy()
    pinned = torch.empty((2, w.frames), dtype=torch.float32, pin_memory=True)
    pinned.copy_(w.tensor())
    out = torch.empty_like(pinned).pin_memory()
    (wp.Wave.from_tensor(pinned, fs) | chain).numpy32(out=out)
    assert np.array_equal(out.numpy(), ref)


# ---- FFT overlap-save path: ragged lengths, odd channel counts ---------------


@pytest.mark.gpu
@pytest.mark.parametrize("n_taps", [513, 2048, 4096])
@pytest.mark.parametrize("frames", [1, 100, 4095, 12288, 12289, 30001])
def test_fft_path_ragged_vs_oracle(n_taps, frames):
    rng = np.random.default_rng(n_taps + frames)
    taps = rng.standard_normal(n_taps) / np.sqrt(n_taps)
    for C in (1, 3):
        x = rng.standard_normal((C, frames)).astype(np.float32).astype(np.float64)
        y = wp.apply_fir(wp.FirFilter.from_taps(taps, 48000), wp.Wave(x, 48000), strategy="fft").samples
        assert oracle.parity_error(y, oracle.fir_direct(taps, x)) <= FIR_TOL, (C, frames)


# ---- C ABI with padded, unaligned row strides --------------------------------


@pytest.mark.gpu
@pytest.mark.parametrize("pads", [(3, 5), (4, 8)], ids=["unaligned", "aligned_padded"])
@pytest.mark.parametrize("chain_kind", ["cfg3", "fir101", "fir4096", "lp8"])
def test_plan_execute_unaligned_strides(chain_kind, pads):
    """(3, 5): rows not 16-byte aligned - scalar edge paths, no TMA stores;
    (4, 8): aligned padded rows - full tiles leave through the TMA tensor map
    (row stride ldy), the last partial tile through the guarded path; the
    padding must stay untouched either way."""
    import torch

    from paper_2504_08624_b200 import engine

    fs = 48000
    stages = {
        "cfg3": _cfg3(),
        "fir101": [wp.design_fir("lp", 101, 1000)],
        "fir4096": [wp.design_fir("lp", 4096, 2000)],
        "lp8": [wp.design_butterworth("lp", 8, 2000)],
    }[chain_kind]
    bound = wp.Chain(stages).bind(fs).stages
    C, N = 3, 30011 if pads[0] % 4 else 30020  # aligned case: N % 4 == 0, N % 64 != 0
    rng = np.random.default_rng(17)
    x = rng.standard_normal((C, N)).astype(np.float32)
    ldx, ldy = N + pads[0], N + pads[1]
    xd = torch.zeros((C, ldx), dtype=torch.float32, device="cuda")
    xd[:, :N] = torch.from_numpy(x)
    yd = torch.full((C, ldy), 7.0, dtype=torch.float32, device="cuda")
    plan = engine.plan_for(bound, device=0)
    nb = plan.workspace_bytes(C, N)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    plan.execute(xd.data_ptr(), yd.data_ptr(), C, N, ldx, ldy, ws.data_ptr(), nb, torch.cuda.current_stream().cuda_stream)
    got = yd.cpu().numpy()
    assert np.all(got[:, N:] == 7.0)  # padding untouched
    ref = oracle.pipe(x.astype(np.float64), bound)
    tol = FIR_TOL if chain_kind.startswith("fir") else IIR_TOL
    assert oracle.parity_error(got[:, :N].astype(np.float64), ref) <= tol


@pytest.mark.gpu
def test_many_channels_lp8_subset_parity():
    fs = 48000
    w = wp.white_noise(0.4, 300, fs, seed=33)
    lp8 = wp.design_butterworth("lp", 8, 2000)
    y = (w | lp8).samples
    for c in (0, 1, 150, 299):
        ref = oracle.pipe(w.samples[c:c + 1], [lp8.bind(fs)])
        assert oracle.parity_error(y[c:c + 1], ref) <= IIR_TOL, c


# ---- chain passes: single-pass chain_lb


@pytest.mark.gpu
@pytest.mark.parametrize("order", [2, 4, 6, 8])
@pytest.mark.parametrize("precision", ["f32", "f64"])
@pytest.mark.parametrize("taps", [2, 16, 101, 129])
def test_chain_pass_matrix_vs_oracle(order, precision, taps):
    """Every section count x scan dtype x FIR length the tensor-core chain
    accepts, on ragged frame counts around the 8192-sample tile."""
    fs = 48000
    kind = "hp" if order % 4 == 0 else "lp"
    # f32 scans only for moderate pole radii (the planner picks f64 above 0.98)
    fc = (150 if precision == "f64" else 1500) if kind == "hp" else 3000
    stages = [wp.design_butterworth(kind, order, fc, fs),
              wp.design_fir("lp", taps, 12000, fs=fs) if taps > 2 else wp.FirFilter.from_taps([0.75, 0.25], fs),
              wp.Gain(0.5)]
    rng = np.random.default_rng(order * 1000 + taps)
    wp.set_iir_precision(precision)
    try:
        for frames in (8191, 8193, 40001):
            w = wp.Wave(rng.standard_normal((3, frames)), fs)
            y = wp.pipe(w, wp.Chain(stages)).samples
            ref = oracle.pipe(w.samples, wp.Chain(stages).bind(fs).stages)
            assert oracle.parity_error(y, ref) <= IIR_TOL, (frames, precision)
    finally:
        wp.set_iir_precision("auto")


@pytest.mark.gpu
@pytest.mark.parametrize("order", [1, 4, 8])
def test_chain_pass_iir_only_forced(order, monkeypatch):
    """IIR-only passes through chain_lb (H = 0, K = 64) at a size where the
    default planner keeps the fused kernel (WP_CHAIN_IMPL=lb forces it)."""
    import torch

    fs = 48000
    filt = wp.design_butterworth("lp", order, 2000, fs)
    bound = wp.Chain([filt]).bind(fs).stages
    monkeypatch.setenv("WP_CHAIN_IMPL", "lb")
    plan = _native.Plan(tuple(wp.engine._entry(s) for s in bound))  # uncached: the env var applies
    assert "chain_lb" in plan.describe_for(5, 60001)[0]
    rng = np.random.default_rng(order)
    C, N = 5, 60001
    x = rng.standard_normal((C, N)).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    nb = plan.workspace_bytes(C, N)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    plan.execute(xd.data_ptr(), yd.data_ptr(), C, N, N, N, ws.data_ptr(), nb, torch.cuda.current_stream().cuda_stream)
    ref = oracle.iir_cascade(filt.sos_rows(), x.astype(np.float64))
    assert oracle.parity_error(yd.cpu().numpy().astype(np.float64), ref) <= IIR_TOL


@pytest.mark.gpu
def test_chain_pass_stopband_input_f64():
    """The hard case for the state term: a low-frequency sine through cfg3's
    100 Hz high-pass, where the output is the small difference of the window
    and state terms."""
    fs = 48000
    n = np.arange(3 * 8192 + 77)
    x = np.stack([0.9 * np.sin(2 * np.pi * 30 * n / fs), 0.5 * np.sin(2 * np.pi * 12 * n / fs + 1.0)])
    stages = _cfg3()
    y = wp.pipe(wp.Wave(x, fs), wp.Chain(stages)).samples
    ref = oracle.pipe(np.asarray(x, np.float32).astype(np.float64), wp.Chain(stages).bind(fs).stages)
    assert oracle.parity_error(y, ref) <= IIR_TOL


@pytest.mark.gpu
def test_multi_pass_chain_normalize_chain():
    """chain pass -> Normalize -> chain pass: ping-pong buffers, workspace reuse
    and workspace reuse between consecutive single-pass chains."""
    fs = 48000
    stages = [wp.design_butterworth("hp", 4, 120, fs), wp.design_fir("lp", 33, 9000, fs=fs), wp.Normalize(0.8),
              wp.design_chebyshev1("lp", 4, 1.0, 6000, fs), wp.design_fir("lp", 65, 12000, fs=fs), wp.Gain(0.5)]
    rng = np.random.default_rng(41)
    w = wp.Wave(rng.standard_normal((3, 50001)), fs)
    from paper_2504_08624_b200 import engine

    plan = engine.plan_for(wp.Chain(stages).bind(fs).stages, device=0)
    desc = plan.describe_for(3, 50001)
    assert len(desc) == 3 and "chain_lb" in desc[0] and desc[1].startswith("normalize") and "chain_lb" in desc[2]
    y = wp.pipe(w, wp.Chain(stages)).samples
    ref = oracle.pipe(w.samples, wp.Chain(stages).bind(fs).stages)
    assert oracle.parity_error(y, ref) <= IIR_TOL


@pytest.mark.gpu
def test_plan_execute_in_cuda_graph():
    """plan.execute never allocates or synchronises, so a chain pass (record
    memset + chain_lb) can be captured once and replayed."""
    import torch

    from paper_2504_08624_b200 import engine

    fs = 48000
    bound = wp.Chain(_cfg3()).bind(fs).stages
    plan = engine.plan_for(bound, device=0)
    C, N = 4, 100003
    rng = np.random.default_rng(9)
    x = torch.from_numpy(rng.standard_normal((C, N)).astype(np.float32)).cuda()
    y_eager = torch.empty_like(x)
    y_graph = torch.full_like(x, 3.0)
    nb = plan.workspace_bytes(C, N)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        plan.execute(x.data_ptr(), y_eager.data_ptr(), C, N, N, N, ws.data_ptr(), nb, s.cuda_stream)  # warm-up
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        plan.execute(x.data_ptr(), y_graph.data_ptr(), C, N, N, N, ws.data_ptr(), nb,
                     torch.cuda.current_stream().cuda_stream)
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y_graph, y_eager)
    ref = oracle.pipe(x.double().cpu().numpy(), bound)
    assert oracle.parity_error(y_graph.double().cpu().numpy(), ref) <= IIR_TOL


@pytest.mark.gpu
def test_fir_passes_back_to_back_programmatic_launch():
    """Two FIR-only tensor-core passes in a row (the second reads the first's
    output) eagerly and captured in one CUDA graph, replayed with NEW input: the
    programmatic dependent launch must still order the second kernel after the
    first one's stores (griddepcontrol.wait before any read of the signal)."""
    import torch

    from paper_2504_08624_b200 import engine

    fs = 48000
    pa = engine.plan_for(wp.Chain([wp.design_fir("lp", 101, 9000)]).bind(fs).stages, device=0)
    pb = engine.plan_for(wp.Chain([wp.design_fir("hp", 31, 300)]).bind(fs).stages, device=0)
    assert "fir_tc" in pa.describe()[0] and "fir_tc" in pb.describe()[0]
    C, N = 6, 1 << 20
    rng = np.random.default_rng(21)
    x = torch.from_numpy(rng.standard_normal((C, N)).astype(np.float32)).cuda()
    mid = torch.empty_like(x)
    out = torch.empty_like(x)
    na, nb = pa.workspace_bytes(C, N), pb.workspace_bytes(C, N)
    wsa = torch.empty(max(na, 1), dtype=torch.uint8, device="cuda")
    wsb = torch.empty(max(nb, 1), dtype=torch.uint8, device="cuda")

    def run(st):
        pa.execute(x.data_ptr(), mid.data_ptr(), C, N, N, N, wsa.data_ptr(), na, st)
        pb.execute(mid.data_ptr(), out.data_ptr(), C, N, N, N, wsb.data_ptr(), nb, st)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            run(s.cuda_stream)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    eager = out.clone()
    ref = oracle.pipe(x.double().cpu().numpy(), wp.Chain([wp.design_fir("lp", 101, 9000),
                                                          wp.design_fir("hp", 31, 300)]).bind(fs).stages)
    assert oracle.parity_error(eager.double().cpu().numpy(), ref) <= 2 * FIR_TOL
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run(torch.cuda.current_stream().cuda_stream)
    x.copy_(torch.from_numpy(rng.standard_normal((C, N)).astype(np.float32)))
    out.fill_(5.0)
    g.replay()
    torch.cuda.synchronize()
    ref2 = oracle.pipe(x.double().cpu().numpy(), wp.Chain([wp.design_fir("lp", 101, 9000),
                                                           wp.design_fir("hp", 31, 300)]).bind(fs).stages)
    assert oracle.parity_error(out.double().cpu().numpy(), ref2) <= 2 * FIR_TOL


# ---- LTI fuser coverage: whole runs of IIR / FIR / gain stages in one pass ----


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["bench_chain_8sos", "fir_then_iir", "iir_fir241_gain", "two_firs_iir",
                                  "iir_long_fir_split"])
def test_fuser_passes_and_parity(name):
    """The reference's mixed FIR -> IIR chain (test_chain.py:167-173) runs as ONE
    pass, its pinned 8-SOS chain (bench.py:93-100) as two balanced 4-section
    passes (measured faster than one 8-section pass; test_eight_sections_one_pass
    covers the single-pass form); a FIR too long for the single-pass kernel gets
    its own FIR-only pass after the IIR pass."""
    fs = 44100 if name in ("bench_chain_8sos", "fir_then_iir") else 48000
    chains = {
        "bench_chain_8sos": (_bench_chain(), 2),  # 4 + 4 sections: 1.86x faster than one 8-section pass
        "fir_then_iir": ([wp.design_fir("lowpass", 33, 4000), wp.design_peaking(1000, gain_db=2.0)], 1),
        "iir_fir241_gain": ([wp.design_chebyshev1("lp", 4, 1.0, 5000), wp.design_fir("lp", 241, 9000), wp.Gain(0.7)], 1),
        "two_firs_iir": ([wp.design_fir("lp", 61, 9000), wp.design_butterworth("hp", 2, 80),
                          wp.design_fir("lp", 41, 12000)], 1),
        "iir_long_fir_split": ([wp.design_butterworth("hp", 4, 100), wp.design_fir("lp", 8193, 3000)], 2),
    }
    stages, passes = chains[name]
    bound = wp.Chain(stages).bind(fs).stages
    from paper_2504_08624_b200 import engine

    plan = engine.plan_for(bound, device=0)
    assert plan.num_passes == passes, plan.describe()
    rng = np.random.default_rng(len(name))
    w = wp.Wave(rng.standard_normal((3, 70001)), fs)
    y = wp.pipe(w, wp.Chain(stages)).samples
    ref = oracle.pipe(w.samples, bound)
    assert oracle.parity_error(y, ref) <= IIR_TOL
    # pipe == stage-by-stage application (the reference's chain/step coherence)
    step = w
    for st in bound:
        step = st.apply(step)
    assert np.array_equal(step.samples, y)


@pytest.mark.gpu
@pytest.mark.parametrize("taps, strategy", [(15361, "auto"), (20001, "auto"), (40961, "fft"), (9001, "direct")])
def test_long_fir_any_length(taps, strategy):
    """FIRs longer than one 16 K-point overlap-save block (> 15361 taps) run as
    accumulating 8192-tap segments (the reference's FFT strategy takes any tap
    count, engine.py:206-233); a forced-direct FIR past the fused direct kernel's
    reach also takes the FFT path. Parity vs the direct oracle at the FIR bar."""
    from paper_2504_08624_b200 import engine

    fs = 48000
    f = wp.design_fir("lp", taps, 3000, fs=fs)
    plan = engine.plan_for(wp.Chain([f]).bind(fs).stages, device=0, strategy=strategy)
    desc = plan.describe()[0]
    assert desc.startswith("fft_ols"), desc
    segs = int(desc.split("segments=")[1].split()[0])
    assert segs == (1 if taps <= 15361 else -(-taps // 8192)), desc
    rng = np.random.default_rng(taps)
    w = wp.Wave(rng.standard_normal((3, 50001)), fs)
    y = wp.apply_fir(f, w, strategy=strategy).samples
    ref = oracle.fir_direct(f.taps, w.samples)
    assert oracle.parity_error(y, ref) <= FIR_TOL


@pytest.mark.gpu
def test_iir_then_very_long_fir():
    """IIR pass followed by a 30000-tap FIR pass (3 accumulating FFT segments)."""
    fs = 48000
    stages = [wp.design_butterworth("hp", 2, 50), wp.design_fir("lp", 30001, 5000)]
    rng = np.random.default_rng(3)
    w = wp.Wave(rng.standard_normal((2, 60001)), fs)
    y = wp.pipe(w, wp.Chain(stages)).samples
    ref = oracle.pipe(w.samples, wp.Chain(stages).bind(fs).stages)
    assert oracle.parity_error(y, ref) <= IIR_TOL


@pytest.mark.gpu
def test_catalog_stages_one_pass():
    """shelves, peaking EQ, a band-pass and a high-pass windowed-sinc
    FIR and gains fuse into chain passes and match the oracle."""
    from paper_2504_08624_b200 import engine

    fs = 48000
    stages = [wp.design_shelf("lo_shelf", 200, gain_db=4.0), wp.design_peaking(2500, gain_db=-6.0, q=2.0),
              wp.design_fir("bandpass", 129, (300, 6000)), wp.design_shelf("hi_shelf", 9000, gain_db=-3.0),
              wp.Gain(0.8), wp.design_fir("highpass", 31, 100)]
    bound = wp.Chain(stages).bind(fs).stages
    plan = engine.plan_for(bound, device=0)
    assert plan.num_passes == 1, plan.describe()
    assert plan.describe()[0].startswith("chain_lb"), plan.describe()
    rng = np.random.default_rng(85)
    w = wp.Wave(rng.standard_normal((4, 90001)), fs)
    y = wp.pipe(w, wp.Chain(stages)).samples
    ref = oracle.pipe(w.samples, bound)
    assert oracle.parity_error(y, ref) <= IIR_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("maxs, passes", [(8, 1), (5, 2), (3, 3)])
def test_eight_sections_one_pass(maxs, passes, monkeypatch):
    """WP_LB_MAXS caps the sections per chain_lb pass: the reference's 8-SOS bench
    chain as ONE 16-state pass (D = 16 kernel), as 5 + 3 and as 3 + 3 + 2, all
    within the IIR bar of the oracle."""
    from paper_2504_08624_b200 import engine

    monkeypatch.setenv("WP_LB_MAXS", str(maxs))
    monkeypatch.setenv("WP_CHAIN_IMPL", "lb")  # chain_lb even for the small 2-section remainder
    fs = 44100
    bound = wp.Chain(_bench_chain()).bind(fs).stages
    plan = _native.Plan(tuple(engine._entry(s) for s in bound))  # uncached: the env var applies
    assert plan.num_passes == passes, plan.describe()
    assert all(d.startswith("chain_lb") for d in plan.describe_for(3, 90001)), plan.describe()
    rng = np.random.default_rng(maxs)
    x = rng.standard_normal((3, 90001)).astype(np.float32)
    import torch

    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    nb = plan.workspace_bytes(3, 90001)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    plan.execute(xd.data_ptr(), yd.data_ptr(), 3, 90001, 90001, 90001, ws.data_ptr(), nb,
                 torch.cuda.current_stream().cuda_stream)
    ref = oracle.pipe(x.astype(np.float64), bound)
    assert oracle.parity_error(yd.cpu().numpy().astype(np.float64), ref) <= IIR_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("sections,taps", [(4, 193), (5, 193), (6, 129), (7, 65), (8, 65)])
def test_fusion_reach_unchanged_by_output_staging(sections, taps, monkeypatch):
    """IIR + FIR passes keep their one-pass reach: the TMA output staging is laid
    out only where it fits next to the operands (else the LDS/STG staging).
    More than 5 sections are split by default (measured faster): WP_LB_MAXS=8
    asks for the one-pass form the reach is about."""
    from paper_2504_08624_b200 import engine

    if sections > 5:
        monkeypatch.setenv("WP_LB_MAXS", "8")
    fs = 48000
    iir = wp.design_butterworth("lp", 2 * sections, 3000 + 7 * taps)  # distinct plans (no cache hits)
    fir = wp.design_fir("lp", taps, 9000)
    bound = wp.Chain([iir, fir]).bind(fs).stages
    plan = engine.plan_for(bound, device=0)
    desc = plan.describe_for(4, 8192 * 20)
    assert plan.num_passes == 1 and desc[0].startswith("chain_lb"), desc
    w = wp.white_noise(0.2, 2, fs, seed=5)
    y = wp.pipe(w, wp.Chain([iir, fir])).samples
    assert oracle.parity_error(y, oracle.pipe(w.samples, bound)) <= IIR_TOL


@pytest.mark.gpu
def test_iir_fir_iir_too_large_for_one_pass():
    """IIR(1) | FIR(252) | IIR(4): 5 sections + a 252-tap FIR do not fit one
    chain_lb pass; the planner closes the pass instead of handing the CUDA-core
    fused kernel a configuration it cannot hold (found by tools/stress_random.py)."""
    from paper_2504_08624_b200 import engine

    fs = 48000
    rng = np.random.default_rng(1971)
    stages = [wp.design_butterworth("hp", 2, 200), wp.FirFilter.from_taps(rng.uniform(-1, 1, 252) / 16, fs),
              wp.design_chebyshev1("lp", 8, 0.5, 9000)]
    bound = wp.Chain(stages).bind(fs).stages
    plan = engine.plan_for(bound, device=0)
    assert plan.num_passes >= 2
    w = wp.white_noise(0.5, 3, fs, seed=4)
    y = wp.pipe(w, wp.Chain(stages)).samples
    assert oracle.parity_error(y, oracle.pipe(w.samples, bound)) <= IIR_TOL
