"""CPU: drop-in API behaviour that needs no GPU (the reference's chain /
wave / engine contract: test_chain.py, test_wave.py, test_engine.py).

Waves built on the host stay on the host until their samples are needed, so
the lazy pipe, binding and validation logic are all testable here; running
the recorded chain needs the sm_100a library and a device (tests marked gpu).
"""

import numpy as np
import pytest

import paper_2504_08624_b200 as wp
from paper_2504_08624_b200 import engine
from paper_2504_08624_b200.chain import Chain

from conftest import random_unbound_stage

FS = 44100


def shelf_pair():
    return wp.design_shelf("hi_shelf", 1000, gain_db=3.0), wp.design_shelf("lo_shelf", 2000, gain_db=3.0)


class TestWave:
    def test_shape_and_props(self):
        w = wp.Wave([[0.0, 0.5, -1.0]], fs=8000)
        assert (w.channels, w.frames) == (1, 3)
        assert w.duration == pytest.approx(3 / 8000)

    def test_1d_is_single_channel(self):
        assert wp.Wave([0.0, 1.0], fs=FS).samples.shape == (1, 2)

    def test_immutable_and_readonly(self):
        w = wp.Wave([[1.0, 2.0]], fs=FS)
        with pytest.raises(ValueError):
            w.samples[0, 0] = 9.0
        with pytest.raises(AttributeError):
            w.fs = 48000

    def test_constructor_copies(self):
        buf = np.zeros((2, 4))
        w = wp.Wave(buf, fs=FS)
        buf[0, 0] = 5.0
        assert w.samples[0, 0] == 0.0

    def test_float32_canonical_values(self):
        x = np.array([[0.1, 1.0 / 3.0]])
        assert np.array_equal(wp.Wave(x, FS).samples, x.astype(np.float32).astype(np.float64))

    def test_equality_and_hash(self):
        a = wp.Wave([[1.0, 2.0]], fs=FS)
        assert a == wp.Wave([[1.0, 2.0]], fs=FS)
        assert a != wp.Wave([[1.0, 2.0]], fs=48000)
        assert a != wp.Wave([[1.0, 3.0]], fs=FS)
        assert hash(a) == hash(wp.Wave([[1.0, 2.0]], fs=FS))

    @pytest.mark.parametrize("fs", [0, -1, 44100.5, True])
    def test_bad_fs(self, fs):
        with pytest.raises(wp.InvalidArgument):
            wp.Wave([[0.0]], fs=fs)

    def test_empty_rejected(self):
        with pytest.raises(wp.InvalidArgument):
            wp.Wave(np.zeros((1, 0)), fs=FS)
        with pytest.raises(wp.InvalidArgument):
            wp.Wave(np.zeros((0, 5)), fs=FS)
        with pytest.raises(wp.InvalidArgument):
            wp.Wave(np.zeros((2, 2, 2)), fs=FS)

    def test_channel_view(self):
        w = wp.Wave(np.arange(6.0).reshape(2, 3), FS)
        assert np.array_equal(w.channel(1).samples, [[3.0, 4.0, 5.0]])

    @pytest.mark.parametrize("kw", [dict(duration_s=0, channels=1, fs=FS), dict(duration_s=1, channels=0, fs=FS),
                                    dict(duration_s=1e-9, channels=1, fs=FS)])
    def test_white_noise_validation(self, kw):
        with pytest.raises(wp.InvalidArgument):
            wp.white_noise(seed=1, **kw)


class TestLazyPipe:
    def test_pipe_records_without_running(self):
        w = wp.Wave(np.zeros((2, 64)), FS)
        y = w | wp.design_butterworth("lp", 2, 1000) | wp.design_fir("lp", 9, 3000) | wp.Gain(0.5)
        assert y.is_lazy and y.pending_stages == 3
        assert (y.channels, y.frames, y.fs) == (2, 64, FS)

    def test_lazy_merges_across_pipes(self):
        w = wp.Wave(np.zeros((1, 16)), FS)
        f, g = shelf_pair()
        a = wp.pipe(wp.pipe(w, f), g)
        b = wp.pipe(w, wp.compose(f, g))
        assert a._src is w and b._src is w
        assert engine._key(a._entries) == engine._key(b._entries)

    def test_binding_errors_raise_at_pipe_time(self):
        w = wp.Wave(np.zeros((1, 16)), 44100)
        with pytest.raises(wp.SampleRateMismatch):
            w | wp.design_peaking(500, gain_db=1.0, fs=48000)
        with pytest.raises(wp.InvalidCutoff):
            w | wp.design_butterworth("lp", 4, 30000)
        with pytest.raises(wp.InvalidArgument):
            wp.pipe("wave", wp.design_peaking(500, gain_db=1.0))

    def test_apply_validation(self):
        w = wp.Wave(np.zeros((1, 16)), FS)
        with pytest.raises(wp.UnboundFilter):
            wp.apply_iir(wp.design_butterworth("lp", 4, 1000), w)
        with pytest.raises(wp.SampleRateMismatch):
            wp.apply_iir(wp.design_butterworth("lp", 4, 1000, 48000), w)
        with pytest.raises(wp.InvalidArgument):
            wp.apply_iir(wp.design_butterworth("lp", 4, 1000, FS), w, backend="gpu")
        with pytest.raises(wp.InvalidArgument):
            wp.apply_fir(wp.design_fir("lp", 9, 1000, fs=FS), w, strategy="winograd")

    def test_gain_folds_into_entries(self):
        w = wp.Wave(np.zeros((1, 16)), FS)
        y = w | wp.Gain(0.25) | wp.design_fir("lp", 9, 3000) | wp.Gain(2.0)
        kinds = [e[0] for e in y._entries]
        assert kinds == [3, 2, 3]

    def test_custom_stage_is_eager(self):
        calls = []

        class Probe:
            def bind(self, fs):
                return self

            def apply(self, wave, backend="auto"):
                calls.append(backend)
                return wave

        w = wp.Wave(np.ones((1, 8)), FS)
        out = wp.pipe(w, Probe(), backend="serial")
        assert calls == ["serial"] and out is w


class TestCompose:
    def test_two_stage_chain(self):
        hi, lo = shelf_pair()
        chain = wp.compose(hi, lo)
        assert len(chain) == 2 and not chain.bound

    def test_flatten_and_associativity(self):
        f, g = shelf_pair()
        h = wp.design_peaking(4000, gain_db=-2.0)
        assert wp.compose(wp.compose(f, g), h).stages == wp.compose(f, wp.compose(g, h)).stages
        assert len(wp.compose(wp.compose(f, g), wp.compose(h, Chain()))) == 3

    def test_bound_unbound_merge_and_conflict(self):
        bound = wp.design_peaking(500, gain_db=1.0, q=1.0, fs=FS)
        chain = wp.compose(bound, wp.design_peaking(900, gain_db=1.0, q=1.0))
        assert chain.bound and chain.binding == FS
        with pytest.raises(wp.SampleRateMismatch):
            wp.compose(wp.design_peaking(500, gain_db=1.0, fs=44100), wp.design_peaking(500, gain_db=1.0, fs=48000))

    def test_operator_or_and_non_stage(self):
        hi, lo = shelf_pair()
        assert isinstance(hi | lo, Chain)
        with pytest.raises(wp.InvalidArgument):
            wp.compose(wp.design_peaking(500, gain_db=1.0), "not a filter")

    def test_chain_with_gain_reports_binding(self):
        chain = wp.compose(wp.design_butterworth("lp", 2, 1000, FS), wp.Gain(0.5))
        assert chain.bound and chain.binding == FS

    def test_bind_idempotent_and_prebound_conflict(self):
        chain = Chain(shelf_pair())
        once = chain.bind(FS)
        assert once.bind(FS).stages == once.stages
        with pytest.raises(wp.SampleRateMismatch):
            Chain([wp.design_peaking(500, gain_db=1.0, fs=48000)]).bind(44100)

    def test_response_is_product(self):
        chain = Chain(shelf_pair()).bind(FS)
        freqs = np.geomspace(10, FS / 2, 16)
        expect = wp.frequency_response(chain.stages[0], freqs) * wp.frequency_response(chain.stages[1], freqs)
        np.testing.assert_allclose(chain.frequency_response(freqs), expect, rtol=1e-12)
        with pytest.raises(wp.UnboundFilter):
            Chain(shelf_pair()).frequency_response([100.0])


def test_algebra_structure_random_chains():
    for seed in range(50):
        rng = np.random.default_rng(seed)
        left = Chain([random_unbound_stage(rng) for _ in range(int(rng.integers(0, 3)))])
        right = Chain([random_unbound_stage(rng) for _ in range(int(rng.integers(1, 3)))])
        composed = wp.compose(left, right)
        assert len(composed) == len(left) + len(right)
        bound = composed.bind(FS)
        assert bound.bind(FS).stages == bound.stages


class TestEngineKnobs:
    def test_resolution_rules(self):
        assert engine._resolve_backend("auto", 1, 100_000) == "serial"
        assert engine._resolve_backend("auto", 2, 100_000) == "parallel"
        assert engine._resolve_strategy("auto", 129, 4097) == "fft"
        assert engine._resolve_strategy("auto", 128, 100_000) == "direct"
        with pytest.raises(wp.InvalidArgument):
            engine._resolve_backend("gpu", 1, 1)

    def test_thread_shim(self):
        prev = engine.get_num_threads()
        try:
            assert engine.set_num_threads(10_000) == engine.max_threads()
            assert engine.set_num_threads(1) == 1
            with pytest.raises(wp.InvalidArgument):
                engine.set_num_threads(0)
        finally:
            engine.set_num_threads(prev)

    def test_no_cpu_fallback(self):
        with pytest.raises(wp.InvalidArgument):
            wp.set_jit_enabled(False)
        with pytest.raises(wp.InvalidArgument):
            wp.set_iir_precision("f16")

    def test_iir_oracle_api(self):
        np.testing.assert_array_equal(wp.iir_oracle([1.0], [1.0, -1.0], np.ones(5)), [1, 2, 3, 4, 5])
        with pytest.raises(wp.InvalidCoefficients):
            wp.iir_oracle([1.0], [2.0, 0.0], np.ones(3))
        with pytest.raises(wp.InvalidArgument):
            wp.iir_oracle([1.0], [1.0], np.ones((2, 3)))
