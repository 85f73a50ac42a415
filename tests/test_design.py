"""CPU: host-side coefficient design matches the reference bit for bit
(fixtures from make_golden.py) and the reference's frozen tool values
(pkg/tests/test_design.py:13-29)."""

import math

import numpy as np
import pytest

import paper_2504_08624_b200 as wp

FS = 44100

REF_CHEBY1_4_1DB_2000 = (
    [8.898545271346152e-05, 0.00035594181085384606, 0.0005339127162807691,
     0.00035594181085384606, 8.898545271346152e-05],
    [1.0, -3.651712987704756, 5.082417591635586, -3.191498904811017, 0.7623917940019291],
)
REF_BUTTER_4_1000 = (
    [2.1520951214109304e-05, 8.608380485643722e-05, 0.00012912570728465582,
     8.608380485643722e-05, 2.1520951214109304e-05],
    [1.0, -3.627844202190272, 4.95122513325103, -3.0119242815053817, 0.6888876856640502],
)
REF_LO_SHELF = ([0.9331406285426834, -1.5516066139004616, 0.6643406183509267],
                [1.0, -1.5287779671849073, 0.6203098936091647])


def expand_ba(f):
    b, a = np.array([f.overall_gain]), np.array([1.0])
    for s in f.sections:
        b = np.polymul(b, [s.b0, s.b1, s.b2])
        a = np.polymul(a, [1.0, s.a1, s.a2])
    return np.trim_zeros(b, "b"), np.trim_zeros(a, "b")


DESIGN_BUILDERS = {
    "cfg1_butter_lp4_1000_44100": lambda: wp.design_butterworth("lp", 4, 1000, 44100),
    "cfg3_butter_hp4_100_48000": lambda: wp.design_butterworth("hp", 4, 100, 48000),
    "cfg3_cheby1_lp4_1db_8000_48000": lambda: wp.design_chebyshev1("lp", 4, 1.0, 8000, 48000),
    "cfg5_butter_lp8_2000_48000": lambda: wp.design_butterworth("lp", 8, 2000, 48000),
    "butter_hp3_1000_44100": lambda: wp.design_butterworth("hp", 3, 1000, 44100),
    "cheby1_hp5_0.5db_3000_44100": lambda: wp.design_chebyshev1("hp", 5, 0.5, 3000, 44100),
    "lo_shelf_2000_-6_0.707_44100": lambda: wp.design_shelf("lo_shelf", 2000, -6.0, 0.707, 44100),
    "hi_shelf_1000_6_0.707_44100": lambda: wp.design_shelf("hi_shelf", 1000, 6.0, 0.707, 44100),
    "peaking_1000_12_1_44100": lambda: wp.design_peaking(1000, 12.0, 1.0, 44100),
}
FIR_BUILDERS = {
    "cfg2_fir_lp101_1000_hamming_48000": lambda: wp.design_fir("lp", 101, 1000, "hamming", 48000),
    "cfg3_fir_lp101_15000_hamming_48000": lambda: wp.design_fir("lp", 101, 15000, "hamming", 48000),
    "cfg4_fir_lp4096_2000_hamming_48000": lambda: wp.design_fir("lp", 4096, 2000, "hamming", 48000),
    "fir_hp65_3000_blackman_44100": lambda: wp.design_fir("hp", 65, 3000, "blackman", 44100),
    "fir_bp129_500_4000_rect_44100": lambda: wp.design_fir("bp", 129, (500, 4000), "rect", 44100),
}


@pytest.mark.parametrize("name", sorted(DESIGN_BUILDERS))
def test_iir_designs_match_reference(name, golden_designs):
    f = DESIGN_BUILDERS[name]()
    ref = golden_designs[name]
    rows = np.array([[s.b0, s.b1, s.b2, s.a1, s.a2] for s in f.sections])
    np.testing.assert_allclose(rows, np.array(ref["sections"]), rtol=0, atol=1e-14)
    assert f.overall_gain == pytest.approx(ref["overall_gain"], rel=1e-13)


@pytest.mark.parametrize("name", sorted(FIR_BUILDERS))
def test_fir_designs_match_reference(name, golden_designs):
    np.testing.assert_allclose(FIR_BUILDERS[name]().taps, golden_designs[name]["taps"], rtol=0, atol=1e-15)


def test_frozen_reference_tool_values():
    b, a = expand_ba(wp.design_butterworth("lowpass", 4, 1000, FS))
    np.testing.assert_allclose(b, REF_BUTTER_4_1000[0], atol=1e-8)
    np.testing.assert_allclose(a, REF_BUTTER_4_1000[1], atol=1e-8)
    b, a = expand_ba(wp.design_chebyshev1("lowpass", 4, 1.0, 2000, FS))
    np.testing.assert_allclose(b, REF_CHEBY1_4_1DB_2000[0], atol=1e-8)
    np.testing.assert_allclose(a, REF_CHEBY1_4_1DB_2000[1], atol=1e-8)
    lo = wp.design_shelf("lo_shelf", 2000, gain_db=-6.0, q=0.707, fs=FS)
    s = lo.sections[0]
    np.testing.assert_allclose([s.b0, s.b1, s.b2], REF_LO_SHELF[0], atol=1e-12)
    np.testing.assert_allclose([1.0, s.a1, s.a2], REF_LO_SHELF[1], atol=1e-12)


def test_analytic_properties():
    for order in (2, 4, 8):
        f = wp.design_butterworth("lowpass", order, 1000, FS)
        assert abs(wp.frequency_response(f, [1000.0])[0]) == pytest.approx(1 / math.sqrt(2), abs=1e-9)
        assert abs(wp.frequency_response(f, [0.0])[0]) == pytest.approx(1.0, abs=1e-12)
    f = wp.design_butterworth("lowpass", 8, 4000, FS)
    radii = [wp.design.pole_radius(s) for s in f.sections]
    assert radii == sorted(radii)
    assert sum(wp.design_fir("lp", 101, 1000, fs=48000).taps) == pytest.approx(1.0, abs=1e-12)


def test_design_errors():
    with pytest.raises(wp.InvalidOrder):
        wp.design_butterworth("lowpass", 0, 1000, FS)
    with pytest.raises(wp.InvalidCutoff):
        wp.design_butterworth("lowpass", 2, 30000, FS)
    with pytest.raises(wp.InvalidArgument):
        wp.design_butterworth("bandpass", 2, 1000, FS)
    with pytest.raises(wp.InvalidRipple):
        wp.design_chebyshev1("lp", 2, 0.0, 1000, FS)
    with pytest.raises(wp.InvalidTapCount):
        wp.design_fir("hp", 64, 1000, fs=FS)
    with pytest.raises(wp.InvalidQ):
        wp.design_peaking(1000, 3.0, q=0.0)
    with pytest.raises(wp.InvalidCoefficients):
        wp.BiquadSection(1.0, 0.0, 0.0, 0.0, 1.0)


def test_lazy_binding_equals_eager():
    lazy = wp.compose(wp.design_butterworth("lp", 4, 1000), wp.Chain()).bind(FS)
    eager = wp.design_butterworth("lp", 4, 1000, FS)
    assert lazy.stages[0].sections == eager.sections
    assert lazy.stages[0].overall_gain == eager.overall_gain


def test_pole_radius_threshold_pins():
    """The fp64 precision switch (pole radius > 0.98) triggers exactly for
    cfg3's 100 Hz high-pass and not for the low-pass configs."""
    hp = wp.design_butterworth("hp", 4, 100, 48000)
    assert max(wp.design.pole_radius(s) for s in hp.sections) > 0.98
    for f in (wp.design_butterworth("lp", 4, 1000, 44100), wp.design_butterworth("lp", 8, 2000, 48000),
              wp.design_chebyshev1("lp", 4, 1.0, 8000, 48000)):
        assert max(wp.design.pole_radius(s) for s in f.sections) < 0.98


def test_gain_and_normalize_stages():
    g = wp.Gain(gain_db=-6.0206)
    assert g.factor == pytest.approx(0.5, rel=1e-4)
    assert not g.bound and g.bind(48000).fs == 48000
    with pytest.raises(wp.SampleRateMismatch):
        g.bind(48000).bind(44100)
    with pytest.raises(wp.InvalidArgument):
        wp.Gain()
    with pytest.raises(wp.InvalidArgument):
        wp.Normalize(0.0)
    assert np.allclose(wp.frequency_response(wp.Gain(2.0, fs=FS), [0.0, 100.0]), 2.0)


def test_bind_memoised_per_spec_and_rate():
    """Binding an unbound design reuses one immutable design per (spec, fs)
    (host-side cache; the coefficients equal a direct design)."""
    import paper_2504_08624_b200 as wp

    lp = wp.design_butterworth("lp", 4, 1000)
    a, b = lp.bind(44100), lp.bind(44100)
    assert a is b
    direct = wp.design_butterworth("lp", 4, 1000, 44100)
    assert np.array_equal(a.sos_rows(), direct.sos_rows())
    assert lp.bind(48000) is not a
    fir = wp.design_fir("lp", 101, 15000)
    assert fir.bind(48000) is fir.bind(48000)
    assert not fir.bind(48000).taps.flags.writeable
    with pytest.raises(wp.SampleRateMismatch):
        a.bind(48000)
