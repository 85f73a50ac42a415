"""FX stage objects and their (host-side) coefficient design.

Coefficient design is O(order) float64 arithmetic done once per filter, so it
stays on the host in numpy; only *application* runs on the GPU. The public
surface mirrors the reference's ``wavepipe.design`` (pkg/src/wavepipe/design.py)
so user code keeps working:

* ``BiquadSection`` (design.py:60-81), ``FilterSpec`` (:87-98),
  ``IirFilter`` (:101-149), ``FirFilter`` (:152-201);
* ``design_butterworth`` (:333-352), ``design_chebyshev1`` (:355-375),
  ``design_shelf`` (:378-419), ``design_peaking`` (:422-443),
  ``design_fir`` (:446-495), ``frequency_response`` (:552-570).

The algorithm is the reference's (analog prototype -> prewarp -> bilinear ->
sections paired in ascending pole radius, ties by angle), re-derived here in
closed form: a conjugate pole pair p, p* becomes the denominator
``1 - 2 Re(p) z^-1 + |p|^2 z^-2`` directly instead of via polynomial
expansion. Coefficients agree with the reference to ~1e-15 (checked against
fixtures in tests/golden/design.json).

Two stages the north star names but the reference only has as a test double
are added: ``Gain`` (the duck-typed stage of tests/test_chain.py:176-187) and
``Normalize`` (absent from the reference; semantics defined here, "parity
unpinned").
"""

from __future__ import annotations

import cmath
import functools
import math
from dataclasses import dataclass
from typing import Optional, Sequence, Union

import numpy as np

from .errors import (
    FrequencyOutOfRange,
    InvalidArgument,
    InvalidCoefficients,
    InvalidCutoff,
    InvalidOrder,
    InvalidQ,
    InvalidRipple,
    InvalidTapCount,
    SampleRateMismatch,
    UnboundFilter,
)

__all__ = [
    "DEFAULT_Q",
    "BiquadSection",
    "FilterSpec",
    "IirFilter",
    "FirFilter",
    "Gain",
    "Normalize",
    "design_butterworth",
    "design_chebyshev1",
    "design_shelf",
    "design_peaking",
    "design_fir",
    "frequency_response",
    "pole_radius",
]

DEFAULT_Q = 1.0 / math.sqrt(2.0)

_KINDS = {
    "lp": "lowpass",
    "lowpass": "lowpass",
    "hp": "highpass",
    "highpass": "highpass",
    "bp": "bandpass",
    "bandpass": "bandpass",
}
_WINDOWS = ("hamming", "blackman", "rect")
_REAL_EPS = 1e-12  # |imag| below this counts as a real root (design.py:284)


# ---------------------------------------------------------------------------
# value types
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class BiquadSection:
    """Second-order section with a0 == 1; rejected unless strictly stable."""

    b0: float
    b1: float
    b2: float
    a1: float
    a2: float

    def __post_init__(self):
        # stability triangle: both poles strictly inside the unit circle
        stable = abs(self.a2) < 1.0 and abs(self.a1) < 1.0 + self.a2
        if not stable:
            raise InvalidCoefficients(
                f"unstable section: a1={self.a1!r}, a2={self.a2!r} violates |a2|<1, |a1|<1+a2"
            )

    def as_row(self) -> np.ndarray:
        return np.array([self.b0, self.b1, self.b2, self.a1, self.a2], dtype=np.float64)


_IDENTITY = BiquadSection(1.0, 0.0, 0.0, 0.0, 0.0)


@dataclass(frozen=True)
class FilterSpec:
    """Design arguments retained so an unbound design can be bound later."""

    family: str
    kind: Optional[str] = None
    order: Optional[int] = None
    fc: Union[float, tuple, None] = None
    ripple_db: Optional[float] = None
    gain_db: Optional[float] = None
    q: Optional[float] = None
    window: Optional[str] = None


def pole_radius(section: BiquadSection) -> float:
    """Largest pole magnitude of ``1 + a1 z^-1 + a2 z^-2``."""
    disc = section.a1 * section.a1 - 4.0 * section.a2
    if disc < 0.0:
        return math.sqrt(section.a2)
    root = math.sqrt(disc)
    return max(abs(-section.a1 + root), abs(-section.a1 - root)) * 0.5


class _StageOps:
    """``|`` between stages composes a Chain (design.py:141-144)."""

    def __or__(self, other):
        from .chain import compose

        return compose(self, other)


@dataclass(frozen=True, eq=False)
class IirFilter(_StageOps):
    """Biquad cascade (bound) or a spec awaiting a sampling rate (unbound)."""

    sections: tuple
    overall_gain: float
    spec: Optional[FilterSpec]
    fs: Optional[int]

    def __post_init__(self):
        if self.fs is not None and not self.sections:
            raise InvalidArgument("bound IIR filter must have at least one section")
        if self.fs is None and self.sections:
            raise InvalidArgument("unbound IIR filter cannot carry sections")
        if self.fs is None and self.spec is None:
            raise InvalidArgument("unbound IIR filter needs a spec to bind later")

    @classmethod
    def from_sections(cls, sections: Sequence, fs: int, overall_gain: float = 1.0) -> "IirFilter":
        """User-supplied sections (tuples or BiquadSection), the raw escape hatch."""
        secs = tuple(s if isinstance(s, BiquadSection) else BiquadSection(*s) for s in sections)
        return cls(sections=secs, overall_gain=float(overall_gain), spec=None, fs=int(fs))

    @property
    def bound(self) -> bool:
        return self.fs is not None

    def bind(self, fs: int) -> "IirFilter":
        if self.fs is not None:
            if self.fs != fs:
                raise SampleRateMismatch(f"filter bound to {self.fs} Hz cannot rebind to {fs} Hz")
            return self
        return _design_iir_from_spec(self.spec, fs)

    def apply(self, wave, backend: str = "auto"):
        from .engine import apply_iir

        return apply_iir(self, wave, backend=backend)

    def sos_rows(self) -> np.ndarray:
        """``[S, 5]`` rows (b0,b1,b2,a1,a2) with the cascade gain folded into
        section 0's feed-forward taps, exactly as engine._sos_array does
        (engine.py:133-139)."""
        rows = np.array([s.as_row() for s in self.sections], dtype=np.float64)
        rows[0, :3] *= self.overall_gain
        return rows

    def __repr__(self) -> str:
        state = f"fs={self.fs}" if self.bound else "unbound"
        family = self.spec.family if self.spec else "raw"
        return f"IirFilter({family}, {len(self.sections)} sections, {state})"


@dataclass(frozen=True, eq=False)
class FirFilter(_StageOps):
    """Tap vector (bound) or windowed-sinc spec awaiting a rate (unbound)."""

    taps: Optional[np.ndarray]
    spec: Optional[FilterSpec]
    fs: Optional[int]

    def __post_init__(self):
        if self.fs is not None:
            if self.taps is None or len(self.taps) == 0:
                raise InvalidArgument("bound FIR filter must have taps")
            arr = np.array(self.taps, dtype=np.float64, order="C", copy=True).reshape(-1)
            arr.setflags(write=False)
            object.__setattr__(self, "taps", arr)
        else:
            if self.taps is not None:
                raise InvalidArgument("unbound FIR filter cannot carry taps")
            if self.spec is None:
                raise InvalidArgument("unbound FIR filter needs a spec to bind later")

    @classmethod
    def from_taps(cls, taps, fs: int) -> "FirFilter":
        return cls(taps=np.asarray(taps, dtype=np.float64), spec=None, fs=int(fs))

    @property
    def bound(self) -> bool:
        return self.fs is not None

    def bind(self, fs: int) -> "FirFilter":
        if self.fs is not None:
            if self.fs != fs:
                raise SampleRateMismatch(f"filter bound to {self.fs} Hz cannot rebind to {fs} Hz")
            return self
        return _design_fir_from_spec(self.spec, fs)

    def apply(self, wave, backend: str = "auto"):
        from .engine import apply_fir

        return apply_fir(self, wave, backend=backend)

    def __repr__(self) -> str:
        state = f"fs={self.fs}" if self.bound else "unbound"
        ntaps = len(self.taps) if self.taps is not None else "?"
        return f"FirFilter({ntaps} taps, {state})"


class _RateAgnostic(_StageOps):
    """Stages whose math ignores fs but which still track a binding, so a chain
    that contains them reports ``bound`` like one made only of filters."""

    __slots__ = ()

    @property
    def bound(self) -> bool:
        return self.fs is not None

    def _rebound(self, fs):
        raise NotImplementedError

    def bind(self, fs: int):
        if self.fs is not None:
            if self.fs != fs:
                raise SampleRateMismatch(f"stage bound to {self.fs} Hz cannot rebind to {fs} Hz")
            return self
        return self._rebound(int(fs))


class Gain(_RateAgnostic):
    """Flat scaling ``y = g * x`` (fp32 multiply on the device).

    The reference has this only as a duck-typed test stage
    (pkg/tests/test_chain.py:177-187: ``Wave(samples * factor)``). Give either
    a linear ``factor`` or ``gain_db`` (20 log10).
    """

    __slots__ = ("factor", "fs")

    def __init__(self, factor: Optional[float] = None, gain_db: Optional[float] = None, fs: Optional[int] = None):
        if (factor is None) == (gain_db is None):
            raise InvalidArgument("Gain needs exactly one of factor or gain_db")
        value = float(factor) if factor is not None else 10.0 ** (float(gain_db) / 20.0)
        if not math.isfinite(value):
            raise InvalidArgument(f"gain must be finite, got {value!r}")
        object.__setattr__(self, "factor", value)
        object.__setattr__(self, "fs", None if fs is None else int(fs))

    def __setattr__(self, name, value):
        raise AttributeError("Gain is immutable")

    def _rebound(self, fs):
        return Gain(self.factor, fs=fs)

    def apply(self, wave, backend: str = "auto"):
        from .engine import apply_stage

        return apply_stage(self, wave, backend=backend)

    def __eq__(self, other):
        return isinstance(other, Gain) and other.factor == self.factor and other.fs == self.fs

    def __hash__(self):
        return hash(("gain", self.factor, self.fs))

    def __repr__(self) -> str:
        return f"Gain({self.factor!r})"


class Normalize(_RateAgnostic):
    """Peak normalisation ``y = x * (peak / max|x|)`` over the whole Wave.

    Absent from the reference (parity unpinned); the
    semantics are defined here: the maximum is taken over every channel and
    frame, an all-zero input is returned unchanged. Runs as a device-side
    reduction followed by a scale that reads the peak from device memory (no
    host round trip).
    """

    __slots__ = ("peak", "fs")

    def __init__(self, peak: float = 1.0, fs: Optional[int] = None):
        peak = float(peak)
        if not (math.isfinite(peak) and peak > 0.0):
            raise InvalidArgument(f"normalize peak must be finite and > 0, got {peak!r}")
        object.__setattr__(self, "peak", peak)
        object.__setattr__(self, "fs", None if fs is None else int(fs))

    def __setattr__(self, name, value):
        raise AttributeError("Normalize is immutable")

    def _rebound(self, fs):
        return Normalize(self.peak, fs=fs)

    def apply(self, wave, backend: str = "auto"):
        from .engine import apply_stage

        return apply_stage(self, wave, backend=backend)

    def __eq__(self, other):
        return isinstance(other, Normalize) and other.peak == self.peak and other.fs == self.fs

    def __hash__(self):
        return hash(("normalize", self.peak, self.fs))

    def __repr__(self) -> str:
        return f"Normalize(peak={self.peak!r})"


# ---------------------------------------------------------------------------
# argument checks
# ---------------------------------------------------------------------------


def _kind(kind, allowed=("lowpass", "highpass")) -> str:
    name = _KINDS.get(str(kind).lower())
    if name is None:
        raise InvalidArgument(f"unknown filter kind {kind!r}")
    if name not in allowed:
        raise InvalidArgument(f"kind {name!r} not supported here (allowed: {', '.join(allowed)})")
    return name


def _order(order) -> int:
    if isinstance(order, bool) or not isinstance(order, (int, np.integer)) or order < 1:
        raise InvalidOrder(f"order must be an integer >= 1, got {order!r}")
    return int(order)


def _cutoff(fc, fs) -> float:
    fc = float(fc)
    if fs is None:
        if not fc > 0.0:
            raise InvalidCutoff(f"cutoff must be positive, got {fc}")
    elif not (0.0 < fc < fs / 2.0):
        raise InvalidCutoff(f"cutoff {fc} Hz outside (0, {fs / 2.0}) for fs={fs}")
    return fc


# ---------------------------------------------------------------------------
# IIR: analog prototype -> prewarp -> bilinear -> sections
# ---------------------------------------------------------------------------


def _prototype(family: str, order: int, ripple_db: Optional[float]):
    """Normalised analog low-pass poles (rad/s, cutoff 1) and the gain that
    makes the passband maximum 1 (design.py:209-227)."""
    idx = np.arange(1, order + 1)
    if family == "butterworth":
        poles = np.exp(1j * math.pi * (2 * idx + order - 1) / (2 * order))
        gain = float(np.real(np.prod(-poles)))
    else:
        eps = math.sqrt(10.0 ** (ripple_db / 10.0) - 1.0)
        mu = math.asinh(1.0 / eps) / order
        theta = math.pi * (2 * idx - 1) / (2 * order)
        poles = -math.sinh(mu) * np.sin(theta) + 1j * math.cosh(mu) * np.cos(theta)
        gain = float(np.real(np.prod(-poles)))
        if order % 2 == 0:
            gain /= math.sqrt(1.0 + eps * eps)  # even order: DC sits at -ripple dB
    return poles, gain


def _digital_zpk(family, kind, order, ripple_db, fc, fs):
    poles, gain = _prototype(family, order, ripple_db)
    wa = 2.0 * fs * math.tan(math.pi * fc / fs)  # prewarped analog cutoff
    if kind == "highpass":
        # s -> wa / s: poles invert, `order` zeros appear at s = 0
        gain *= float(np.real(1.0 / np.prod(-poles)))
        poles = wa / poles
        zeros = np.zeros(order, dtype=complex)
    else:
        poles = poles * wa
        gain *= wa**order
        zeros = np.zeros(0, dtype=complex)
    two_fs = 2.0 * fs
    # bilinear map s -> 2 fs (z - 1) / (z + 1); missing zeros land at z = -1
    gain *= float(np.real((np.prod(two_fs - zeros) if zeros.size else 1.0) / np.prod(two_fs - poles)))
    zd = (two_fs + zeros) / (two_fs - zeros)
    pd = (two_fs + poles) / (two_fs - poles)
    zd = np.concatenate([zd, -np.ones(order - zeros.size)])
    return zd, pd, gain


def _pole_groups(poles) -> list:
    """Conjugate pairs (upper-half representative first), then real poles
    paired two at a time in order of |x|; an odd leftover stays single
    (design.py:282-295). Groups are then ordered by (radius, |angle|)."""
    upper = [p for p in poles if abs(p.imag) > _REAL_EPS and p.imag > 0]
    upper.sort(key=lambda p: (abs(p), cmath.phase(p)))
    reals = sorted((p.real for p in poles if abs(p.imag) <= _REAL_EPS), key=lambda x: (abs(x), x))
    groups = [[p, p.conjugate()] for p in upper]
    while len(reals) >= 2:
        groups.append([complex(reals.pop(0)), complex(reals.pop(0))])
    if reals:
        groups.append([complex(reals.pop())])
    groups.sort(key=lambda g: (abs(g[0]), abs(cmath.phase(g[0]))))
    return groups


def _monic(roots) -> np.ndarray:
    """Real coefficients of prod (1 - r z^-1), padded to length 3."""
    if len(roots) == 0:
        out = [1.0, 0.0, 0.0]
    elif len(roots) == 1:
        out = [1.0, -roots[0].real, 0.0]
    else:
        r0, r1 = roots
        if r1 == r0.conjugate() and abs(r0.imag) > _REAL_EPS:
            out = [1.0, -2.0 * r0.real, r0.real * r0.real + r0.imag * r0.imag]
        else:
            s = r0 + r1
            p = r0 * r1
            out = [1.0, -s.real, p.real]
    return np.asarray(out, dtype=np.float64)


def _sections_from_zpk(zd, pd, gain):
    remaining = list(zd)
    sections = []
    for group in _pole_groups(pd):
        anchor = group[0]
        taken = []
        for _ in range(len(group)):
            if remaining:
                best = min(range(len(remaining)), key=lambda i: (abs(remaining[i] - anchor), i))
                taken.append(remaining.pop(best))
        a = _monic(group)
        b = _monic(taken)
        sections.append(BiquadSection(b[0], b[1], b[2], a[1], a[2]))
    return tuple(sections), float(gain)


def _design_recursive(family, kind, order, fc, fs, ripple_db=None):
    zd, pd, gain = _digital_zpk(family, kind, order, ripple_db, fc, fs)
    return _sections_from_zpk(zd, pd, gain)


def design_butterworth(kind, order: int, fc: float, fs: Optional[int] = None) -> IirFilter:
    """Maximally flat low/high-pass; |H(fc)| = 1/sqrt(2) (design.py:333-352)."""
    kind = _kind(kind)
    order = _order(order)
    fc = _cutoff(fc, fs)
    spec = FilterSpec(family="butterworth", kind=kind, order=order, fc=fc)
    if fs is None:
        return IirFilter(sections=(), overall_gain=1.0, spec=spec, fs=None)
    sections, gain = _design_recursive("butterworth", kind, order, fc, fs)
    return IirFilter(sections=sections, overall_gain=gain, spec=spec, fs=int(fs))


def design_chebyshev1(kind, order: int, ripple_db: float, fc: float, fs: Optional[int] = None) -> IirFilter:
    """Equiripple passband, maximum normalised to 1 (design.py:355-375)."""
    kind = _kind(kind)
    order = _order(order)
    if not ripple_db > 0:
        raise InvalidRipple(f"ripple_db must be > 0, got {ripple_db!r}")
    fc = _cutoff(fc, fs)
    spec = FilterSpec(family="chebyshev1", kind=kind, order=order, fc=fc, ripple_db=float(ripple_db))
    if fs is None:
        return IirFilter(sections=(), overall_gain=1.0, spec=spec, fs=None)
    sections, gain = _design_recursive("chebyshev1", kind, order, fc, fs, float(ripple_db))
    return IirFilter(sections=sections, overall_gain=gain, spec=spec, fs=int(fs))


def _cookbook(kind: str, fc: float, gain_db: float, q: float, fs: int) -> BiquadSection:
    """RBJ audio-EQ cookbook biquads, normalised by a0."""
    big_a = 10.0 ** (gain_db / 40.0)
    w0 = 2.0 * math.pi * fc / fs
    cw, sw = math.cos(w0), math.sin(w0)
    alpha = sw / (2.0 * q)
    if kind == "peaking":
        b = (1 + alpha * big_a, -2 * cw, 1 - alpha * big_a)
        a = (1 + alpha / big_a, -2 * cw, 1 - alpha / big_a)
    else:
        k = 2.0 * math.sqrt(big_a) * alpha
        ap, am = big_a + 1, big_a - 1
        if kind == "lo_shelf":
            b = (big_a * (ap - am * cw + k), 2 * big_a * (am - ap * cw), big_a * (ap - am * cw - k))
            a = (ap + am * cw + k, -2 * (am + ap * cw), ap + am * cw - k)
        else:
            b = (big_a * (ap + am * cw + k), -2 * big_a * (am + ap * cw), big_a * (ap + am * cw - k))
            a = (ap - am * cw + k, 2 * (am - ap * cw), ap - am * cw - k)
    return BiquadSection(b[0] / a[0], b[1] / a[0], b[2] / a[0], a[1] / a[0], a[2] / a[0])


def design_shelf(kind, fc: float, gain_db: float, q: float = DEFAULT_Q, fs: Optional[int] = None) -> IirFilter:
    """Single-biquad low/high shelf (design.py:378-419); gain_db is required."""
    if kind not in ("lo_shelf", "hi_shelf", "loshelf", "hishelf"):
        raise InvalidArgument(f"shelf kind must be lo_shelf or hi_shelf, got {kind!r}")
    kind = {"loshelf": "lo_shelf", "hishelf": "hi_shelf"}.get(kind, kind)
    if not q > 0:
        raise InvalidQ(f"q must be > 0, got {q!r}")
    fc = _cutoff(fc, fs)
    spec = FilterSpec(family=kind, fc=fc, gain_db=float(gain_db), q=float(q))
    if fs is None:
        return IirFilter(sections=(), overall_gain=1.0, spec=spec, fs=None)
    if gain_db == 0.0:
        # zero gain: the literal identity section, not a cancelling pole/zero pair
        return IirFilter(sections=(_IDENTITY,), overall_gain=1.0, spec=spec, fs=int(fs))
    section = _cookbook(kind, fc, float(gain_db), float(q), fs)
    return IirFilter(sections=(section,), overall_gain=1.0, spec=spec, fs=int(fs))


def design_peaking(fc: float, gain_db: float, q: float = DEFAULT_Q, fs: Optional[int] = None) -> IirFilter:
    """Peaking EQ: gain_db at fc, unity at DC and Nyquist (design.py:422-443)."""
    if not q > 0:
        raise InvalidQ(f"q must be > 0, got {q!r}")
    fc = _cutoff(fc, fs)
    spec = FilterSpec(family="peaking", fc=fc, gain_db=float(gain_db), q=float(q))
    if fs is None:
        return IirFilter(sections=(), overall_gain=1.0, spec=spec, fs=None)
    if gain_db == 0.0:
        return IirFilter(sections=(_IDENTITY,), overall_gain=1.0, spec=spec, fs=int(fs))
    section = _cookbook("peaking", fc, float(gain_db), float(q), fs)
    return IirFilter(sections=(section,), overall_gain=1.0, spec=spec, fs=int(fs))


# ---------------------------------------------------------------------------
# FIR: windowed ideal sinc
# ---------------------------------------------------------------------------


def _ideal_lowpass(fc: float, fs: float, m: np.ndarray) -> np.ndarray:
    wc = 2.0 * math.pi * fc / fs
    out = np.full(m.shape, wc / math.pi)
    nz = m != 0.0
    out[nz] = np.sin(wc * m[nz]) / (math.pi * m[nz])
    return out


def _window(name: str, n_taps: int) -> np.ndarray:
    phase = 2.0 * math.pi * np.arange(n_taps, dtype=np.float64) / (n_taps - 1)
    if name == "hamming":
        return 0.54 - 0.46 * np.cos(phase)
    if name == "blackman":
        return 0.42 - 0.5 * np.cos(phase) + 0.08 * np.cos(2.0 * phase)
    return np.ones(n_taps)


def design_fir(kind, num_taps: int, fc, window: str = "hamming", fs: Optional[int] = None) -> FirFilter:
    """Windowed-sinc FIR (design.py:446-495).

    Low-pass taps sum to 1; high-pass has |H(Nyquist)| = 1; band-pass has
    |H| = 1 at (f1 + f2) / 2. High/band-pass need an odd tap count.
    """
    kind = _kind(kind, allowed=("lowpass", "highpass", "bandpass"))
    if isinstance(num_taps, bool) or not isinstance(num_taps, (int, np.integer)) or num_taps < 3:
        raise InvalidTapCount(f"num_taps must be an integer >= 3, got {num_taps!r}")
    num_taps = int(num_taps)
    if kind in ("highpass", "bandpass") and num_taps % 2 == 0:
        raise InvalidTapCount(f"{kind} needs an odd tap count, got {num_taps}")
    if window not in _WINDOWS:
        raise InvalidArgument(f"window must be one of {_WINDOWS}, got {window!r}")
    if kind == "bandpass":
        try:
            f1, f2 = (float(v) for v in fc)
        except TypeError:
            raise InvalidCutoff(f"bandpass needs an (f1, f2) pair, got {fc!r}") from None
        if not f1 < f2:
            raise InvalidCutoff(f"bandpass needs f1 < f2, got ({f1}, {f2})")
        spec_fc = (_cutoff(f1, fs), _cutoff(f2, fs))
    else:
        spec_fc = _cutoff(fc, fs)
    spec = FilterSpec(family="fir_sinc", kind=kind, order=num_taps, fc=spec_fc, window=window)
    if fs is None:
        return FirFilter(taps=None, spec=spec, fs=None)

    n = np.arange(num_taps, dtype=np.float64)
    m = n - (num_taps - 1) / 2.0
    win = _window(window, num_taps)
    if kind == "lowpass":
        taps = _ideal_lowpass(spec_fc, fs, m) * win
        taps = taps / np.sum(taps)
    elif kind == "highpass":
        taps = ((m == 0.0).astype(np.float64) - _ideal_lowpass(spec_fc, fs, m)) * win
        taps = taps / abs(float(np.sum(taps * np.cos(math.pi * n))))
    else:
        f1, f2 = spec_fc
        taps = (_ideal_lowpass(f2, fs, m) - _ideal_lowpass(f1, fs, m)) * win
        taps = taps / abs(_fir_response(taps, np.array([(f1 + f2) / 2.0]), fs)[0])
    return FirFilter(taps=taps, spec=spec, fs=int(fs))


# ---------------------------------------------------------------------------
# lazy binding and inspection
# ---------------------------------------------------------------------------


@functools.lru_cache(maxsize=512)
def _design_iir_from_spec(spec: FilterSpec, fs: int) -> IirFilter:
    """Bind-time design, memoised per (spec, fs): a bound filter is immutable
    (frozen sections), so every ``pipe`` of the same unbound chain at the same
    rate reuses one design instead of re-running the zpk/bilinear maths on the
    host (the reference re-designs on every bind, chain.py:56-64)."""
    fam = spec.family
    if fam == "butterworth":
        return design_butterworth(spec.kind, spec.order, spec.fc, fs)
    if fam == "chebyshev1":
        return design_chebyshev1(spec.kind, spec.order, spec.ripple_db, spec.fc, fs)
    if fam in ("lo_shelf", "hi_shelf"):
        return design_shelf(fam, spec.fc, spec.gain_db, spec.q, fs)
    if fam == "peaking":
        return design_peaking(spec.fc, spec.gain_db, spec.q, fs)
    raise InvalidArgument(f"cannot bind IIR spec of family {fam!r}")


@functools.lru_cache(maxsize=512)
def _design_fir_from_spec(spec: FilterSpec, fs: int) -> FirFilter:
    """Memoised like _design_iir_from_spec (taps are a read-only copy)."""
    if spec.family == "fir_sinc":
        return design_fir(spec.kind, spec.order, spec.fc, spec.window, fs)
    raise InvalidArgument(f"cannot bind FIR spec of family {spec.family!r}")


def _fir_response(taps: np.ndarray, freqs: np.ndarray, fs: float) -> np.ndarray:
    phase = -2j * math.pi * np.outer(freqs, np.arange(len(taps))) / fs
    return np.exp(phase) @ taps


def frequency_response(filt, freqs) -> np.ndarray:
    """Complex gain at each probe frequency in [0, fs/2] (design.py:552-570).

    Works for IirFilter, FirFilter, Gain and Normalize (the latter has no
    fixed response and is rejected).
    """
    if getattr(filt, "fs", None) is None:
        raise UnboundFilter("cannot evaluate the response of an unbound filter")
    freqs = np.atleast_1d(np.asarray(freqs, dtype=np.float64))
    nyquist = filt.fs / 2.0
    bad = (freqs < 0) | (freqs > nyquist)
    if np.any(bad):
        raise FrequencyOutOfRange(f"frequencies {freqs[bad].tolist()} outside [0, {nyquist}]")
    if isinstance(filt, FirFilter):
        return _fir_response(filt.taps, freqs, float(filt.fs))
    if isinstance(filt, Gain):
        return np.full(freqs.shape, filt.factor, dtype=complex)
    if isinstance(filt, Normalize):
        raise InvalidArgument("Normalize depends on the signal; it has no frequency response")
    zi = np.exp(-2j * math.pi * freqs / filt.fs)
    out = np.full(freqs.shape, filt.overall_gain, dtype=complex)
    for s in filt.sections:
        out = out * (s.b0 + s.b1 * zi + s.b2 * zi * zi) / (1.0 + s.a1 * zi + s.a2 * zi * zi)
    return out
