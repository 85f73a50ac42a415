"""CPU ORACLE - TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` leg may import this package, and only as the checker or
the timed CPU baseline. The product (``paper_2504_08624_b200``) never imports
it and has no CPU fallback.

Contents (each restates the reference path, citations into /root/reference):

* ``iir_cascade`` / ``fir_direct`` / ``transversal``: ctypes bindings to the C
  restatement in wp_oracle.c (bit-identical to the reference's numba kernels,
  _kernels_jit.py:14-100; pinned by tests/test_oracle.py).
* ``fir_fft``: numpy restatement of the overlap-add path ``engine._fir_fft`` +
  ``_ola_channel`` (engine.py:206-233); the FFT itself is numpy's pocketfft,
  the same third-party code the reference calls (numpy 2.3.5 here; the
  reference pins only ``numpy>=1.24``, pyproject.toml:11).
* ``white_noise``: restatement of the splitmix64 + Box-Muller generator
  (wave.py:103-168), pinned by the reference's frozen head (test_wave.py:8-16).
* ``apply_stage`` / ``pipe``: the reference's per-stage, left-to-right chain
  semantics (chain.py:66-71) incl. auto strategy rules (engine.py:106-123).
* ``save_wav_float32`` / ``load_wav``: the float32 WAV path of wavio.py:49-114,
  only to reproduce the reference's end-to-end golden sha256
  (tests/golden/golden_hashes.json, test_acceptance.py:203-245).
* ``wav_encode`` / ``wav_decode`` / ``wav_file_bytes``: pcm16/pcm24/float32
  payload restatement of wavio.py:69-98 and :193-200 (checker of the device
  WAV codec; pinned by tests/golden/wav_golden.json from the reference).
"""

from __future__ import annotations

import ctypes
import math
import os
import struct
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libwporacle.so")
_SRC = os.path.join(_HERE, "wp_oracle.c")
_lib = None

# reference thresholds (engine.py:41-45)
FFT_MIN_TAPS = 128
FFT_MIN_FRAMES = 4096


def build(force: bool = False) -> str:
    """Compile wp_oracle.c with gcc (no FMA contraction, like numba fastmath=off)."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(_SRC):
        cmd = [
            "gcc", "-O2", "-fPIC", "-shared", "-pthread", "-ffp-contract=off",
            "-fno-fast-math", "-o", LIB_PATH, _SRC,
        ]
        subprocess.run(cmd, check=True)
    return LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        lib.wpo_iir_cascade.argtypes = [dp, i64, dp, dp, i64, i64, ctypes.c_int]
        lib.wpo_fir_direct.argtypes = [dp, i64, dp, dp, i64, i64, ctypes.c_int]
        lib.wpo_transversal.argtypes = [dp, i64, dp, i64, dp, dp, i64]
        for f in (lib.wpo_iir_cascade, lib.wpo_fir_direct, lib.wpo_transversal):
            f.restype = None
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _planar(x) -> np.ndarray:
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if x.ndim == 1:
        x = x.reshape(1, -1)
    return x


def default_threads() -> int:
    return os.cpu_count() or 1


def iir_cascade(sos, x, threads: int = 1) -> np.ndarray:
    """DF2T cascade, sos [S,5] with the gain already folded into row 0."""
    sos = np.ascontiguousarray(np.asarray(sos, dtype=np.float64).reshape(-1, 5))
    x = _planar(x)
    y = np.empty_like(x)
    _load().wpo_iir_cascade(_ptr(sos), sos.shape[0], _ptr(x), _ptr(y), x.shape[0], x.shape[1], int(threads))
    return y


def fir_direct(taps, x, threads: int = 1) -> np.ndarray:
    taps = np.ascontiguousarray(np.asarray(taps, dtype=np.float64).reshape(-1))
    x = _planar(x)
    y = np.empty_like(x)
    _load().wpo_fir_direct(_ptr(taps), taps.shape[0], _ptr(x), _ptr(y), x.shape[0], x.shape[1], int(threads))
    return y


def transversal(b, a, x) -> np.ndarray:
    b = np.ascontiguousarray(np.atleast_1d(np.asarray(b, dtype=np.float64)))
    a = np.ascontiguousarray(np.atleast_1d(np.asarray(a, dtype=np.float64)))
    if a[0] != 1.0:
        raise ValueError("a[0] must be exactly 1")
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    y = np.empty_like(x)
    _load().wpo_transversal(_ptr(b), b.size, _ptr(a), a.size, _ptr(x), _ptr(y), x.size)
    return y


def section_chained(sections, overall_gain, x) -> np.ndarray:
    """conftest.oracle_cascade: one transversal call per section, then the gain
    (pkg/tests/conftest.py:67-72)."""
    y = np.asarray(x, dtype=np.float64)
    for s in sections:
        y = transversal([s.b0, s.b1, s.b2], [1.0, s.a1, s.a2], y)
    return y * overall_gain


def fir_fft(taps, x, threads: int = 1) -> np.ndarray:
    """Overlap-add: nfft = 2^max(3, ceil(log2(8T))), block = nfft - T + 1
    (engine.py:206-233)."""
    taps = np.asarray(taps, dtype=np.float64).reshape(-1)
    x = _planar(x)
    n_taps = taps.size
    frames = x.shape[1]
    nfft = 1 << max(3, math.ceil(math.log2(8 * n_taps)))
    block = nfft - (n_taps - 1)
    taps_f = np.fft.rfft(taps, nfft)
    out = np.empty_like(x)

    def one(c):
        acc = np.zeros(frames + n_taps - 1, dtype=np.float64)
        row = x[c]
        for start in range(0, frames, block):
            seg = row[start : start + block]
            conv = np.fft.irfft(np.fft.rfft(seg, nfft) * taps_f, nfft)
            stop = min(start + nfft, acc.shape[0])
            acc[start:stop] += conv[: stop - start]
        out[c] = acc[:frames]

    if threads > 1 and x.shape[0] > 1:
        with ThreadPoolExecutor(max_workers=min(threads, x.shape[0])) as pool:
            list(pool.map(one, range(x.shape[0])))
    else:
        for c in range(x.shape[0]):
            one(c)
    return out


def fir_auto(taps, x, threads: int = 1) -> np.ndarray:
    """``apply_fir`` with strategy "auto" (engine.py:116-123)."""
    taps = np.asarray(taps, dtype=np.float64).reshape(-1)
    x = _planar(x)
    if taps.size > FFT_MIN_TAPS and x.shape[1] > FFT_MIN_FRAMES:
        return fir_fft(taps, x, threads)
    return fir_direct(taps, x, threads)


# --- noise (wave.py:103-168) -------------------------------------------------

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(seed: int, first: int, count: int) -> np.ndarray:
    ctr = np.arange(first + 1, first + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + ctr * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def standard_normal(count: int, seed: int, first_pair: int = 0) -> np.ndarray:
    """Flat N(0,1) stream; pair j uses counters (2j, 2j+1)."""
    pairs = (count + 1) // 2
    bits = _mix(seed, 2 * first_pair, 2 * pairs)
    u1 = ((bits[0::2] >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0**-53
    u2 = (bits[1::2] >> np.uint64(11)).astype(np.float64) * 2.0**-53
    radius = np.sqrt(-2.0 * np.log(u1))
    angle = 2.0 * np.pi * u2
    out = np.empty(2 * pairs, dtype=np.float64)
    out[0::2] = radius * np.cos(angle)
    out[1::2] = radius * np.sin(angle)
    return out[:count]


def white_noise(duration_s: float, channels: int, fs: int, seed: int) -> np.ndarray:
    frames = int(round(float(duration_s) * fs))
    return standard_normal(channels * frames, seed).reshape(channels, frames)


def sine_bank(channels: int, frames: int, fs: int, amplitude: float = 0.5) -> np.ndarray:
    """Pinned sine workload of SURVEY.md §8(d): 0.5 sin(2 pi f_c n / fs),
    f_c = 440 * 2^(c / C)."""
    n = np.arange(frames, dtype=np.float64)
    f = 440.0 * 2.0 ** (np.arange(channels, dtype=np.float64) / channels)
    return amplitude * np.sin(2.0 * np.pi * f[:, None] * n[None, :] / fs)


# --- chain semantics (chain.py:66-71) ---------------------------------------


def apply_stage(stage, x: np.ndarray, threads: int = 1, strategy: str = "auto") -> np.ndarray:
    """One reference stage over planar float64 ``x``. Stages are duck-typed:
    ``sections``/``overall_gain`` (IIR), ``taps`` (FIR), ``factor`` (Gain),
    ``peak`` (Normalize, semantics defined by this build)."""
    if hasattr(stage, "sections"):
        rows = np.array([[s.b0, s.b1, s.b2, s.a1, s.a2] for s in stage.sections], dtype=np.float64)
        rows[0, :3] *= stage.overall_gain  # engine.py:138
        return iir_cascade(rows, x, threads)
    if hasattr(stage, "taps"):
        if strategy == "fft":
            return fir_fft(stage.taps, x, threads)
        if strategy == "direct":
            return fir_direct(stage.taps, x, threads)
        return fir_auto(stage.taps, x, threads)
    if hasattr(stage, "factor"):
        return x * stage.factor
    if hasattr(stage, "peak"):
        m = float(np.max(np.abs(x)))
        return x if m == 0.0 else x * (stage.peak / m)
    raise TypeError(f"oracle does not know stage {stage!r}")


def pipe(x, stages, threads: int = 1) -> np.ndarray:
    y = _planar(x)
    for st in stages:
        y = apply_stage(st, y, threads)
    return y


# --- float32 WAV (wavio.py:49-114) --------------------------------------------


def save_wav_float32(samples: np.ndarray, fs: int, path: str) -> None:
    samples = _planar(samples)
    payload = np.ascontiguousarray(samples.T).astype(np.float32).tobytes()
    channels = samples.shape[0]
    block = channels * 4
    fmt = struct.pack("<4sIHHIIHH", b"fmt ", 16, 3, channels, fs, fs * block, block, 32)
    pad = b"\x00" if len(payload) % 2 else b""
    data = struct.pack("<4sI", b"data", len(payload)) + payload + pad
    with open(path, "wb") as fh:
        fh.write(struct.pack("<4sI4s", b"RIFF", 4 + len(fmt) + len(data), b"WAVE"))
        fh.write(fmt)
        fh.write(data)


def load_wav_float32(path: str):
    with open(path, "rb") as fh:
        raw = fh.read()
    assert raw[:4] == b"RIFF" and raw[8:12] == b"WAVE"
    off, fs, channels, data = 12, None, None, None
    while off + 8 <= len(raw):
        cid, size = struct.unpack_from("<4sI", raw, off)
        body = raw[off + 8 : off + 8 + size]
        if cid == b"fmt ":
            tag, channels, fs, _, _, bits = struct.unpack_from("<HHIIHH", body, 0)
            assert tag == 3 and bits == 32
        elif cid == b"data":
            data = body
        off += 8 + size + (size & 1)
    inter = np.frombuffer(data, dtype="<f4").astype(np.float64)
    return np.ascontiguousarray(inter.reshape(-1, channels).T), fs


# --- WAV payloads (wavio.py:69-98 encode, :193-200 decode) ------------------

_WAV_BITS = {"pcm16": 16, "pcm24": 24, "float32": 32}


def wav_encode(samples, encoding: str):
    """Interleaved little-endian payload bytes and the clipped-sample count
    of planar ``samples`` (save_wav, wavio.py:69-98)."""
    inter = np.ascontiguousarray(_planar(samples).T)
    if encoding == "float32":
        return inter.astype(np.float32).tobytes(), 0
    bits = _WAV_BITS[encoding]
    clipped = int(np.count_nonzero(np.abs(inter) > 1.0))
    full = float(2 ** (bits - 1))
    c = np.clip(inter, -1.0, 1.0)
    q = np.clip(np.copysign(np.floor(np.abs(c) * full + 0.5), c), -full, full - 1).astype(np.int32)
    if bits == 16:
        return q.astype("<i2").tobytes(), clipped
    b4 = np.frombuffer(q.astype("<i4").tobytes(), dtype=np.uint8).reshape(-1, 4)
    return np.ascontiguousarray(b4[:, :3]).tobytes(), clipped


def wav_decode(payload: bytes, encoding: str, channels: int) -> np.ndarray:
    """Planar float64 samples of an interleaved payload (wavio.py:193-200)."""
    if encoding == "pcm16":
        v = np.frombuffer(payload, dtype="<i2").astype(np.float64) / 2.0**15
    elif encoding == "pcm24":
        t = np.frombuffer(payload, dtype=np.uint8).reshape(-1, 3).astype(np.int32)
        v = (((t[:, 0] << 8) | (t[:, 1] << 16) | (t[:, 2] << 24)) >> 8).astype(np.float64) / 2.0**23
    else:
        v = np.frombuffer(payload, dtype="<f4").astype(np.float64)
    return np.ascontiguousarray(v.reshape(-1, channels).T)


def wav_file_bytes(samples, fs: int, encoding: str):
    """Canonical RIFF/WAVE file bytes (fmt + data chunk) and clipped count."""
    samples = _planar(samples)
    payload, clipped = wav_encode(samples, encoding)
    bits = _WAV_BITS[encoding]
    tag = 3 if encoding == "float32" else 1
    channels = samples.shape[0]
    block = channels * bits // 8
    fmt = struct.pack("<4sIHHIIHH", b"fmt ", 16, tag, channels, fs, fs * block, block, bits)
    pad = b"\x00" if len(payload) % 2 else b""
    data = struct.pack("<4sI", b"data", len(payload)) + payload + pad
    return struct.pack("<4sI4s", b"RIFF", 4 + len(fmt) + len(data), b"WAVE") + fmt + data, clipped


def parity_error(y, y_ref) -> float:
    """SURVEY.md §8(c) metric: max |y - y_ref| / max |y_ref|."""
    y = np.asarray(y, dtype=np.float64)
    y_ref = np.asarray(y_ref, dtype=np.float64)
    peak = float(np.max(np.abs(y_ref))) if y_ref.size else 0.0
    err = float(np.max(np.abs(y - y_ref))) if y_ref.size else 0.0
    return err / peak if peak > 0 else err
