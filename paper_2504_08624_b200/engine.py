"""Filter application on the B200: stage lists -> fused plans -> C-ABI launches.

Public surface of the reference's ``wavepipe.engine`` (pkg/src/wavepipe/engine.py)
kept as a drop-in: ``apply_iir`` (:142-156), ``apply_fir`` (:159-178),
``iir_oracle`` (:181-198), ``BACKENDS``/``CONV_STRATEGIES`` (:38-39), the
backend/strategy resolvers (:106-123) and the thread/JIT knobs (:58-103).

What changes underneath:

* ``backend`` is validated exactly like the reference (unknown names raise
  InvalidArgument) but every backend runs the same GPU path; results do not
  depend on it (the reference guarantees the same across its backends).
* Application is lazy: stages are converted to plan entries
  ``(kind, coefficients, value, flags)`` and recorded on the output Wave; the
  whole recorded list becomes one ``wp_plan`` (cached per device) whose fused
  passes run when the samples are first needed.
* There is no CPU fallback. ``set_jit_enabled(False)`` is refused.
"""

from __future__ import annotations

import os
import threading
from collections import OrderedDict

import numpy as np

from . import _native
from .design import FirFilter, Gain, IirFilter, Normalize
from .errors import (
    InvalidArgument,
    InvalidCoefficients,
    NativeUnavailable,
    SampleRateMismatch,
    UnboundFilter,
)
from .wave import Wave

__all__ = [
    "BACKENDS",
    "CONV_STRATEGIES",
    "apply_iir",
    "apply_fir",
    "apply_stage",
    "iir_oracle",
    "jit_available",
    "jit_enabled",
    "set_jit_enabled",
    "get_num_threads",
    "set_num_threads",
    "max_threads",
    "set_iir_precision",
    "get_iir_precision",
    "run_chain",
    "execute_entries",
    "plan_for",
]

BACKENDS = ("serial", "parallel", "auto")
CONV_STRATEGIES = ("direct", "fft", "auto")
PRECISIONS = ("auto", "f32", "f64")

# reference heuristics, kept for API compatibility (engine.py:41-45)
_PARALLEL_MIN_SAMPLES = 32768
_FFT_MIN_TAPS = 128
_FFT_MIN_FRAMES = 4096

_precision = "auto"


# ---------------------------------------------------------------------------
# compatibility knobs
# ---------------------------------------------------------------------------


def jit_available() -> bool:
    """True when the compiled sm_100a library is present (the analogue of the
    reference's numba availability)."""
    return os.path.exists(_native.lib_path())


def jit_enabled() -> bool:
    return True


def set_jit_enabled(flag: bool) -> None:
    if not flag:
        raise InvalidArgument("the B200 engine has no CPU fallback; compiled kernels cannot be disabled")
    if not jit_available():
        raise NativeUnavailable("libwpb200.so is not built")


def max_threads() -> int:
    return os.cpu_count() or 1


_num_threads = max_threads()


def get_num_threads() -> int:
    return _num_threads


def set_num_threads(n: int) -> int:
    """Host worker count (compatibility shim: GPU execution ignores it)."""
    global _num_threads
    if isinstance(n, bool) or not isinstance(n, int) or n < 1:
        raise InvalidArgument(f"thread count must be a positive integer, got {n!r}")
    _num_threads = min(n, max_threads())
    return _num_threads


def set_iir_precision(mode: str) -> None:
    """IIR scan precision: "auto" (fp64 for blocks with a pole radius > 0.98),
    "f32" or "f64" (forced; for experiments and tests)."""
    global _precision
    if mode not in PRECISIONS:
        raise InvalidArgument(f"precision must be one of {PRECISIONS}, got {mode!r}")
    _precision = mode


def get_iir_precision() -> str:
    return _precision


def _resolve_backend(backend: str, channels: int, frames: int) -> str:
    if backend not in BACKENDS:
        raise InvalidArgument(f"backend must be one of {BACKENDS}, got {backend!r}")
    if backend != "auto":
        return backend
    if channels >= 2 and channels * frames >= _PARALLEL_MIN_SAMPLES:
        return "parallel"
    return "serial"


def _resolve_strategy(strategy: str, taps: int, frames: int) -> str:
    if strategy not in CONV_STRATEGIES:
        raise InvalidArgument(f"conv strategy must be one of {CONV_STRATEGIES}, got {strategy!r}")
    if strategy != "auto":
        return strategy
    if taps > _FFT_MIN_TAPS and frames > _FFT_MIN_FRAMES:
        return "fft"
    return "direct"


def _check_bound(filt, wave: Wave) -> None:
    if filt.fs is None:
        raise UnboundFilter("filter must be bound to a sampling rate before application")
    if filt.fs != wave.fs:
        raise SampleRateMismatch(f"filter designed for {filt.fs} Hz applied to a {wave.fs} Hz wave")


# ---------------------------------------------------------------------------
# stages -> plan entries
# ---------------------------------------------------------------------------

_PREC_FLAG = {"auto": _native.WP_IIR_PREC_AUTO, "f32": _native.WP_IIR_PREC_F32, "f64": _native.WP_IIR_PREC_F64}
_FIR_FLAG = {"auto": _native.WP_FIR_AUTO, "direct": _native.WP_FIR_DIRECT, "fft": _native.WP_FIR_FFT}


def _is_builtin(stage) -> bool:
    return isinstance(stage, (IirFilter, FirFilter, Gain, Normalize))


def _entry(stage, strategy: str = "auto"):
    if isinstance(stage, IirFilter):
        rows = stage.sos_rows()  # gain folded into section 0 (engine.py:133-139)
        rows.setflags(write=False)
        return (_native.WP_STAGE_IIR, rows, 0.0, _PREC_FLAG[_precision])
    if isinstance(stage, FirFilter):
        return (_native.WP_STAGE_FIR, stage.taps, 0.0, _FIR_FLAG[strategy])
    if isinstance(stage, Gain):
        return (_native.WP_STAGE_GAIN, None, stage.factor, 0)
    if isinstance(stage, Normalize):
        return (_native.WP_STAGE_NORMALIZE, None, stage.peak, 0)
    raise InvalidArgument(f"not a built-in stage: {stage!r}")


def _key(entries) -> tuple:
    return tuple(
        (k, None if c is None else (c.shape, c.tobytes()), float(v), int(f)) for (k, c, v, f) in entries
    )


class _PlanCache:
    def __init__(self, capacity: int = 256):
        self._plans = OrderedDict()
        self._cap = capacity
        self._lock = threading.Lock()

    def get(self, device: int, entries) -> _native.Plan:
        key = (device, _key(entries))
        with self._lock:
            plan = self._plans.get(key)
            if plan is not None:
                self._plans.move_to_end(key)
                return plan
        plan = _native.Plan(entries)
        with self._lock:
            self._plans[key] = plan
            while len(self._plans) > self._cap:
                self._plans.popitem(last=False)
        return plan


_plans = _PlanCache()
_workspaces = {}
_ws_lock = threading.Lock()


def plan_for(stages, device: int = None, strategy: str = "auto") -> _native.Plan:
    """The fused plan for a bound stage list (exposed for bench/diagnostics)."""
    import torch

    entries = tuple(_entry(s, strategy) for s in stages)
    dev = torch.cuda.current_device() if device is None else int(device)
    with torch.cuda.device(dev):
        return _plans.get(dev, entries)


def _workspace(device, stream_ptr: int, nbytes: int):
    import torch

    key = (device.index, stream_ptr)
    with _ws_lock:
        buf = _workspaces.get(key)
        if buf is None or buf.numel() < nbytes:
            size = max(nbytes, 1 << 20)
            if buf is not None:
                size = max(size, int(buf.numel() * 1.5))
            buf = torch.empty(size, dtype=torch.uint8, device=device)
            _workspaces[key] = buf
    return buf


def execute_entries(entries, src, out=None):
    """Run a recorded entry list on ``src`` (float32 CUDA ``[C, N]``)."""
    import torch

    if not src.is_cuda:
        raise NativeUnavailable("execute_entries needs a CUDA tensor")
    src = src.contiguous()
    C, N = src.shape
    if out is None:
        out = torch.empty_like(src)
    dev = src.device
    with torch.cuda.device(dev):
        plan = _plans.get(dev.index, entries)
        stream = torch.cuda.current_stream(dev).cuda_stream
        nbytes = plan.workspace_bytes(C, N)
        ws = _workspace(dev, stream, nbytes)
        plan.execute(src.data_ptr(), out.data_ptr(), C, N, src.stride(0), out.stride(0), ws.data_ptr(), ws.numel(), stream)
    return out


def has_normalize(entries) -> bool:
    """A Normalize stage needs the peak of the WHOLE wave (design.Normalize), so
    such a chain cannot run block by block."""
    return any(k == _native.WP_STAGE_NORMALIZE for (k, _c, _v, _f) in entries)


def normalize_scale(peak: float, target: float):
    """The factor scale_by_peak applies (fp32 target / fp32 peak), None for an
    all-zero input (returned unchanged)."""
    p = np.float32(peak)
    if not p > 0:
        return None
    return float(np.float32(target) / p)


def stream_host_entries(entries, host_src, host_out, device=None, blocks: int = 0, sync: bool = True):
    """Host -> device -> host execution of a recorded chain, overlapped.

    ``host_src`` and ``host_out`` are pinned float32 CPU tensors ``[C, N]``.
    Channels are cut into blocks (single channels, or pairs when a pass runs
    the FFT path, which filters pairs together; results are bit-identical to
    one launch over all channels); block b's upload, the fused pass over block
    b-1 and block b-2's download run concurrently on three streams, so the
    PCIe link carries both directions at once instead of one after the other.
    ``sync=False`` returns once the work is enqueued (the device's current
    stream waits for the last download; the device buffers go back to the
    caching allocator on that stream, so reuse is ordered after it).
    """
    import torch

    from ._native import _require_cuda

    _require_cuda()
    if has_normalize(entries):
        raise InvalidArgument("a chain with Normalize needs the whole wave's peak: it cannot be streamed in blocks")
    C, N = host_src.shape
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    with torch.cuda.device(dev):
        plan = _plans.get(dev.index, entries)
        # the block loop (partition, three streams, events) runs in the native
        # library: wp_plan_execute_host cuts single-channel blocks (pairs when
        # a pass runs the FFT path), 16 (32 from 4 GiB), and overlaps block b's upload,
        # block b-1's pass and block b-2's download
        x = torch.empty((C, N), dtype=torch.float32, device=dev)
        y = torch.empty_like(x)
        cur = torch.cuda.current_stream(dev)
        ws = _workspace(dev, cur.cuda_stream, plan.workspace_bytes(C, N))
        plan.execute_host(host_src.data_ptr(), host_out.data_ptr(), C, N, host_src.stride(0), host_out.stride(0),
                          x.data_ptr(), y.data_ptr(), ws.data_ptr(), ws.numel(), int(blocks), cur.cuda_stream)
        if sync:
            cur.synchronize()
    return host_out


def run_chain(wave: Wave, stages, backend: str = "auto", strategy: str = "auto") -> Wave:
    """Record bound ``stages`` on ``wave``; custom stages run eagerly."""
    if not isinstance(wave, Wave):
        raise InvalidArgument(f"expected a Wave, got {type(wave).__name__}")
    _resolve_backend(backend, wave.channels, wave.frames)
    current = wave
    pending = []
    for stage in stages:
        if _is_builtin(stage):
            _check_bound(stage, current)
            pending.append(_entry(stage, strategy))
            continue
        current = _record(current, pending)
        pending = []
        current = stage.apply(current, backend=backend)
        if not isinstance(current, Wave):
            raise InvalidArgument(f"stage {stage!r} returned {type(current).__name__}, not a Wave")
    return _record(current, pending)


def _record(wave: Wave, entries) -> Wave:
    if not entries:
        return wave
    if wave.is_lazy:
        return Wave._lazy(wave._src, wave._entries + tuple(entries))
    return Wave._lazy(wave, tuple(entries))


def apply_iir(filt: IirFilter, wave: Wave, backend: str = "auto") -> Wave:
    """Biquad cascade (DF2T, zero initial state) over every channel."""
    _check_bound(filt, wave)
    _resolve_backend(backend, wave.channels, wave.frames)
    return _record(wave, [_entry(filt)])


def apply_fir(filt: FirFilter, wave: Wave, backend: str = "auto", strategy: str = "auto") -> Wave:
    """Same-length causal convolution of every channel with the taps."""
    _check_bound(filt, wave)
    if strategy not in CONV_STRATEGIES:
        raise InvalidArgument(f"conv strategy must be one of {CONV_STRATEGIES}, got {strategy!r}")
    _resolve_backend(backend, wave.channels, wave.frames)
    return _record(wave, [_entry(filt, strategy)])


def apply_stage(stage, wave: Wave, backend: str = "auto") -> Wave:
    """Gain / Normalize application (bound or rate-agnostic)."""
    if getattr(stage, "fs", None) is not None and stage.fs != wave.fs:
        raise SampleRateMismatch(f"stage bound to {stage.fs} Hz applied to a {wave.fs} Hz wave")
    _resolve_backend(backend, wave.channels, wave.frames)
    return _record(wave, [_entry(stage)])


def iir_oracle(b, a, x) -> np.ndarray:
    """Literal difference equation (engine.py:181-198), kept for API parity.

    The reference uses it as ground truth for tests; it is not on the
    filtering path. It runs the same literal recursion here, in float64, as
    a single-channel transversal filter on the host: it is the reference's
    own checker function, not a fallback for ``apply_*``.
    """
    b = np.atleast_1d(np.asarray(b, dtype=np.float64))
    a = np.atleast_1d(np.asarray(a, dtype=np.float64))
    if b.size == 0 or a.size == 0:
        raise InvalidCoefficients("b and a must be nonempty")
    if a[0] != 1.0:
        raise InvalidCoefficients(f"a[0] must be exactly 1, got {a[0]}")
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 1:
        raise InvalidArgument(f"oracle input must be a 1-D sample vector, got shape {x.shape}")
    y = np.zeros_like(x)
    for i in range(x.size):
        acc = 0.0
        for k in range(min(b.size, i + 1)):
            acc += b[k] * x[i - k]
        for k in range(1, min(a.size, i + 1)):
            acc -= a[k] * y[i - k]
        y[i] = acc
    return y
