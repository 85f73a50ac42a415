"""Drop-in kernel module for the reference's kernel seam.

The reference picks its kernel module in one place,
``pkg/src/wavepipe/engine.py:74-75``::

    def _kernels():
        return _kernels_jit if _jit_enabled else _kernels_py

This module has the same functions as ``_kernels_jit`` / ``_kernels_py``
(``_kernels_jit.py:35-100``, ``_kernels_py.py:13-63``) -- float64 numpy in,
new float64 numpy array out -- backed by the C ABI: calls up to 2 GiB of float32 run through
``wp_plan_execute_host`` from page-locked staging (uploads, passes and
downloads of channel blocks overlapped), larger ones through the one-shot
entry points (``wp_iir_cascade`` / ``wp_fir``, include/wavepipe_b200.h) with
the device workspace sized per call by ``wp_*_workspace``. INTEGRATION.md shows
the two-line change that makes ``engine._kernels()`` return it. It is the
seam for code that keeps the reference's per-stage engine; the lazy ``Wave``
/ ``Chain`` of this package fuses whole chains instead.

Numerics: the input is rounded to float32 and the kernels compute in
float32 (tensor-core split products, fp32 scan in a balanced state basis);
outputs match the float64 kernels within 1e-5 (FIR) / 1e-4 (IIR) of the
output peak, not bit for bit.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .errors import InvalidArgument

__all__ = [
    "iir_cascade_serial",
    "iir_cascade_parallel",
    "fir_direct_serial",
    "fir_direct_parallel",
    "fir_fft",
    "oracle_transversal",
]

_dp = ctypes.POINTER(ctypes.c_double)
_PIN_MAX_BYTES = 2 << 30  # larger calls copy through pageable memory (no page-locking of huge buffers)


def _planar(x) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 2:
        raise InvalidArgument(f"kernels take planar [channels, frames] arrays, got shape {x.shape}")
    return x


def _run(kind: str, coef: np.ndarray, n: int, x: np.ndarray, flags: int) -> np.ndarray:
    import torch

    lib = _native.load(require_device=True)
    x = _planar(x)
    C, N = x.shape
    if C == 0 or N == 0:
        return np.empty_like(x)
    c = np.ascontiguousarray(coef, dtype=np.float64)
    cp = c.ctypes.data_as(_dp)
    need = ctypes.c_size_t()
    query = lib.wp_iir_cascade_workspace if kind == "iir" else lib.wp_fir_workspace
    _native.check(query(cp, n, C, N, flags, ctypes.byref(need)), f"{kind} workspace")
    if C * N * 4 <= _PIN_MAX_BYTES:
        # page-locked staging (the caching host allocator reuses it): the
        # float64 -> float32 rounding writes straight into it, and
        # wp_plan_execute_host overlaps uploads, passes and downloads of
        # channel blocks (same plan and kernels as the one-shot entry below)
        from . import engine

        kind_id = _native.WP_STAGE_IIR if kind == "iir" else _native.WP_STAGE_FIR
        c_ro = c.copy()
        c_ro.setflags(write=False)
        hx = torch.empty((C, N), dtype=torch.float32, pin_memory=True)
        np.copyto(hx.numpy(), x, casting="same_kind")
        hy = torch.empty((C, N), dtype=torch.float32, pin_memory=True)
        engine.stream_host_entries(((kind_id, c_ro, 0.0, int(flags)),), hx, hy)
        return hy.numpy().astype(np.float64)
    x32 = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
    y32 = torch.empty_like(x32)
    ws = torch.empty(max(int(need.value), 1), dtype=torch.uint8, device=x32.device)
    fn = lib.wp_iir_cascade if kind == "iir" else lib.wp_fir
    stream = torch.cuda.current_stream(x32.device).cuda_stream
    _native.check(fn(cp, n, x32.data_ptr(), y32.data_ptr(), C, N, N, N, flags, ws.data_ptr(), ws.numel(), stream),
                  kind)
    return y32.cpu().numpy().astype(np.float64)


def iir_cascade_serial(sos, x) -> np.ndarray:
    """_kernels_jit.py:35-40: DF2T cascade of ``sos[S, 5]`` (gain folded into
    section 0) over every channel of ``x[C, N]``."""
    sos = np.asarray(sos, dtype=np.float64).reshape(-1, 5)
    return _run("iir", sos, sos.shape[0], x, _native.WP_IIR_PREC_AUTO)


iir_cascade_parallel = iir_cascade_serial  # _kernels_jit.py:43-48 (channels run in parallel on the GPU anyway)


def fir_direct_serial(taps, x) -> np.ndarray:
    """_kernels_jit.py:65-70: causal same-length convolution."""
    taps = np.asarray(taps, dtype=np.float64).reshape(-1)
    return _run("fir", taps, taps.size, x, _native.WP_FIR_DIRECT)


fir_direct_parallel = fir_direct_serial  # _kernels_jit.py:73-78


def fir_fft(taps, x) -> np.ndarray:
    """engine._fir_fft (engine.py:206-223): the long-FIR path (FFT
    overlap-save on the GPU instead of overlap-add on the host)."""
    taps = np.asarray(taps, dtype=np.float64).reshape(-1)
    return _run("fir", taps, taps.size, x, _native.WP_FIR_FFT)


def oracle_transversal(b, a, x) -> np.ndarray:
    """_kernels_jit.py:81-100: the literal difference equation, the reference's
    own ground-truth checker. Kept as the same host loop (engine.iir_oracle);
    it is not a filtering path."""
    from .engine import iir_oracle

    return iir_oracle(b, a, x)
