"""ctypes binding of libwpb200.so (C ABI in include/wavepipe_b200.h).

This is the only place the package touches native code. There is no CPU
fallback: if the library or a CUDA device is missing, ``NativeUnavailable`` is
raised (the driver's GPU tier checks that this .so is what actually runs).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import KernelError, NativeUnavailable

HERE = os.path.dirname(os.path.abspath(__file__))
# WP_LIB: load another build of the same library (A/B diagnostics: tools/lb_variants.py)
LIB_PATH = os.environ.get("WP_LIB") or os.path.join(HERE, "libwpb200.so")

WP_STAGE_IIR = 1
WP_STAGE_FIR = 2
WP_STAGE_GAIN = 3
WP_STAGE_NORMALIZE = 4

WP_FIR_AUTO = 0
WP_FIR_DIRECT = 1
WP_FIR_FFT = 2
WP_IIR_PREC_AUTO = 0
WP_IIR_PREC_F32 = 16
WP_IIR_PREC_F64 = 32

# every symbol include/wavepipe_b200.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "wp_plan_create",
    "wp_set_trace",
    "wp_wav_decode",
    "wp_wav_encode",
    "wp_plan_destroy",
    "wp_plan_workspace_bytes",
    "wp_plan_execute",
    "wp_plan_execute_host",
    "wp_plan_num_passes",
    "wp_plan_launches",
    "wp_plan_describe",
    "wp_plan_launches_for",
    "wp_plan_describe_for",
    "wp_iir_cascade",
    "wp_fir",
    "wp_iir_cascade_workspace",
    "wp_fir_workspace",
    "wp_white_noise",
    "wp_peak_abs",
    "wp_last_error",
    "wp_abi_version",
    "wp_check_device",
    "wp_launch_count",
)


class Stage(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("n", ctypes.c_int32),
        ("coef", ctypes.POINTER(ctypes.c_double)),
        ("value", ctypes.c_double),
        ("flags", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


_lib = None
_lock = threading.Lock()


def lib_path() -> str:
    return LIB_PATH


def load(require_device: bool = False):
    """Load libwpb200.so (once) and declare prototypes."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeUnavailable(
                    f"{LIB_PATH} is missing; run __graft_entry__.build() (nvcc, sm_100a). "
                    "There is no CPU fallback."
                )
            lib = ctypes.CDLL(LIB_PATH)
            i32, i64, sz, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t, ctypes.c_void_p
            dp = ctypes.POINTER(ctypes.c_double)
            pp = ctypes.POINTER(ctypes.c_void_p)
            lib.wp_plan_create.argtypes = [ctypes.POINTER(Stage), i32, pp]
            lib.wp_plan_destroy.argtypes = [vp]
            lib.wp_plan_workspace_bytes.argtypes = [vp, i64, i64, ctypes.POINTER(sz)]
            lib.wp_plan_execute.argtypes = [vp, vp, vp, i64, i64, i64, i64, vp, sz, vp]
            lib.wp_plan_execute_host.argtypes = [vp, vp, vp, i64, i64, i64, i64, vp, vp, vp, sz, i32, vp]
            lib.wp_plan_num_passes.argtypes = [vp]
            lib.wp_plan_launches.argtypes = [vp]
            lib.wp_plan_describe.argtypes = [vp, i32]
            lib.wp_plan_describe.restype = ctypes.c_char_p
            lib.wp_plan_launches_for.argtypes = [vp, i64, i64]
            lib.wp_plan_describe_for.argtypes = [vp, i32, i64, i64]
            lib.wp_plan_describe_for.restype = ctypes.c_char_p
            lib.wp_iir_cascade.argtypes = [dp, i32, vp, vp, i64, i64, i64, i64, i32, vp, sz, vp]
            lib.wp_fir.argtypes = [dp, i32, vp, vp, i64, i64, i64, i64, i32, vp, sz, vp]
            lib.wp_iir_cascade_workspace.argtypes = [dp, i32, i64, i64, i32, ctypes.POINTER(sz)]
            lib.wp_fir_workspace.argtypes = [dp, i32, i64, i64, i32, ctypes.POINTER(sz)]
            lib.wp_white_noise.argtypes = [vp, i64, i64, i64, ctypes.c_uint64, vp]
            lib.wp_peak_abs.argtypes = [vp, i64, i64, i64, vp, vp]
            lib.wp_last_error.restype = ctypes.c_char_p
            lib.wp_launch_count.restype = ctypes.c_uint64
            lib.wp_set_trace.argtypes = [vp, sz]
            lib.wp_wav_decode.argtypes = [vp, i32, vp, i64, i64, i64, vp]
            lib.wp_wav_encode.argtypes = [vp, i64, i64, i64, i32, vp, vp, vp]
            for name in ("wp_plan_create", "wp_plan_destroy", "wp_plan_workspace_bytes", "wp_plan_execute",
                         "wp_plan_execute_host", "wp_plan_num_passes", "wp_plan_launches", "wp_plan_launches_for", "wp_iir_cascade", "wp_fir",
                         "wp_iir_cascade_workspace", "wp_fir_workspace",
                         "wp_white_noise", "wp_peak_abs", "wp_abi_version", "wp_check_device", "wp_set_trace",
                         "wp_wav_decode", "wp_wav_encode"):
                getattr(lib, name).restype = ctypes.c_int
            _lib = lib
    if require_device:
        _require_cuda()
    return _lib


def _require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device visible; the B200 engine has no CPU fallback")


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = load().wp_last_error().decode(errors="replace")
        raise KernelError(f"{what}: {msg} (code {rc})" if what else f"{msg} (code {rc})", rc)


def check_device() -> None:
    lib = load(require_device=True)
    check(lib.wp_check_device(), "device check")


def wav_decode(payload_ptr: int, encoding: int, y_ptr: int, channels: int, frames: int, ld: int, stream: int) -> None:
    check(load(require_device=True).wp_wav_decode(payload_ptr, encoding, y_ptr, channels, frames, ld, stream), "wav decode")


def wav_encode(x_ptr: int, channels: int, frames: int, ld: int, encoding: int, payload_ptr: int, clipped_ptr,
               stream: int) -> None:
    check(load(require_device=True).wp_wav_encode(x_ptr, channels, frames, ld, encoding, payload_ptr, clipped_ptr, stream),
          "wav encode")


def set_trace(ptr: int, entries: int) -> None:
    """Diagnostics: per-tile stage timestamps of tensor-core chain launches
    into a device uint64 buffer (0 disables)."""
    check(load().wp_set_trace(ptr or None, entries), "set_trace")


def launch_count() -> int:
    return int(load().wp_launch_count())


class Plan:
    """Owns a wp_plan* built from a tuple of stage entries.

    entry = (kind, coef ndarray or None, value, flags)
    """

    def __init__(self, entries):
        lib = load(require_device=True)
        self._lib = lib
        arr = (Stage * max(1, len(entries)))()
        keep = []
        for i, (kind, coef, value, flags) in enumerate(entries):
            st = arr[i]
            st.kind = kind
            st.value = float(value)
            st.flags = int(flags)
            if coef is not None:
                c = np.ascontiguousarray(coef, dtype=np.float64).reshape(-1)
                keep.append(c)
                st.coef = c.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
                st.n = c.size // 5 if kind == WP_STAGE_IIR else c.size
            else:
                st.n = 0
        handle = ctypes.c_void_p()
        check(lib.wp_plan_create(arr, len(entries), ctypes.byref(handle)), "wp_plan_create")
        self.handle = handle

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.wp_plan_destroy(h)
            except Exception:
                pass
            self.handle = None

    @property
    def num_passes(self) -> int:
        return int(self._lib.wp_plan_num_passes(self.handle))

    @property
    def launches(self) -> int:
        return int(self._lib.wp_plan_launches(self.handle))

    def describe(self):
        return [self._lib.wp_plan_describe(self.handle, i).decode() for i in range(self.num_passes)]

    def describe_for(self, channels: int, frames: int):
        """Kernels each pass launches for this call shape (IIR-only passes
        switch from the fused scan to chain_lb on large calls)."""
        return [self._lib.wp_plan_describe_for(self.handle, i, channels, frames).decode()
                for i in range(self.num_passes)]

    def launches_for(self, channels: int, frames: int) -> int:
        return int(self._lib.wp_plan_launches_for(self.handle, channels, frames))

    def workspace_bytes(self, channels: int, frames: int) -> int:
        out = ctypes.c_size_t()
        check(self._lib.wp_plan_workspace_bytes(self.handle, channels, frames, ctypes.byref(out)), "workspace")
        return int(out.value)

    def execute(self, x_ptr: int, y_ptr: int, channels: int, frames: int, ldx: int, ldy: int,
                ws_ptr: int, ws_bytes: int, stream: int) -> None:
        check(
            self._lib.wp_plan_execute(self.handle, x_ptr, y_ptr, channels, frames, ldx, ldy, ws_ptr, ws_bytes, stream),
            "wp_plan_execute",
        )

    def execute_host(self, hx_ptr: int, hy_ptr: int, channels: int, frames: int, ld_hx: int, ld_hy: int,
                     dx_ptr: int, dy_ptr: int, ws_ptr: int, ws_bytes: int, blocks: int, stream: int) -> None:
        """Host in -> host out in overlapped channel blocks (wp_plan_execute_host)."""
        check(
            self._lib.wp_plan_execute_host(self.handle, hx_ptr, hy_ptr, channels, frames, ld_hx, ld_hy,
                                           dx_ptr, dy_ptr, ws_ptr, ws_bytes, blocks, stream),
            "wp_plan_execute_host",
        )


def peak_abs(tensor) -> float:
    """max |x| of a float32 CUDA tensor [C, N] (device reduction, one float back)."""
    import torch

    lib = load(require_device=True)
    t = tensor.contiguous()
    C, N = t.shape
    out = torch.empty(1, dtype=torch.float32, device=t.device)
    with torch.cuda.device(t.device):
        check(lib.wp_peak_abs(t.data_ptr(), C, N, N, out.data_ptr(), torch.cuda.current_stream(t.device).cuda_stream),
              "wp_peak_abs")
    return float(out.item())


def white_noise(y_ptr: int, channels: int, frames: int, ld: int, seed: int, stream: int) -> None:
    lib = load(require_device=True)
    check(lib.wp_white_noise(y_ptr, channels, frames, ld, seed & 0xFFFFFFFFFFFFFFFF, stream), "wp_white_noise")
