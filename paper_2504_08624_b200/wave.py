"""The signal value type: planar float32 samples + sampling rate, lazily piped.

Drop-in for the reference's ``wavepipe.Wave`` (pkg/src/wavepipe/wave.py:17-78)
with two B200-first changes:

* Storage is float32 ``[channels, frames]`` (the north star's engine dtype),
  kept in HBM as a torch CUDA tensor once the wave has touched the GPU. The
  constructor rounds its input to float32 once, so every later comparison is
  between float32 values; ``samples`` returns them widened to a read-only
  float64 ndarray, as reference callers expect (wave.py:24-33).
* ``wave | stage`` is LAZY for built-in stages: the result records the bound
  stage list and is materialised on first data access, so ``w | a | b | c``
  reaches the GPU as ONE fused chain (the reference evaluates ``(w|a)|b``
  eagerly, two HBM passes; its own TypeScript client is lazy in the same way,
  frontend/src/wave.ts:83-128). Custom duck-typed stages run eagerly.

Everything else keeps the reference's semantics: immutability, 1-D input as
one channel, validation errors, exact ``==`` and ``hash``.
"""

from __future__ import annotations

import warnings

import numpy as np

from .errors import InvalidArgument

__all__ = ["Wave", "white_noise"]


def _torch():
    import torch

    return torch


def _check_fs(fs) -> int:
    if isinstance(fs, float):
        if not fs.is_integer():
            raise InvalidArgument(f"fs must be a positive integer, got {fs}")
        fs = int(fs)
    if isinstance(fs, bool) or not isinstance(fs, (int, np.integer)):
        raise InvalidArgument(f"fs must be a positive integer, got {fs!r}")
    if fs <= 0:
        raise InvalidArgument(f"fs must be positive, got {fs}")
    return int(fs)


def _check_shape(shape) -> tuple:
    if len(shape) == 1:
        shape = (1, shape[0])
    if len(shape) != 2:
        raise InvalidArgument(f"samples must be 1-D or 2-D, got {len(shape)}-D")
    if shape[0] < 1 or shape[1] < 1:
        raise InvalidArgument(f"wave needs at least one channel and one frame, got shape {tuple(shape)}")
    return (int(shape[0]), int(shape[1]))


class Wave:
    """Immutable multichannel signal ``(channels, frames)`` + integer ``fs``."""

    __slots__ = ("_fs", "_shape", "_dev", "_host32", "_host64", "_src", "_entries", "_pinned", "__weakref__")

    def __init__(self, samples, fs: int):
        fs = _check_fs(fs)
        torch = _torch()
        if isinstance(samples, torch.Tensor):
            t = samples.detach()
            shape = _check_shape(tuple(t.shape))
            t = t.reshape(shape).to(torch.float32)
            if t.is_cuda:
                dev, host = t.contiguous().clone(), None
            else:
                dev, host = None, t.contiguous().numpy().copy()
        else:
            arr = np.array(samples, dtype=np.float64, copy=True)
            shape = _check_shape(arr.shape)
            dev, host = None, np.ascontiguousarray(arr.reshape(shape).astype(np.float32))
        self._init(fs, shape, dev=dev, host32=host)

    def _init(self, fs, shape, dev=None, host32=None, src=None, entries=None):
        object.__setattr__(self, "_fs", fs)
        object.__setattr__(self, "_shape", shape)
        object.__setattr__(self, "_dev", dev)
        if host32 is not None:
            host32.setflags(write=False)
        object.__setattr__(self, "_host32", host32)
        object.__setattr__(self, "_host64", None)
        object.__setattr__(self, "_src", src)
        object.__setattr__(self, "_entries", entries)
        object.__setattr__(self, "_pinned", None)

    # ---- constructors ------------------------------------------------------

    @classmethod
    def from_tensor(cls, tensor, fs: int, copy: bool = False) -> "Wave":
        """Wrap a float32 ``[C, N]`` tensor (CUDA or CPU, e.g. pinned) without
        copying unless ``copy``; the caller must not mutate it afterwards."""
        torch = _torch()
        fs = _check_fs(fs)
        t = tensor.detach()
        shape = _check_shape(tuple(t.shape))
        t = t.reshape(shape)
        if t.dtype != torch.float32 or not t.is_contiguous() or copy:
            t = t.to(torch.float32).contiguous().clone()
        self = object.__new__(cls)
        if t.is_cuda:
            self._init(fs, shape, dev=t)
        else:
            self._init(fs, shape, dev=None, host32=None)
            object.__setattr__(self, "_host32", t.numpy())
            object.__setattr__(self, "_pinned", t)
        return self

    @classmethod
    def _lazy(cls, src: "Wave", entries: tuple) -> "Wave":
        self = object.__new__(cls)
        self._init(src._fs, src._shape, src=src, entries=entries)
        return self

    @classmethod
    def _wrap_device(cls, tensor, fs: int) -> "Wave":
        self = object.__new__(cls)
        self._init(fs, tuple(tensor.shape), dev=tensor)
        return self

    def __setattr__(self, name, value):
        raise AttributeError("Wave is immutable")

    # ---- shape -------------------------------------------------------------

    @property
    def fs(self) -> int:
        return self._fs

    @property
    def channels(self) -> int:
        return self._shape[0]

    @property
    def frames(self) -> int:
        return self._shape[1]

    @property
    def shape(self) -> tuple:
        return self._shape

    @property
    def duration(self) -> float:
        """Length in seconds."""
        return self.frames / self.fs

    @property
    def is_lazy(self) -> bool:
        """True while the wave is a recorded chain not yet run on the GPU."""
        return self._entries is not None

    @property
    def pending_stages(self) -> int:
        return 0 if self._entries is None else len(self._entries)

    # ---- materialisation ---------------------------------------------------

    def _materialize(self):
        if self._entries is None:
            return
        from . import engine

        src = self._src
        out = engine.execute_entries(self._entries, src.tensor())
        object.__setattr__(self, "_dev", out)
        object.__setattr__(self, "_src", None)
        object.__setattr__(self, "_entries", None)

    def tensor(self, device=None):
        """The samples as a contiguous float32 CUDA tensor ``[C, N]`` (runs any
        pending chain). Do not mutate it."""
        torch = _torch()
        self._materialize()
        if self._dev is None:
            from ._native import _require_cuda

            _require_cuda()
            dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
            if self._pinned is not None:
                host = self._pinned
            else:
                with warnings.catch_warnings():  # read-only array: only copied to the device
                    warnings.simplefilter("ignore", UserWarning)
                    host = torch.from_numpy(np.ascontiguousarray(self._host32))
            object.__setattr__(self, "_dev", host.to(dev, non_blocking=True))
        if device is not None and self._dev.device != torch.device(device):
            return self._dev.to(device)
        return self._dev

    def _host_streamable(self) -> bool:
        """A pending chain over a host-resident (pinned) source: its result can
        be streamed host -> device -> host in channel blocks."""
        src = self._src
        if not (self._entries is not None and src is not None and src._dev is None and src._entries is None
                and src._pinned is not None):
            return False
        from .engine import has_normalize

        return not has_normalize(self._entries)  # Normalize needs the whole wave's peak

    def numpy32(self, out=None) -> np.ndarray:
        """Float32 host copy (``out`` may be a preallocated, e.g. pinned, array
        or tensor to copy into). A chain over a pinned host source is streamed:
        uploads, the fused passes and downloads of channel blocks overlap."""
        torch = _torch()
        if self._host_streamable() and (out is None or (isinstance(out, torch.Tensor) and out.is_pinned())):
            from . import engine

            dst = out if out is not None else torch.empty(self._shape, dtype=torch.float32, pin_memory=True)
            engine.stream_host_entries(self._entries, self._src._pinned, dst)
            if out is not None:
                return out
            host = dst.numpy()
            host.setflags(write=False)
            object.__setattr__(self, "_host32", host)
            object.__setattr__(self, "_pinned", dst)
            object.__setattr__(self, "_src", None)
            object.__setattr__(self, "_entries", None)
            return host
        self._materialize()
        if out is not None:
            torch = _torch()
            dst = out if isinstance(out, torch.Tensor) else torch.from_numpy(out)
            dst.copy_(self.tensor(), non_blocking=False)
            return out
        if self._host32 is None:
            host = self._dev.cpu().numpy()
            host.setflags(write=False)
            object.__setattr__(self, "_host32", host)
        return self._host32

    @property
    def samples(self) -> np.ndarray:
        """Read-only float64 ``[C, N]`` (the float32 samples, widened)."""
        if self._host64 is None:
            arr = self.numpy32().astype(np.float64)
            arr.setflags(write=False)
            object.__setattr__(self, "_host64", arr)
        return self._host64

    # ---- operations --------------------------------------------------------

    def channel(self, index: int) -> "Wave":
        """Single-channel wave of channel ``index``."""
        c = range(self.channels)[index]
        if self._dev is not None or self._entries is not None:
            t = self.tensor()[c : c + 1].contiguous()
            return Wave._wrap_device(t, self._fs)
        out = object.__new__(Wave)
        out._init(self._fs, (1, self.frames), host32=np.ascontiguousarray(self.numpy32()[c : c + 1]))
        return out

    def __or__(self, stage) -> "Wave":
        from .chain import pipe

        return pipe(self, stage)

    def __eq__(self, other) -> bool:
        if not isinstance(other, Wave):
            return NotImplemented
        if self._fs != other._fs or self._shape != other._shape:
            return False
        on_device = (self._dev is not None or self._entries is not None) and (
            other._dev is not None or other._entries is not None
        )
        if on_device:
            torch = _torch()
            a, b = self.tensor(), other.tensor()
            if a.device != b.device:
                b = b.to(a.device)
            return bool(torch.equal(a, b))
        return bool(np.array_equal(self.numpy32(), other.numpy32()))

    def __ne__(self, other):
        eq = self.__eq__(other)
        return eq if eq is NotImplemented else not eq

    def __hash__(self):
        return hash((self._fs, self._shape, self.numpy32().tobytes()))

    def __repr__(self) -> str:
        lazy = f", pending={len(self._entries)}" if self._entries is not None else ""
        return f"Wave(channels={self.channels}, frames={self.frames}, fs={self.fs}{lazy})"


def white_noise(duration_s: float, channels: int, fs: int, seed: int, device=None) -> Wave:
    """Deterministic N(0, 1) noise generated ON THE DEVICE.

    Same pinned stream as the reference (wave.py:141-168: splitmix64 counters,
    Box-Muller in float64, channel-major, prefix-stable), rounded to float32.
    """
    if isinstance(channels, bool) or not isinstance(channels, (int, np.integer)) or channels < 1:
        raise InvalidArgument(f"channels must be >= 1, got {channels!r}")
    if isinstance(duration_s, bool) or not (
        isinstance(duration_s, (int, float, np.floating, np.integer)) and duration_s > 0
    ):
        raise InvalidArgument(f"duration_s must be > 0, got {duration_s!r}")
    fs = _check_fs(fs)
    frames = int(round(float(duration_s) * fs))
    if frames < 1:
        raise InvalidArgument(f"duration {duration_s} s at fs {fs} rounds to zero frames")
    from ._native import white_noise as _noise, _require_cuda

    _require_cuda()
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    out = torch.empty((int(channels), frames), dtype=torch.float32, device=dev)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        _noise(out.data_ptr(), int(channels), frames, frames, int(seed), stream)
    return Wave._wrap_device(out, fs)
