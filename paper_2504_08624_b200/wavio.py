"""RIFF/WAVE files <-> device-resident Waves.

Same public surface and behaviour as the reference's ``wavepipe.wavio``
(pkg/src/wavepipe/wavio.py:17-200): ``WavFormat``, ``ENCODINGS``,
``load_wav(path)``, ``save_wav(wave, path, encoding="float32") -> clipped``;
pcm16 / pcm24 / float32 little-endian interleaved frames, odd chunks padded,
the same error classes (``MalformedRiff``, ``UnsupportedEncoding``,
``InvalidArgument``).

The container (a few dozen header bytes) is parsed and written on the host;
the data chunk moves through pinned memory in one copy and is de-interleaved
and decoded - or encoded and interleaved - on the GPU by ``wp_wav_decode`` /
``wp_wav_encode`` (csrc/wp_wav.cu). Decoding is exact (every pcm16/pcm24/
float32 value is a float32), and encoding reproduces the reference's
round-half-away-from-zero quantisation byte for byte for float32 samples.
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass


from .errors import InvalidArgument, MalformedRiff, UnsupportedEncoding
from .wave import Wave, _torch

__all__ = ["WavFormat", "load_wav", "save_wav", "ENCODINGS"]

_PCM, _IEEE_FLOAT = 1, 3

# encoding -> (format tag, bits per sample); bits also select the device codec
ENCODINGS = {"pcm16": (_PCM, 16), "pcm24": (_PCM, 24), "float32": (_IEEE_FLOAT, 32)}


@dataclass(frozen=True)
class WavFormat:
    """Validated stream format of a WAV file."""

    encoding: str
    fs: int
    channels: int

    def __post_init__(self):
        if self.encoding not in ENCODINGS:
            raise UnsupportedEncoding(f"encoding must be one of {sorted(ENCODINGS)}, got {self.encoding!r}")
        if self.channels < 1:
            raise InvalidArgument(f"channels must be >= 1, got {self.channels}")
        if self.fs <= 0:
            raise InvalidArgument(f"fs must be positive, got {self.fs}")


def _encoding_of(tag: int, bits: int) -> str:
    for name, (t, b) in ENCODINGS.items():
        if t == tag and b == bits:
            return name
    raise UnsupportedEncoding(f"format tag {tag} with {bits} bits per sample is not supported")


def _scan(fh, total: int):
    """Walk the RIFF chunks of an open file (chunk headers and the fmt body
    only): (WavFormat, bits, data offset, data length)."""
    fh.seek(0)
    head = fh.read(12)
    if len(head) < 12:
        raise MalformedRiff("file shorter than a RIFF header")
    magic, riff_size, form = struct.unpack_from("<4sI4s", head, 0)
    if magic != b"RIFF" or form != b"WAVE":
        raise MalformedRiff(f"not a RIFF/WAVE file (magic {magic!r}/{form!r})")
    end = 8 + riff_size
    if end > total:
        raise MalformedRiff(f"RIFF size {riff_size} exceeds file length {total}")
    fmt = payload = None
    pos = 12
    while pos + 8 <= end:
        fh.seek(pos)
        cid, size = struct.unpack("<4sI", fh.read(8))
        body = pos + 8
        if body + size > end:
            raise MalformedRiff(f"chunk {cid!r} of size {size} overruns the file")
        if cid == b"fmt ":
            if size < 16:
                raise MalformedRiff(f"fmt chunk too short ({size} bytes)")
            tag, channels, fs, _rate, block_align, bits = struct.unpack("<HHIIHH", fh.read(16))
            enc = _encoding_of(tag, bits)
            if channels < 1:
                raise MalformedRiff("fmt chunk declares zero channels")
            if fs <= 0:
                raise MalformedRiff(f"fmt chunk declares sample rate {fs}")
            if block_align != channels * (bits // 8):
                raise MalformedRiff(f"block align {block_align} inconsistent with {channels} ch x {bits} bits")
            fmt = (WavFormat(enc, fs, channels), bits, block_align)
        elif cid == b"data":
            payload = (body, size)
        pos = body + size + (size & 1)
    if fmt is None:
        raise MalformedRiff("missing fmt chunk")
    if payload is None:
        raise MalformedRiff("missing data chunk")
    if payload[1] == 0:
        raise MalformedRiff("empty data chunk")
    if payload[1] % fmt[2] != 0:
        raise MalformedRiff(f"data size {payload[1]} is not a multiple of block align {fmt[2]}")
    return fmt[0], fmt[1], payload[0], payload[1]


def load_wav(path, device=None) -> Wave:
    """Read a WAV file into a device-resident float32 Wave (planar).

    pcm16/pcm24 samples are divided by 2^15 / 2^23, float32 samples are taken
    as they are - exactly the reference's values (wavio.py:49-66)."""
    torch = _torch()
    from ._native import _require_cuda, wav_decode

    _require_cuda()
    with open(os.fspath(path), "rb") as fh:
        # the header walk reads chunk headers only; the data chunk lands straight
        # in pinned memory (no intermediate host copy)
        total = os.fstat(fh.fileno()).st_size
        try:
            fmt, bits, off, size = _scan(fh, total)
        except struct.error as exc:
            raise MalformedRiff(f"{path}: truncated chunk ({exc})") from None
        C = fmt.channels
        N = size // (C * bits // 8)
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        host = torch.empty(size, dtype=torch.uint8, pin_memory=True)
        fh.seek(off)
        if fh.readinto(memoryview(host.numpy())) != size:
            raise MalformedRiff(f"{path}: data chunk shorter than declared")
    with torch.cuda.device(dev):
        raw = host.to(dev, non_blocking=True)
        out = torch.empty((C, N), dtype=torch.float32, device=dev)
        wav_decode(raw.data_ptr(), bits, out.data_ptr(), C, N, N, torch.cuda.current_stream(dev).cuda_stream)
        raw.record_stream(torch.cuda.current_stream(dev))
    return Wave._wrap_device(out, fmt.fs)


def save_wav(wave: Wave, path, encoding: str = "float32") -> int:
    """Write ``wave`` as a canonical RIFF/WAVE file; returns the number of
    samples outside [-1, 1] (clipped by the integer encodings), as
    wavio.save_wav (wavio.py:69-114) does."""
    torch = _torch()
    from ._native import wav_encode

    if encoding not in ENCODINGS:
        raise UnsupportedEncoding(f"encoding must be one of {sorted(ENCODINGS)}, got {encoding!r}")
    if not isinstance(wave, Wave):
        raise InvalidArgument(f"expected a Wave, got {type(wave).__name__}")
    tag, bits = ENCODINGS[encoding]
    x = wave.tensor()
    C, N = x.shape
    nbytes = C * N * bits // 8
    with torch.cuda.device(x.device):
        stream = torch.cuda.current_stream(x.device).cuda_stream
        payload = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
        clipped = torch.zeros(1, dtype=torch.int64, device=x.device)
        wav_encode(x.data_ptr(), C, N, x.stride(0), bits, payload.data_ptr(), clipped.data_ptr(), stream)
        host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        host.copy_(payload, non_blocking=True)
        n_clip = int(clipped.item())  # synchronises the stream
    block_align = C * (bits // 8)
    fmt_chunk = struct.pack("<4sIHHIIHH", b"fmt ", 16, tag, C, wave.fs, wave.fs * block_align, block_align, bits)
    pad = b"\x00" if nbytes % 2 else b""
    riff_size = 4 + len(fmt_chunk) + 8 + nbytes + len(pad)
    with open(os.fspath(path), "wb") as fh:
        fh.write(struct.pack("<4sI4s", b"RIFF", riff_size, b"WAVE"))
        fh.write(fmt_chunk)
        fh.write(struct.pack("<4sI", b"data", nbytes))
        fh.write(memoryview(host.numpy()))
        fh.write(pad)
    return n_clip if encoding != "float32" else 0
