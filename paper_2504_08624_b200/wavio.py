"""RIFF/WAVE files <-> device-resident Waves.

Same public surface and behaviour as the reference's ``wavepipe.wavio``
(pkg/src/wavepipe/wavio.py:17-200): ``WavFormat``, ``ENCODINGS``,
``load_wav(path)``, ``save_wav(wave, path, encoding="float32") -> clipped``;
pcm16 / pcm24 / float32 little-endian interleaved frames, odd chunks padded,
the same error classes (``MalformedRiff``, ``UnsupportedEncoding``,
``InvalidArgument``).

The container (a few dozen header bytes) is parsed and written on the host;
the data chunk streams through NBUF pinned staging buffers in chunks of whole
frames (``chunk_bytes``, 32 MiB by default): the file reads of the next chunks
(parallel threads, ``os.preadv``) overlap the host->device copy and the GPU
de-interleave/decode of the current one (``wp_wav_decode`` into the chunk's
columns of the planar wave), and on the way out the GPU encode +
device->host copy of the next chunks overlap the parallel file writes of
earlier ones (``wp_wav_encode``, csrc/wp_wav.cu). Host memory stays at NBUF
chunks whatever the file size. Decoding is exact (every pcm16/pcm24/float32
value is a float32), and encoding reproduces the reference's
round-half-away-from-zero quantisation byte for byte for float32 samples.
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass


from .errors import InvalidArgument, MalformedRiff, UnsupportedEncoding
from .wave import Wave, _torch

__all__ = ["WavFormat", "load_wav", "save_wav", "ENCODINGS"]

CHUNK_BYTES = 32 << 20  # payload bytes per pinned staging buffer
NBUF = 4                # staging buffers in flight (and file I/O threads)

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


def _chunk_frames(block_align: int, chunk_bytes: int) -> int:
    return max(1, chunk_bytes // block_align)


_POOL = None


def _io_pool():
    """Threads for the file reads / writes of the chunked pipelines (os.preadv /
    os.pwrite release the GIL, so several chunks move at once: 737 MB load
    0.12 -> 0.04 s, save 0.36 -> 0.32 s from the page cache; tools/wav_stream_bench.py)."""
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor

        _POOL = ThreadPoolExecutor(max_workers=NBUF, thread_name_prefix="wavio")
    return _POOL


def _pread_exact(fd: int, view, offset: int) -> int:
    got = 0
    while got < len(view):
        n = os.preadv(fd, [view[got:]], offset + got)
        if n <= 0:
            break
        got += n
    return got


def load_wav(path, device=None, chunk_bytes: int = CHUNK_BYTES) -> Wave:
    """Read a WAV file into a device-resident float32 Wave (planar).

    pcm16/pcm24 samples are divided by 2^15 / 2^23, float32 samples are taken
    as they are - exactly the reference's values (wavio.py:49-66). The data
    chunk streams through NBUF pinned buffers: file reads of the next chunks
    (parallel threads) overlap the copy and decode of the current one on the
    GPU."""
    torch = _torch()
    from ._native import _require_cuda, wav_decode

    _require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    with open(os.fspath(path), "rb") as fh:
        total = os.fstat(fh.fileno()).st_size
        try:
            fmt, bits, off, size = _scan(fh, total)
        except struct.error as exc:
            raise MalformedRiff(f"{path}: truncated chunk ({exc})") from None
        C = fmt.channels
        align = C * bits // 8
        N = size // align
        step = min(_chunk_frames(align, chunk_bytes), N)
        chunks = list(range(0, N, step))
        nbuf = min(NBUF, len(chunks))
        fd = fh.fileno()
        pool = _io_pool()
        with torch.cuda.device(dev):
            stream = torch.cuda.Stream(dev)
            out = torch.empty((C, N), dtype=torch.float32, device=dev)
            host = [torch.empty(step * align, dtype=torch.uint8, pin_memory=True) for _ in range(nbuf)]
            raw = [torch.empty(step * align, dtype=torch.uint8, device=dev) for _ in range(nbuf)]
            done = [None] * nbuf  # event: the copy out of pinned buffer b has completed

            def read(k):
                b, nf = k % nbuf, min(step, N - chunks[k])
                view = memoryview(host[b].numpy())[: nf * align]
                return pool.submit(_pread_exact, fd, view, off + chunks[k] * align)

            pending = {k: read(k) for k in range(nbuf)}
            for k, f0 in enumerate(chunks):
                b, nf = k % nbuf, min(step, N - f0)
                if pending.pop(k).result() != nf * align:
                    raise MalformedRiff(f"{path}: data chunk shorter than declared")
                with torch.cuda.stream(stream):
                    raw[b][: nf * align].copy_(host[b][: nf * align], non_blocking=True)
                    done[b] = torch.cuda.Event()
                    done[b].record(stream)
                    # decode into columns [f0, f0 + nf) of the planar wave (row stride N)
                    wav_decode(raw[b].data_ptr(), bits, out.data_ptr() + 4 * f0, C, nf, N, stream.cuda_stream)
                if k + nbuf < len(chunks):
                    done[b].synchronize()  # pinned buffer b is free again
                    pending[k + nbuf] = read(k + nbuf)
            torch.cuda.current_stream(dev).wait_stream(stream)
            for t in raw:
                t.record_stream(torch.cuda.current_stream(dev))
    return Wave._wrap_device(out, fmt.fs)


def save_wav(wave: Wave, path, encoding: str = "float32", chunk_bytes: int = CHUNK_BYTES) -> int:
    """Write ``wave`` as a canonical RIFF/WAVE file; returns the number of
    samples outside [-1, 1] (clipped by the integer encodings), as
    wavio.save_wav (wavio.py:69-114) does. The payload streams through NBUF
    pinned buffers: the GPU encodes and copies the next chunks while earlier
    ones are written by parallel threads."""
    torch = _torch()
    from ._native import wav_encode

    if encoding not in ENCODINGS:
        raise UnsupportedEncoding(f"encoding must be one of {sorted(ENCODINGS)}, got {encoding!r}")
    if not isinstance(wave, Wave):
        raise InvalidArgument(f"expected a Wave, got {type(wave).__name__}")
    tag, bits = ENCODINGS[encoding]
    x = wave.tensor()
    C, N = x.shape
    align = C * (bits // 8)
    nbytes = N * align
    step = min(_chunk_frames(align, chunk_bytes), N)
    chunks = list(range(0, N, step))
    nbuf = min(NBUF, len(chunks))
    fmt_chunk = struct.pack("<4sIHHIIHH", b"fmt ", 16, tag, C, wave.fs, wave.fs * align, align, bits)
    pad = b"\x00" if nbytes % 2 else b""
    riff_size = 4 + len(fmt_chunk) + 8 + nbytes + len(pad)
    head = struct.pack("<4sI4s", b"RIFF", riff_size, b"WAVE") + fmt_chunk + struct.pack("<4sI", b"data", nbytes)
    pool = _io_pool()
    with torch.cuda.device(x.device), open(os.fspath(path), "wb") as fh:
        fd = fh.fileno()
        os.pwrite(fd, head, 0)
        base = len(head)
        stream = torch.cuda.Stream(x.device)
        stream.wait_stream(torch.cuda.current_stream(x.device))  # the wave's producers
        clipped = torch.zeros(len(chunks), dtype=torch.int64, device=x.device)  # wp_wav_encode zeroes its counter
        payload = [torch.empty(step * align, dtype=torch.uint8, device=x.device) for _ in range(nbuf)]
        host = [torch.empty(step * align, dtype=torch.uint8, pin_memory=True) for _ in range(nbuf)]
        ready = [None] * nbuf
        writes = [None] * nbuf

        def launch(k):
            b, f0 = k % nbuf, chunks[k]
            nf = min(step, N - f0)
            if writes[b] is not None:
                writes[b].result()  # pinned buffer b has been written out
            with torch.cuda.stream(stream):
                wav_encode(x.data_ptr() + 4 * f0, C, nf, x.stride(0), bits, payload[b].data_ptr(),
                           clipped.data_ptr() + 8 * k, stream.cuda_stream)
                host[b][: nf * align].copy_(payload[b][: nf * align], non_blocking=True)
                ready[b] = torch.cuda.Event()
                ready[b].record(stream)

        def write(fd_, view, offset):
            while len(view):
                n = os.pwrite(fd_, view, offset)
                view, offset = view[n:], offset + n

        for k in range(nbuf):
            launch(k)
        for k in range(len(chunks)):
            b, nf = k % nbuf, min(step, N - chunks[k])
            ready[b].synchronize()
            writes[b] = pool.submit(write, fd, memoryview(host[b].numpy())[: nf * align], base + chunks[k] * align)
            if k + nbuf < len(chunks):
                launch(k + nbuf)
        for w in writes:
            if w is not None:
                w.result()
        if pad:
            os.pwrite(fd, pad, base + nbytes)
        n_clip = int(clipped.sum().item())
    return n_clip if encoding != "float32" else 0
