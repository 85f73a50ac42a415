"""Channel sharding across the GPUs of one box.

Every channel of a Wave is filtered independently (the reference's channel
independence, test_engine.py:39-45), so the hot path shards with NO exchange
step: contiguous channel blocks go to different GPUs, each GPU runs the same
fused plan on its block, and the only communication is a gather of the
outputs after compute. Time-axis splitting is not used (it would need a state
carry between GPUs).

Two launchers:

* ``shard_pipe`` - one process drives every visible device: one stream per
  device, asynchronous launches, host gather into one pinned buffer.
* ``distributed_pipe`` - one process per GPU under ``torch.distributed``
  (torchrun): each rank filters its own block on its own device; the optional
  gather to one rank is a single ``gather`` of the finished blocks (gloo or
  NCCL), never part of the filter itself.

``partition`` and ``gather_blocks`` hold the host logic and run on CPU
(tests/test_sharding.py drives them with gloo, world size 2).
"""

from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np

from .errors import InvalidArgument
from .wave import Wave, _torch

__all__ = ["partition", "shard_pipe", "distributed_pipe", "gather_blocks", "local_block"]


def partition(channels: int, parts: int, align: int = 2) -> List[Tuple[int, int]]:
    """Contiguous channel blocks ``[(c0, c1), ...]`` covering ``range(channels)``.

    Blocks start at multiples of ``align`` (default 2: the FFT overlap-save
    kernel filters channels 2j and 2j+1 together, so keeping pairs on one
    device makes every result bit-identical to the unsharded run) and their
    sizes differ by at most ``align``, larger blocks first. With more parts than
    units the trailing blocks are empty (a replica has nothing to do)."""
    if isinstance(channels, bool) or not isinstance(channels, (int, np.integer)) or channels < 0:
        raise InvalidArgument(f"channels must be >= 0, got {channels!r}")
    if isinstance(parts, bool) or not isinstance(parts, (int, np.integer)) or parts < 1:
        raise InvalidArgument(f"parts must be >= 1, got {parts!r}")
    if isinstance(align, bool) or not isinstance(align, (int, np.integer)) or align < 1:
        raise InvalidArgument(f"align must be >= 1, got {align!r}")
    units = -(-int(channels) // int(align))
    base, extra = divmod(units, int(parts))
    out, u = [], 0
    for i in range(int(parts)):
        n = base + (1 if i < extra else 0)
        out.append((min(u * align, channels), min((u + n) * align, channels)))
        u += n
    return out


def local_block(channels: int, rank: int, world: int) -> Tuple[int, int]:
    """The channel block of ``rank`` among ``world`` ranks."""
    if not 0 <= rank < world:
        raise InvalidArgument(f"rank {rank} outside world of {world}")
    return partition(channels, world)[rank]


def _chain(stages):
    from .chain import Chain

    if isinstance(stages, Chain):
        return stages
    if isinstance(stages, (list, tuple)):
        return Chain(list(stages))
    return Chain([stages])


_PIN_MAX_BYTES = 4 << 30  # a gathered output larger than this is not page-locked


def shard_pipe(wave: Wave, stages, devices: Optional[Sequence] = None, gather: str = "host", out=None):
    """Filter ``wave`` through ``stages`` with its channels split across
    ``devices`` (default: every visible CUDA device).

    gather="host": returns one host-resident Wave, each device's block copied
    back as soon as it is done. ``out`` (optional): a CPU float32 tensor
    ``[C, N]`` to gather into (pinned: asynchronous copies); without it the
    gather buffer is pinned only up to 4 GiB (cfg5's 59 GB output would
    otherwise page-lock all of it). gather=None: returns the list of
    device-resident per-block Waves (no copies at all)."""
    torch = _torch()
    from ._native import _require_cuda

    _require_cuda()
    if not isinstance(wave, Wave):
        raise InvalidArgument(f"expected a Wave, got {type(wave).__name__}")
    if gather not in ("host", None):
        raise InvalidArgument(f"gather must be 'host' or None, got {gather!r}")
    if devices is None:
        devices = list(range(torch.cuda.device_count()))
    devs = [torch.device("cuda", d) if isinstance(d, int) else torch.device(d) for d in devices]
    if not devs:
        raise InvalidArgument("no devices to shard over")
    chain = _chain(stages).bind(wave.fs)
    C, N = wave.channels, wave.frames
    blocks = partition(C, len(devs))
    src = wave.tensor() if wave._dev is not None or wave._entries is not None else None
    host_src = None
    if src is None:
        host_src = wave._pinned if getattr(wave, "_pinned", None) is not None else torch.from_numpy(
            np.ascontiguousarray(wave.numpy32()))
    if host_src is not None and gather == "host" and host_src.is_pinned():
        lazy = Wave.from_tensor(host_src, wave.fs) | chain
        if lazy._host_streamable():
            # pinned host in -> pinned host out: every device streams its block
            # through wp_plan_execute_host (uploads, passes and downloads
            # overlapped per device, all devices at once)
            from .engine import stream_host_entries

            if out is None:
                out = torch.empty((C, N), dtype=torch.float32, pin_memory=C * N * 4 <= _PIN_MAX_BYTES)
            _check_out(out, C, N)
            if out.is_pinned():
                used = []
                for dev, (c0, c1) in zip(devs, blocks):
                    if c1 > c0:
                        stream_host_entries(lazy._entries, host_src[c0:c1], out[c0:c1], device=dev, sync=False)
                        used.append(dev)
                for dev in used:
                    torch.cuda.synchronize(dev)
                return Wave.from_tensor(out, wave.fs)
    shards = []
    for dev, (c0, c1) in zip(devs, blocks):
        if c1 == c0:
            continue
        with torch.cuda.device(dev):
            part = (src[c0:c1] if src is not None else host_src[c0:c1]).to(dev, non_blocking=True)
            shards.append(((c0, c1), dev, Wave._wrap_device(part.contiguous(), wave.fs)))
    shards = _run_segments(shards, chain, lambda peaks: max(peaks))
    if gather is None:
        return [w for _, _, w in shards]
    if out is None:
        out = torch.empty((C, N), dtype=torch.float32, pin_memory=C * N * 4 <= _PIN_MAX_BYTES)
    _check_out(out, C, N)
    pinned = out.is_pinned()
    for (c0, c1), dev, w in shards:
        with torch.cuda.device(dev):
            out[c0:c1].copy_(w.tensor(), non_blocking=pinned)
    for _, dev, _ in shards:
        torch.cuda.synchronize(dev)
    return Wave.from_tensor(out, wave.fs)


def _check_out(out, C, N):
    torch = _torch()
    if (not isinstance(out, torch.Tensor) or out.device.type != "cpu" or out.dtype != torch.float32
            or tuple(out.shape) != (C, N)):
        raise InvalidArgument(f"out must be a CPU float32 tensor of shape {(C, N)}")


def _run_segments(shards, chain, combine_peaks):
    """Apply a bound chain to every shard. Stages between Normalize stages run
    as one lazy (fused) chain per shard; a Normalize takes the peak over ALL
    shards (``combine_peaks``: host max, or an all-reduce across ranks) and
    applies the same fp32 factor as the unsharded scale_by_peak, as its own
    pass, so results stay bit-identical to the single-device run."""
    from .chain import Chain
    from .design import Gain, Normalize
    from .engine import normalize_scale
    from ._native import peak_abs

    torch = _torch()
    seg = []
    stages = list(chain.stages) + [None]
    for st in stages:
        if st is not None and not isinstance(st, Normalize):
            seg.append(st)
            continue
        if seg:
            fs = shards[0][2].fs if shards else None
            new = []
            for blk, dev, w in shards:
                with torch.cuda.device(dev):
                    y = w | Chain(seg).bind(fs)
                    y.tensor()  # materialise: the next step is a separate pass
                new.append((blk, dev, y))
            shards = new
            seg = []
        if st is None:
            break
        peaks = []
        for _, dev, w in shards:
            with torch.cuda.device(dev):
                peaks.append(peak_abs(w.tensor()))
        factor = normalize_scale(combine_peaks(peaks) if peaks else 0.0, st.peak)
        if factor is not None:
            new = []
            for blk, dev, w in shards:
                with torch.cuda.device(dev):
                    y = w | Gain(factor)
                    y.tensor()
                new.append((blk, dev, y))
            shards = new
    return shards


def gather_blocks(local, channels: int, group=None, dst: int = 0):
    """Gather per-rank channel blocks (``partition(channels, world)``) into the
    full ``[channels, frames]`` tensor on rank ``dst`` (None elsewhere).

    ``local`` is this rank's ``[c1 - c0, frames]`` tensor (CPU for gloo, CUDA
    for NCCL). Blocks are padded to the largest block for the collective and
    trimmed after it."""
    import torch.distributed as dist

    torch = _torch()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    blocks = partition(channels, world)
    c0, c1 = blocks[rank]
    if local.shape[0] != c1 - c0:
        raise InvalidArgument(f"rank {rank} holds {local.shape[0]} channels, its block is {c1 - c0}")
    frames = local.shape[1]
    width = max(b - a for a, b in blocks)
    send = torch.zeros((width, frames), dtype=local.dtype, device=local.device)
    send[: c1 - c0] = local
    bufs = [torch.empty_like(send) for _ in range(world)] if rank == dst else None
    dist.gather(send, gather_list=bufs, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([bufs[r][: b - a] for r, (a, b) in enumerate(blocks)], dim=0)


def distributed_pipe(local: Wave, stages, channels: int, group=None, gather_to: Optional[int] = 0):
    """One process per GPU: filter this rank's channel block ``local`` (already
    resident on this rank's device, e.g. generated there) and, if
    ``gather_to`` is not None, gather the finished blocks to that rank.

    Returns the local filtered Wave (and on ``gather_to`` the gathered full
    Wave as a second element)."""
    import torch.distributed as dist

    import torch

    chain = _chain(stages).bind(local.fs)

    def allreduce_max(peaks):
        t = torch.tensor([max(peaks) if peaks else 0.0], dtype=torch.float32,
                         device=local.tensor().device if dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        return float(t.item())

    dev = local.tensor().device
    out = _run_segments([((0, local.channels), dev, local)], chain, allreduce_max)[0][2]
    if gather_to is None:
        return out, None
    full = gather_blocks(out.tensor(), channels, group=group, dst=gather_to)
    if full is None:
        return out, None
    return out, Wave._wrap_device(full, local.fs) if full.is_cuda else Wave.from_tensor(full, local.fs)
