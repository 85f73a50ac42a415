"""Channel sharding: partition properties on CPU, the
multi-rank gather with gloo at world size 2 (each rank filters its own block
with the CPU oracle standing in for its GPU), and - on a GPU - shard_pipe
bit-identical to the unsharded pipe."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2504_08624_b200 as wp
from paper_2504_08624_b200.sharding import gather_blocks, local_block, partition


@pytest.mark.parametrize("C", [0, 1, 2, 3, 7, 32, 33, 1024])
@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
def test_partition_covers_contiguously(C, parts):
    blocks = partition(C, parts)
    assert len(blocks) == parts
    c = 0
    for a, b in blocks:
        assert a == c and b >= a
        assert a % 2 == 0 or a == C  # channel pairs never straddle devices
        c = b
    assert c == C
    sizes = [b - a for a, b in blocks]
    assert max(sizes) - min(sizes) <= 3  # align 2, plus an odd last channel


def test_partition_align_one_is_balanced():
    sizes = [b - a for a, b in partition(1024, 3, align=1)]
    assert sizes == [342, 341, 341]


def test_partition_rejects_bad_arguments():
    with pytest.raises(wp.InvalidArgument):
        partition(-1, 2)
    with pytest.raises(wp.InvalidArgument):
        partition(4, 0)
    with pytest.raises(wp.InvalidArgument):
        local_block(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, C, N, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fs = 48000
        stages = wp.Chain([wp.design_butterworth("hp", 2, 200), wp.design_fir("lp", 31, 5000)]).bind(fs).stages
        x = oracle.white_noise(N / fs, C, fs, 5).astype(np.float32).astype(np.float64)
        c0, c1 = local_block(C, rank, world)
        # this rank's block, filtered locally (the CPU oracle stands in for the GPU)
        local = torch.from_numpy(oracle.pipe(x[c0:c1], stages)) if c1 > c0 else torch.zeros((0, N), dtype=torch.float64)
        full = gather_blocks(local, C, dst=0)
        if rank == 0:
            ref = oracle.pipe(x, stages)
            result_q.put(bool(np.array_equal(full.numpy(), ref)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("C", [5, 8])
def test_gather_blocks_gloo_world2(C):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, C, 3000, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


@pytest.mark.gpu
@pytest.mark.parametrize("C", [1, 3, 8])
def test_shard_pipe_matches_pipe_bit_exact(C):
    fs = 48000
    w = wp.white_noise(0.5, C, fs, seed=3)
    chain = wp.Chain([wp.design_butterworth("hp", 4, 100), wp.design_fir("lp", 101, 15000), wp.Gain(0.5)])
    ref = (w | chain).samples
    # every visible device, and the same device listed twice (two shards, one GPU)
    for devices in (None, [0, 0]):
        got = wp.shard_pipe(w, chain, devices=devices).samples
        assert np.array_equal(got, ref)


@pytest.mark.gpu
def test_shard_pipe_fft_path_pairs_bit_exact():
    fs = 48000
    w = wp.white_noise(2.0, 6, fs, seed=9)
    fir = wp.design_fir("lp", 2048, 2000)
    ref = (w | fir).samples
    got = wp.shard_pipe(w, fir, devices=[0, 0, 0]).samples
    assert np.array_equal(got, ref)
    shards = wp.shard_pipe(w, fir, devices=[0, 0], gather=None)
    assert [s.channels for s in shards] == [4, 2]


@pytest.mark.gpu
@pytest.mark.parametrize("C", [3, 8])
def test_shard_pipe_normalize_uses_the_global_peak(C):
    """Normalize over a sharded wave takes the peak of ALL channels (not each
    shard's own), bit-identical to the unsharded chain (high)."""
    fs = 48000
    rng = np.random.default_rng(C)
    x = rng.standard_normal((C, 30000))
    x[-1] *= 10.0  # the loudest channel lives on the last shard only
    w = wp.Wave(x, fs)
    chain = wp.Chain([wp.design_butterworth("hp", 4, 100), wp.Normalize(0.8),
                      wp.design_fir("lp", 33, 9000), wp.Gain(0.5)])
    ref = (w | chain).samples
    for devices in ([0, 0], [0, 0, 0]):
        got = wp.shard_pipe(w, chain, devices=devices).samples
        assert np.array_equal(got, ref), devices
    assert np.max(np.abs(ref[:, :]))  # sanity


@pytest.mark.gpu
def test_pinned_source_chain_with_normalize_is_not_streamed_per_block():
    """A lazy chain with Normalize over a pinned host source is materialised on
    the whole wave (one peak), not streamed block by block (high)."""
    import torch

    fs = 48000
    rng = np.random.default_rng(2)
    x = rng.standard_normal((6, 40000)).astype(np.float32)
    x[0] *= 5.0
    chain = wp.Chain([wp.design_butterworth("lp", 4, 2000), wp.Normalize(1.0)])
    ref = (wp.Wave(x.astype(np.float64), fs) | chain).samples
    pinned = torch.from_numpy(x).pin_memory()
    lazy = wp.Wave.from_tensor(pinned, fs) | chain
    assert not lazy._host_streamable()
    got = lazy.numpy32().astype(np.float64)
    assert np.array_equal(got, ref)
    assert np.max(np.abs(got)) == pytest.approx(1.0, rel=1e-6)


@pytest.mark.gpu
@pytest.mark.parametrize("fft", [False, True])
def test_shard_pipe_pinned_source_streams_per_device(fft):
    """A pinned host source is streamed per device through wp_plan_execute_host
    (all devices enqueued, then synchronised), bit-identical to one device;
    a pageable caller buffer takes the upload/run/gather path."""
    import torch

    fs = 48000
    w = wp.white_noise(0.5, 7, fs, seed=13)
    chain = wp.Chain([wp.design_fir("lp", 2048, 2000)]) if fft else \
        wp.Chain([wp.design_butterworth("hp", 4, 100), wp.design_fir("lp", 101, 15000), wp.Gain(0.5)])
    ref = (w | chain).samples
    pinned = torch.empty((7, w.frames), dtype=torch.float32, pin_memory=True)
    pinned.copy_(w.tensor())
    src = wp.Wave.from_tensor(pinned, fs)
    for devices in (None, [0, 0], [0, 0, 0]):
        got = wp.shard_pipe(src, chain, devices=devices)
        assert got._pinned is not None and got._pinned.is_pinned()
        assert np.array_equal(got.samples, ref), devices
    out = torch.empty((7, w.frames), dtype=torch.float32)
    assert np.array_equal(wp.shard_pipe(src, chain, devices=[0, 0], out=out).samples, ref)


@pytest.mark.gpu
def test_shard_pipe_into_caller_buffer():
    """gather into a caller-provided host tensor (pinned or pageable), as a
    59 GB cfg5 output should be, instead of a fresh page-locked buffer."""
    import torch

    fs = 48000
    w = wp.white_noise(0.5, 5, fs, seed=11)
    chain = wp.Chain([wp.design_butterworth("lp", 8, 2000)])
    ref = (w | chain).samples
    for pin in (True, False):
        out = torch.empty((5, w.frames), dtype=torch.float32, pin_memory=pin)
        got = wp.shard_pipe(w, chain, devices=[0, 0], out=out)
        assert np.array_equal(got.samples, ref)
        assert np.array_equal(out.numpy().astype(np.float64), ref)
    with pytest.raises(wp.InvalidArgument):
        wp.shard_pipe(w, chain, devices=[0], out=torch.empty((4, w.frames)))


@pytest.mark.gpu
@pytest.mark.skipif(not __import__("torch").cuda.is_available() or __import__("torch").cuda.device_count() < 2,
                    reason="needs >= 2 visible GPUs")
def test_shard_pipe_real_devices():
    """Channels split over every visible GPU (one stream each), bit-identical to one GPU."""
    import torch

    fs = 48000
    n = torch.cuda.device_count()
    w = wp.white_noise(1.0, 4 * n + 1, fs, seed=12)
    chain = wp.Chain([wp.design_butterworth("hp", 4, 100), wp.design_chebyshev1("lp", 4, 1.0, 8000),
                      wp.design_fir("lp", 101, 15000), wp.Gain(0.5)])
    ref = (w | chain).samples
    got = wp.shard_pipe(w, chain, devices=list(range(n))).samples
    assert np.array_equal(got, ref)
