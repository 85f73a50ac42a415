"""The reference-side kernel seam (engine._kernels(), engine.py:74-75) backed
by the C ABI: paper_2504_08624_b200.kernels_b200 at BASELINE-shaped sizes, the
one-shot workspace queries, and the plan cache under threads."""

import ctypes
import threading

import numpy as np
import pytest

import oracle
import paper_2504_08624_b200 as wp
from paper_2504_08624_b200 import _native

pytestmark = pytest.mark.gpu

IIR_TOL = 1e-4
FIR_TOL = 1e-5


def _sos(*filters):
    return np.vstack([f.sos_rows() for f in filters])


def _x(C, N, seed):
    return np.random.default_rng(seed).standard_normal((C, N)).astype(np.float32).astype(np.float64)


def test_seam_module_exports_reference_names():
    from paper_2504_08624_b200 import kernels_b200 as k

    for name in ("iir_cascade_serial", "iir_cascade_parallel", "fir_direct_serial", "fir_direct_parallel",
                 "oracle_transversal"):
        assert callable(getattr(k, name))


def test_seam_cfg3_shaped_stage_by_stage():
    """cfg3's stages through the seam one at a time, as the reference's
    per-stage engine would call them (8 of the 32 channels, full 120 s)."""
    from paper_2504_08624_b200 import kernels_b200 as k

    fs, C, N = 48000, 8, 5_760_000
    hp = wp.design_butterworth("hp", 4, 100, fs)
    lp = wp.design_chebyshev1("lp", 4, 1.0, 8000, fs)
    fir = wp.design_fir("lp", 101, 15000, fs=fs)
    x = _x(C, N, 1)
    sos = _sos(hp, lp)
    y = k.iir_cascade_parallel(sos, x)
    ref = oracle.iir_cascade(sos, x, oracle.default_threads())
    assert oracle.parity_error(y, ref) <= IIR_TOL
    y2 = k.fir_direct_parallel(np.asarray(fir.taps), y.astype(np.float32).astype(np.float64))
    ref2 = oracle.fir_direct(np.asarray(fir.taps), y.astype(np.float32).astype(np.float64), oracle.default_threads())
    assert oracle.parity_error(y2, ref2) <= FIR_TOL


def test_seam_cfg5_shaped_large_call():
    """cfg5's LP8 through the seam on a call large enough for the single-pass
    chain (64 channels x 1.44 M samples)."""
    from paper_2504_08624_b200 import kernels_b200 as k

    lp8 = wp.design_butterworth("lp", 8, 2000, 48000)
    x = _x(64, 1_440_000, 2)
    y = k.iir_cascade_serial(lp8.sos_rows(), x)
    ref = oracle.iir_cascade(lp8.sos_rows(), x, oracle.default_threads())
    assert oracle.parity_error(y, ref) <= IIR_TOL


def test_seam_fir_fft_cfg4_taps():
    from paper_2504_08624_b200 import kernels_b200 as k

    taps = np.asarray(wp.design_fir("lp", 4096, 2000, "hamming", 48000).taps)
    x = _x(2, 2_000_000, 3)
    y = k.fir_fft(taps, x)
    assert oracle.parity_error(y, oracle.fir_direct(taps, x, oracle.default_threads())) <= FIR_TOL


def test_workspace_queries_at_baseline_shapes():
    """The one-shot size queries answer for the full BASELINE shapes (no
    allocation needed to ask) and the answer is what execute requires."""
    lib = _native.load(require_device=True)
    dp = ctypes.POINTER(ctypes.c_double)
    lp8 = np.ascontiguousarray(wp.design_butterworth("lp", 8, 2000, 48000).sos_rows())
    need = ctypes.c_size_t()
    _native.check(lib.wp_iir_cascade_workspace(lp8.ctypes.data_as(dp), lp8.shape[0], 1024, 14_400_000, 0,
                                               ctypes.byref(need)))
    tiles = 1024 * ((14_400_000 + 8191) // 8192)
    assert need.value >= tiles * 8 * 8  # published states: D = 8 words of 8 B per tile
    assert need.value < 1 << 30  # ~0.12 GB, not the 59 GB signal
    taps = np.ascontiguousarray(wp.design_fir("lp", 4096, 2000, "hamming", 48000).taps)
    _native.check(lib.wp_fir_workspace(taps.ctypes.data_as(dp), taps.size, 128, 28_800_000, _native.WP_FIR_FFT,
                                       ctypes.byref(need)))
    assert need.value < 1 << 20  # the FFT path keeps no per-tile state

    # too small a workspace is refused with the size it needs
    import torch

    x = torch.zeros((4, 400_000), device="cuda")
    y = torch.empty_like(x)
    _native.check(lib.wp_iir_cascade_workspace(lp8.ctypes.data_as(dp), lp8.shape[0], 4, 400_000, 0,
                                               ctypes.byref(need)))
    ws = torch.empty(16, dtype=torch.uint8, device="cuda")
    rc = lib.wp_iir_cascade(lp8.ctypes.data_as(dp), lp8.shape[0], x.data_ptr(), y.data_ptr(), 4, 400_000, 400_000,
                            400_000, 0, ws.data_ptr(), 16, torch.cuda.current_stream().cuda_stream)
    assert rc == -3 and str(need.value) in lib.wp_last_error().decode()


def test_plan_cache_eviction_under_threads():
    """More distinct one-shot filters than the 64-entry cache, from several
    threads at once: evicted plans stay alive while in use (shared ownership)."""
    from paper_2504_08624_b200 import kernels_b200 as k

    import torch

    errs = []

    def worker(t):
        try:
            torch.cuda.set_device(0)
            rng = np.random.default_rng(100 + t)
            for j in range(30):
                sec = wp.BiquadSection(float(rng.uniform(0.1, 1)), 0.0, 0.0, float(-rng.uniform(0.1, 0.9)), 0.0)
                f = wp.IirFilter.from_sections([sec], fs=48000)
                x = rng.standard_normal((2, 5000)).astype(np.float32).astype(np.float64)
                y = k.iir_cascade_serial(f.sos_rows(), x)
                if oracle.parity_error(y, oracle.iir_cascade(f.sos_rows(), x)) > IIR_TOL:
                    errs.append((t, j))
        except Exception as e:  # pragma: no cover - reported below
            errs.append(repr(e))

    ts = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs


def test_fused_plan_graph_replay_with_new_input():
    """A small IIR-only call (fused look-back kernel) captured in a CUDA graph
    and replayed after the input changed: the look-back records are zeroed by
    the captured memset, so no stale state from the previous replay is read."""
    import torch

    from paper_2504_08624_b200 import engine

    fs = 48000
    bound = wp.Chain([wp.design_butterworth("lp", 4, 1000)]).bind(fs).stages
    plan = engine.plan_for(bound, device=0)
    C, N = 2, 100_000
    assert plan.describe_for(C, N)[0].startswith("fused")
    x = torch.from_numpy(_x(C, N, 4).astype(np.float32)).cuda()
    y = torch.empty_like(x)
    nb = plan.workspace_bytes(C, N)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        plan.execute(x.data_ptr(), y.data_ptr(), C, N, N, N, ws.data_ptr(), nb, s.cuda_stream)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        plan.execute(x.data_ptr(), y.data_ptr(), C, N, N, N, ws.data_ptr(), nb, torch.cuda.current_stream().cuda_stream)
    for seed in (5, 6, 7):
        x.copy_(torch.from_numpy(_x(C, N, seed).astype(np.float32)))
        g.replay()
        torch.cuda.synchronize()
        ref = oracle.pipe(x.double().cpu().numpy(), bound)
        assert oracle.parity_error(y.double().cpu().numpy(), ref) <= IIR_TOL, seed
