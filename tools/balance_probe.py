"""Why chain_lb scans in fp32 in a BALANCED state basis (host emulation, numpy).

The chained row scan s_{m+1} = M s_m + e_m (M = A^64, 64-sample rows) and the
state term E s are evaluated in float32 in two realizations of the same cascade:
the reference's DF2T states (_kernels_jit.py:27-32) and the per-section balanced
basis chain_lb uses (csrc/wp_lb.cu balance_section). The output error is printed
relative to the output peak against a float64 direct DF2T run, for cfg3's IIR part
(Butterworth HP4 100 Hz | Chebyshev-I LP4 1 dB 8 kHz) on noise and on the
stopband input 0.9 sin(2 pi 30 t) (output ~100x smaller than the state terms).

python tools/balance_probe.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2504_08624_b200 as wp  # noqa: E402

FS = 48000


def df2t_ss(sos):
    """State space (A, B, C, d) of the DF2T cascade, states section-major."""
    S = len(sos)
    D = 2 * S

    def step(st, u):
        out = np.zeros(D)
        for s, (b0, b1, b2, a1, a2) in enumerate(sos):
            y = b0 * u + st[2 * s]
            out[2 * s] = b1 * u - a1 * y + st[2 * s + 1]
            out[2 * s + 1] = b2 * u - a2 * y
            u = y
        return out, u

    A = np.zeros((D, D))
    C = np.zeros(D)
    for j in range(D):
        e = np.zeros(D)
        e[j] = 1
        A[:, j], C[j] = step(e, 0.0)
    B, d = step(np.zeros(D), 1.0)
    return A, B, C, d


def lyap(A, Q):
    # W = A W A^T + Q by Smith doubling
    W, Ak = Q.copy(), A.copy()
    for _ in range(60):
        W = W + Ak @ W @ Ak.T
        Ak = Ak @ Ak
    return W


def balanced(A, B, C, sos):
    """Per-section balancing transform (block-diagonal T): each section balanced on its own
    DF2T realization (A_s = [[-a1, 1], [-a2, 0]], B_s = (b1 - a1 b0, b2 - a2 b0), C_s = (1, 0)),
    as csrc/wp_lb.cu balance_section does."""
    D = A.shape[0]
    T = np.eye(D)
    Ti = np.eye(D)
    for s, (b0, b1, b2, a1, a2) in enumerate(sos):
        As = np.array([[-a1, 1.0], [-a2, 0.0]])
        Bs = np.array([b1 - a1 * b0, b2 - a2 * b0])
        Cs = np.array([1.0, 0.0])
        Wc = lyap(As, np.outer(Bs, Bs))
        Wo = lyap(As.T, np.outer(Cs, Cs))
        Lc = np.linalg.cholesky(Wc + 1e-15 * np.trace(Wc) * np.eye(2))
        Lo = np.linalg.cholesky(Wo + 1e-15 * np.trace(Wo) * np.eye(2))
        U, sv, Vt = np.linalg.svd(Lo.T @ Lc)
        sl = slice(2 * s, 2 * s + 2)
        T[sl, sl] = np.diag(sv ** -0.5) @ U.T @ Lo.T
        Ti[sl, sl] = Lc @ Vt.T @ np.diag(sv ** -0.5)
    return T @ A @ Ti, T @ B, C @ Ti


def run_chunked_f32(A, B, C, d, x, rows=64):
    """fp32 emulation of the chain's state path: e_m, row-chained states, E s per output."""
    D = A.shape[0]
    n = len(x) // rows * rows
    x = x[:n]
    M = np.linalg.matrix_power(A, rows).astype(np.float32)
    Ke = np.stack([np.linalg.matrix_power(A, rows - 1 - j) @ B for j in range(rows)]).astype(np.float32)  # [rows][D]
    Ep = np.stack([C @ np.linalg.matrix_power(A, p) for p in range(rows)]).astype(np.float32)  # [rows][D]
    h = np.array([d] + [C @ np.linalg.matrix_power(A, t - 1) @ B for t in range(1, rows)])  # impulse (fp64 GEMM part)
    X = x.reshape(-1, rows)
    e = (X.astype(np.float32) @ Ke).astype(np.float32)  # [R][D]
    s = np.zeros(D, np.float32)
    y = np.empty_like(X, dtype=np.float64)
    for m in range(X.shape[0]):
        # window part exactly (the GEMM is f16x3 ~ fp32 accurate; not the point here)
        y[m] = np.convolve(X[m].astype(np.float64), h)[:rows] + (Ep @ s).astype(np.float64)
        s = (M @ s + e[m]).astype(np.float32)
    return y.reshape(-1)


def direct_f64(sos, x):
    from scipy.signal import sosfilt
    sos = np.asarray(sos, dtype=np.float64)  # rows (b0, b1, b2, a1, a2) -> scipy's (b0, b1, b2, 1, a1, a2)
    return sosfilt(np.hstack([sos[:, :3], np.ones((len(sos), 1)), sos[:, 3:]]), x)


def main():
    hp = wp.design_butterworth("hp", 4, 100).bind(FS)
    lp = wp.design_chebyshev1("lp", 4, 1.0, 8000).bind(FS)
    sos = np.vstack([hp.sos_rows(), lp.sos_rows()])
    A, B, C, d = df2t_ss(sos)
    Ab, Bb, Cb = balanced(A, B, C, sos)
    n = 48000 * 2
    t = np.arange(n) / FS
    inputs = {"noise": np.random.default_rng(1).standard_normal(n).astype(np.float32).astype(np.float64),
              "0.9 sin 30 Hz": (0.9 * np.sin(2 * np.pi * 30 * t)).astype(np.float32).astype(np.float64)}
    for name, x in inputs.items():
        ref = direct_f64(sos, x)[: n // 64 * 64]
        peak = np.max(np.abs(ref))
        for label, (AA, BB, CC) in {"DF2T": (A, B, C), "balanced": (Ab, Bb, Cb)}.items():
            y = run_chunked_f32(AA, BB, CC, d, x)
            print(f"{name:14s} {label:9s} fp32 scan: max err / peak = {np.max(np.abs(y - ref)) / peak:.2e}"
                  f"   (state norm {np.linalg.norm(CC):.2e}, |M| {np.abs(np.linalg.matrix_power(AA, 64)).max():.2e})")


if __name__ == "__main__":
    main()
