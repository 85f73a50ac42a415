"""Numerics emulation of the tensor-core chain formulation (design evidence,
not product code). Run: python tools/emulate_tcchain.py

For a fused pass  pre-gain -> IIR cascade (state s, D = 2S) -> FIR f -> gain
every 64-output row m of a tile is

    y[n] = sum_{t=0}^{n-w} g[t] x[n-t]  +  E[n-w] . s_w ,   w = c_m - H

with g = gain * (f * h) (h = cascade impulse response), E[t] = gain *
sum_k f[k] C A^(t-k), and s_w the cascade state at the window start, obtained
by a float64 scan over 64-sample chunks  s_{w+64} = A^64 s_w + e,
e = sum_j A^(63-j) B x[w+j]. Products run as fp16 x3 split (hi*hi + hi*lo +
lo*hi) with fp32 accumulation per K-block of 16 (tcgen05 kind::f16).
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import oracle  # noqa: E402
import paper_2504_08624_b200 as wp  # noqa: E402


def cascade_ss(sos):
    S = sos.shape[0]
    D = 2 * S

    def step(s, u):
        out = np.zeros(D)
        for k in range(S):
            b0, b1, b2, a1, a2 = sos[k]
            w1, w2 = s[2 * k], s[2 * k + 1]
            y = b0 * u + w1
            out[2 * k] = b1 * u - a1 * y + w2
            out[2 * k + 1] = b2 * u - a2 * y
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


def split16(v, scale):
    v = v * scale
    hi = v.astype(np.float16).astype(np.float64)
    lo = ((v - hi) * 2048).astype(np.float16).astype(np.float64)
    return hi, lo


def mma_acc(a_hi, a_lo, b_hi, b_lo, kblk=16):
    """a [R,K], b [P,K] -> [R,P]; fp32 accumulate, one rounding per K block."""
    R, K = a_hi.shape
    acc_m = np.zeros((R, b_hi.shape[0]), dtype=np.float32)
    acc_c = np.zeros_like(acc_m)
    for k0 in range(0, K, kblk):
        sl = slice(k0, k0 + kblk)
        acc_m = (acc_m.astype(np.float64) + a_hi[:, sl] @ b_hi[:, sl].T).astype(np.float32)
        acc_c = (acc_c.astype(np.float64) + a_lo[:, sl] @ b_hi[:, sl].T).astype(np.float32)
        acc_c = (acc_c.astype(np.float64) + a_hi[:, sl] @ b_lo[:, sl].T).astype(np.float32)
    return acc_m.astype(np.float64) + acc_c.astype(np.float64) / 2048


def emulate(x, sos, taps, gain, H=112, tile_rows=128, exact=False, state_mode='f32', acc=True):
    A, B, C, d = cascade_ss(sos)
    D = A.shape[0]
    T = taps.size
    Kw = H + 64
    # impulse response of the cascade and combined g
    nh = Kw
    h = np.zeros(nh)
    s = np.zeros(D)
    for n in range(nh):
        u = 1.0 if n == 0 else 0.0
        h[n] = C @ s + d * u
        s = A @ s + B * u
    g = gain * np.convolve(taps, h)[:Kw]
    # CA^t for t up to Kw
    CA = np.zeros((Kw + 1, D))
    row = C.copy()
    for t in range(Kw + 1):
        CA[t] = row
        row = row @ A
    E = np.zeros((64, D))
    for p in range(64):
        t = H + p
        for k in range(T):
            E[p] += taps[k] * CA[t - k]
    E *= gain
    Kc = np.zeros((64, D))
    v = B.copy()
    for j in range(63, -1, -1):
        Kc[j] = v
        v = A @ v
    M = np.linalg.matrix_power(A, 64)

    N = x.size
    rows = (N + 63) // 64
    xp = np.concatenate([np.zeros(H), x, np.zeros(64 * rows + 64 - N)])
    # Hankel rows: window start w_m = 64 m - H  -> xp index 64 m
    idx = 64 * np.arange(rows)[:, None] + np.arange(Kw)[None, :]
    Aw = xp[idx]  # [rows, Kw]
    Bg = np.zeros((64, Kw))
    for p in range(64):
        for k in range(Kw):
            t = p + H - k
            if 0 <= t < Kw:
                Bg[p, k] = g[t]
    Bk = np.zeros((16, Kw))
    Bk[:D, :64] = Kc.T  # chunk [w, w+64) end state
    y = np.zeros(rows * 64)
    # per tile scaling as on the GPU
    gmax = np.max(np.abs(Bg))
    fB = 14 - np.frexp(gmax)[1]
    kmax = np.max(np.abs(Bk))
    fK = 14 - np.frexp(kmax)[1]
    Emax = np.max(np.abs(E), axis=0)
    fE = np.array([14 - np.frexp(m)[1] if m > 0 else 0 for m in Emax])
    s = np.zeros(D)
    for t0 in range(0, rows, tile_rows):
        r = slice(t0, min(rows, t0 + tile_rows))
        a = Aw[r]
        xm = np.max(np.abs(a))
        ex = np.frexp(xm)[1] if xm > 0 else 0
        sc = 2.0 ** (14 - ex)
        if exact:
            e = a @ Bk.T
            main = a @ Bg.T
        else:
            ah, al = split16(a, sc)
            bh, bl = split16(Bk, 2.0**fK)
            e = mma_acc(ah, al, bh, bl) / sc / 2.0**fK
            bh, bl = split16(Bg, 2.0**fB)
            main = mma_acc(ah, al, bh, bl) / sc / 2.0**fB
        e = e[:, :D]
        # fp64 scan over rows of this tile
        S_rows = np.zeros((a.shape[0], D))
        for i in range(a.shape[0]):
            S_rows[i] = s
            s = M @ s + e[i]
        if exact:
            st = S_rows @ E.T
        elif state_mode == 'f32':
            # CUDA cores: fp32 E, fp32 s, fp32 FMA chain over the D states
            E32 = E.astype(np.float32)
            S32 = S_rows.astype(np.float32)
            st = np.zeros((a.shape[0], 64), dtype=np.float32)
            for i in range(D):
                st = (st.astype(np.float64) + np.float64(1) * S32[:, i:i+1].astype(np.float64) * E32[None, :, i].astype(np.float64)).astype(np.float32)
        elif state_mode == 'f64':
            st = S_rows @ E.T
        else:
            # per-row scale of the state operand, per-column scale of E
            Es = E * 2.0 ** fE[None, :]
            Ss = S_rows * 2.0 ** (-fE[None, :])
            rm = np.max(np.abs(Ss), axis=1)
            rs = np.array([2.0 ** (14 - np.frexp(v)[1]) if v > 0 else 1.0 for v in rm])
            sh, sl = split16(Ss * rs[:, None], 1.0)
            eh, el = split16(Es, 1.0)
            st = mma_acc(sh, sl, eh, el) / rs[:, None]
        yt = (main.astype(np.float32) + st.astype(np.float32)).astype(np.float32)
        y[64 * t0 : 64 * t0 + yt.size] = yt.reshape(-1)
    return y[:N]


def main():
    fs = 48000
    stages = wp.Chain([wp.design_butterworth("hp", 4, 100), wp.design_chebyshev1("lp", 4, 1.0, 8000),
                       wp.design_fir("lp", 101, 15000), wp.Gain(0.5)]).bind(fs).stages
    rows = []
    for st in stages[:2]:
        r = np.array([[s.b0, s.b1, s.b2, s.a1, s.a2] for s in st.sections])
        r[0, :3] *= st.overall_gain
        rows.append(r)
    sos = np.vstack(rows)
    taps = np.asarray(stages[2].taps)
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 48000 * 2
    n = np.arange(N)
    inputs = {
        "noise": oracle.white_noise(N / fs, 1, fs, 42)[0],
        "sin50+440": 0.5 * np.sin(2 * np.pi * 50 * n / fs) + 0.3 * np.sin(2 * np.pi * 440 * n / fs),
        "0.9sin30": 0.9 * np.sin(2 * np.pi * 30 * n / fs),
        "sin440": 0.5 * np.sin(2 * np.pi * 440 * n / fs),
    }
    for name, x in inputs.items():
        x = x.astype(np.float32).astype(np.float64)
        ref = oracle.pipe(x[None], stages)[0]
        ye = emulate(x, sos, taps, 0.5, exact=True)
        yt = emulate(x, sos, taps, 0.5)
        print(f"{name:10s} peak_in {np.max(np.abs(x)):.3f} peak_out {np.max(np.abs(ref)):.4f} "
              f"formulation(f64) {oracle.parity_error(ye, ref):.2e}  fp16x3 {oracle.parity_error(yt, ref):.2e}")


if __name__ == "__main__":
    main()
