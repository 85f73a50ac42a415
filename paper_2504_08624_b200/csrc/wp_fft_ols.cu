// Long-FIR path for sm_100a: fused FFT overlap-save, one kernel per pass.
//
// Replaces the reference's overlap-add FFT strategy (engine._fir_fft +
// _ola_channel, engine.py:206-233: per block rfft -> multiply -> irfft, block
// sum on the host). Here every CTA turns a whole block of TWO channels into
// outputs without leaving the SM:
//
//   z[n] = x_c0[s+n] + i x_c1[s+n]        n < M = 16384 (two real channels as one
//                                         complex signal: h is real, so
//   y_c0 + i y_c1 = IFFT(FFT(z) . H)      re/im stay separate)
//
// and keeps outputs n >= Tpad (Tpad >= taps-1, multiple of 512): overlap-save,
// L = M - Tpad new outputs per block (12288 for 4096 taps), each input sample
// read (1 + Tpad/L) times, the re-reads coming from L2 (blocks of one channel
// run on neighbouring CTAs at the same time).
//
// FFT: M = 32 x 32 x 16, three register-resident passes per direction with
// two padded shared-memory transposes in between (512 threads, 32 complex
// each). The spectrum is never reordered: the forward transform leaves it in
// digit-reversed order, the host stores H in that order, and the inverse
// passes run the forward ones backwards - so the pointwise product happens
// in registers between the two last passes, with no smem round trip. Inter-
// pass twiddles W_M^n come from a two-level table (W_M^(n mod 128) x
// W_M^(128 floor(n/128)), <= 2 ulp).
#include <cuda_runtime.h>

#include "wp_internal.h"

namespace wpk {

namespace {

constexpr int FM = FFT_M;          // 16384
constexpr int FT = FFT_THREADS;    // 512
constexpr int FBUF = 17 * 1024;    // padded complex buffer
constexpr int FTW = 256 + 512 + 2048;  // twiddles: two-level W_M^n | pass 2 W_M^(32 bp k) [k][bp] | W_M^(8 m)

__constant__ float2 c_w32[16] = {
    {1.000000000e+00f, -0.000000000e+00f}, {9.807852804e-01f, -1.950903220e-01f},
    {9.238795325e-01f, -3.826834324e-01f}, {8.314696123e-01f, -5.555702330e-01f},
    {7.071067812e-01f, -7.071067812e-01f}, {5.555702330e-01f, -8.314696123e-01f},
    {3.826834324e-01f, -9.238795325e-01f}, {1.950903220e-01f, -9.807852804e-01f},
    {0.000000000e+00f, -1.000000000e+00f}, {-1.950903220e-01f, -9.807852804e-01f},
    {-3.826834324e-01f, -9.238795325e-01f}, {-5.555702330e-01f, -8.314696123e-01f},
    {-7.071067812e-01f, -7.071067812e-01f}, {-8.314696123e-01f, -5.555702330e-01f},
    {-9.238795325e-01f, -3.826834324e-01f}, {-9.807852804e-01f, -1.950903220e-01f}};

__host__ __device__ constexpr int brev(int i, int bits) {
    int r = 0;
    for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1) << (bits - 1 - b);
    return r;
}

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
    return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}

// In-register radix-2 DIF FFT of R points (R = 16 or 32), natural order in,
// v[i] = X[bitrev(i)] out. INV: conjugate twiddles (unnormalised inverse).
template <int R, bool INV>
__device__ __forceinline__ void fft_reg(float2 (&v)[R]) {
#pragma unroll
    for (int len = R; len >= 2; len >>= 1) {
        const int half = len >> 1;
#pragma unroll
        for (int st = 0; st < R; st += len) {
#pragma unroll
            for (int j = 0; j < half; ++j) {
                const float2 a = v[st + j], b = v[st + j + half];
                v[st + j] = make_float2(a.x + b.x, a.y + b.y);
                const float2 d = make_float2(a.x - b.x, a.y - b.y);
                const int m = j * (32 / len);  // W_len^j = W_32^m
                if (m == 0) {
                    v[st + j + half] = d;
                } else if (m == 8) {  // -i (forward), +i (inverse)
                    v[st + j + half] = INV ? make_float2(-d.y, d.x) : make_float2(d.y, -d.x);
                } else {
                    const float2 w = c_w32[m];
                    v[st + j + half] = INV ? cmulc(d, w) : cmul(d, w);
                }
            }
        }
    }
}

__device__ __forceinline__ float2 twid(const float2 *tw, int n) {  // W_M^n, 0 <= n < M
    return cmul(tw[n & 127], tw[128 + (n >> 7)]);
}

// v[k] *= W_M^(base k) (INV: conjugate) for k < 32, with v[k] addressed through
// brev: powers re-anchored from the table every 8 steps (<= ~8 ulp).
template <bool INV, bool BREV>
__device__ __forceinline__ void twiddle32(float2 (&v)[32], const float2 *tw, int base) {
    const float2 w1 = twid(tw, base);
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        float2 w = twid(tw, base * 8 * g);
#pragma unroll
        for (int k = 8 * g; k < 8 * g + 8; ++k) {
            const int idx = BREV ? brev(k, 5) : k;
            if (k > 0) v[idx] = INV ? cmulc(v[idx], w) : cmul(v[idx], w);
            w = cmul(w, w1);
        }
    }
}

// pass-1 twiddles v[k] *= W_M^(t k): the recurrence w <- w W_M^t, re-anchored every 8
// powers from the table t8[m] = W_M^(8 m) (t g mod 2048: odd strides, few bank conflicts;
// the two-level product it replaces read tw[8 g t mod 128] - 16-way conflicts)
template <bool INV, bool BREV>
__device__ __forceinline__ void twiddle32_p1(float2 (&v)[32], const float2 *tw, const float2 *t8, int t) {
    const float2 w1 = twid(tw, t);
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        float2 w = g == 0 ? make_float2(1.f, 0.f) : t8[(t * g) & 2047];
#pragma unroll
        for (int k = 8 * g; k < 8 * g + 8; ++k) {
            const int idx = BREV ? brev(k, 5) : k;
            if (k > 0) v[idx] = INV ? cmulc(v[idx], w) : cmul(v[idx], w);
            if (k + 1 < 8 * g + 8) w = cmul(w, w1);
        }
    }
}

// pass-2 twiddles v[k] *= W_M^(32 bp k) (INV: conjugate) straight from a table
// t2[k][bp] (512 entries; bp = thread & 15 varies fastest: conflict-free) - one
// complex multiply per point instead of the recurrence's two
template <bool INV, bool BREV>
__device__ __forceinline__ void twiddle32_tab(float2 (&v)[32], const float2 *t2, int bp) {
#pragma unroll
    for (int k = 1; k < 32; ++k) {
        const int idx = BREV ? brev(k, 5) : k;
        const float2 w = t2[16 * k + bp];
        v[idx] = INV ? cmulc(v[idx], w) : cmul(v[idx], w);
    }
}

}  // namespace

__global__ void __launch_bounds__(FT, 1) fft_ols_kernel(const FftArgs a) {
    extern __shared__ __align__(16) float2 fsm[];
    float2 *buf = fsm;
    float2 *tws = fsm + FBUF;
    const int t = threadIdx.x;
    for (int i = t; i < FTW; i += FT) tws[i] = a.tw[i];
    const float2 *tw2 = tws + 256;
    const float2 *tw8 = tws + 768;
    __syncthreads();
    const int k1p = t >> 4, bp = t & 15;  // pass-2 coordinates of this thread
    for (long long w = blockIdx.x; w < a.total; w += gridDim.x) {
        const long long pair = w / a.nblk, blk = w - pair * a.nblk;
        const long long c0 = 2 * pair, c1 = c0 + 1;
        const bool has1 = c1 < a.C;
        const long long s = blk * a.L - a.Tpad - a.delay;  // window start sample (delayed input for taps segment > 0)
        const float *x0 = a.x + c0 * a.ldx, *x1 = a.x + (has1 ? c1 : c0) * a.ldx;
        if (t == 0) {
            // warm L2 with the next work item's windows while this block is transformed
            const long long nw = w + gridDim.x;
            if (nw < a.total) {
                const long long npair = nw / a.nblk, nblk = nw - npair * a.nblk;
                const long long ns = nblk * a.L - a.Tpad - a.delay;
                long long lo = ns > 0 ? ns : 0, hi = ns + FM;
                if (hi > a.N) hi = a.N;
                lo &= ~3LL;
                hi &= ~3LL;
                if (hi > lo && (a.ldx & 3) == 0 && (reinterpret_cast<uintptr_t>(a.x) & 15) == 0) {
                    const uint32_t bytes = (uint32_t)(4 * (hi - lo));
                    const long long nc0 = 2 * npair, nc1 = nc0 + 1;
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.x + nc0 * a.ldx + lo), "r"(bytes)
                                 : "memory");
                    if (nc1 < a.C)
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.x + nc1 * a.ldx + lo),
                                     "r"(bytes)
                                     : "memory");
                }
            }
        }
        float2 v[32];
        const bool interior = s >= 0 && s + FM <= a.N;
        if (interior) {
            const float *p0 = x0 + s + t, *p1 = x1 + s + t;
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = make_float2(__ldcs(p0 + 512 * j), has1 ? __ldcs(p1 + 512 * j) : 0.f);
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const long long n = s + t + 512 * j;
                const bool ok = n >= 0 && n < a.N;
                v[j] = make_float2(ok ? x0[n] : 0.f, (ok && has1) ? x1[n] : 0.f);
            }
        }
        // ---- forward pass 1: DFT32 over j, twiddle W_M^(t k1) -> buf[k1*512 + t] ----
        fft_reg<32, false>(v);
        twiddle32_p1<false, true>(v, tws, tw8, t);
        __syncthreads();  // previous block's last reads of buf are done
#pragma unroll
        for (int k1 = 0; k1 < 32; ++k1) buf[k1 * 512 + t] = v[brev(k1, 5)];
        __syncthreads();
        // ---- forward pass 2: thread (k1p, bp): DFT32 over c, twiddle W_512^(b k2) ----
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = buf[k1p * 512 + bp + 16 * c];
        fft_reg<32, false>(v);
        twiddle32_tab<false, true>(v, tw2, bp);
        __syncthreads();
#pragma unroll
        for (int k2 = 0; k2 < 32; ++k2) buf[17 * (k1p * 32 + k2) + bp] = v[brev(k2, 5)];
        __syncthreads();
        // ---- pass 3 + pointwise product + inverse pass 3 (registers only) ----
#pragma unroll 1
        for (int gi = 0; gi < 2; ++gi) {
            const int g = t + 512 * gi;  // g = k1 * 32 + k2
            float2 u[16];
#pragma unroll
            for (int b = 0; b < 16; ++b) u[b] = buf[17 * g + b];
            fft_reg<16, false>(u);  // u[i] = Z[k3 = brev4(i)]
            float2 z[16];
#pragma unroll
            for (int k3 = 0; k3 < 16; ++k3) z[k3] = cmul(u[brev(k3, 4)], __ldg(a.H + k3 * 1024 + g));
            fft_reg<16, true>(z);  // z[i] = V[b = brev4(i)]
#pragma unroll
            for (int b = 0; b < 16; ++b) buf[17 * g + b] = z[brev(b, 4)];
        }
        __syncthreads();
        // ---- inverse pass 2: conj twiddle, IDFT32 over k2 -> c ----
#pragma unroll
        for (int k2 = 0; k2 < 32; ++k2) v[k2] = buf[17 * (k1p * 32 + k2) + bp];
        twiddle32_tab<true, false>(v, tw2, bp);
        fft_reg<32, true>(v);
        __syncthreads();
#pragma unroll
        for (int c = 0; c < 32; ++c) buf[k1p * 512 + bp + 16 * c] = v[brev(c, 5)];
        __syncthreads();
        // ---- inverse pass 1: conj twiddle W_M^(t k1), IDFT32 over k1 -> j ----
#pragma unroll
        for (int k1 = 0; k1 < 32; ++k1) v[k1] = buf[k1 * 512 + t];
        twiddle32_p1<true, false>(v, tws, tw8, t);
        fft_reg<32, true>(v);
        // outputs n = t + 512 j >= Tpad of this block (1/M folded into H)
        float *y0 = a.y + c0 * a.ldy, *y1 = a.y + (has1 ? c1 : c0) * a.ldy;
        const long long o0 = blk * a.L - a.Tpad;  // output index of window position 0
        float *q0 = y0 + o0 + t, *q1 = y1 + o0 + t;
        const int j0 = a.Tpad >> 9;  // Tpad is a multiple of 512: n = t + 512 j >= Tpad <=> j >= j0
        if (a.accumulate) {
            // taps segment > 0 of a long FIR: add to the previous segments' sum
            const long long lim = a.N - o0 - t;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                if (j >= j0 && 512LL * j < lim) {
                    const float2 r = v[brev(j, 5)];
                    q0[512 * j] += r.x;
                    if (has1) q1[512 * j] += r.y;
                }
            }
        } else if (o0 + FM <= a.N) {
            // whole block inside the signal: no per-element bound (the common case)
            if (has1) {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (j >= j0) {
                        const float2 r = v[brev(j, 5)];
                        __stcs(q0 + 512 * j, r.x);
                        __stcs(q1 + 512 * j, r.y);
                    }
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (j >= j0) __stcs(q0 + 512 * j, v[brev(j, 5)].x);
            }
        } else {
            const long long lim = a.N - o0 - t;  // valid while 512 j < lim
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                if (j >= j0 && 512LL * j < lim) {
                    const float2 r = v[brev(j, 5)];
                    __stcs(q0 + 512 * j, r.x);
                    if (has1) __stcs(q1 + 512 * j, r.y);
                }
            }
        }
    }
}

}  // namespace wpk

namespace wp {

size_t fft_ols_smem_bytes() { return sizeof(float2) * (size_t)(wpk::FBUF + wpk::FTW); }

cudaError_t fft_ols_prepare() {
    return cudaFuncSetAttribute(wpk::fft_ols_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)fft_ols_smem_bytes());
}

cudaError_t launch_fft_ols(const wpk::FftArgs &a, int grid, cudaStream_t st) {
    const size_t smem = fft_ols_smem_bytes();  // attribute set at plan build (fft_ols_prepare)
    wpk::fft_ols_kernel<<<grid, wpk::FFT_THREADS, smem, st>>>(a);
    count_launch();
    return cudaGetLastError();
}

}  // namespace wp
