// Fused filter-chain kernel for sm_100a: [pre-gain] -> IIR SOS cascade
// (chunked linear-recurrence scan) -> [FIR direct] -> [post-gains], one HBM
// read and one HBM write per sample. Replaces the reference's per-stage
// passes: _iir_channel (_kernels_jit.py:14-32), _fir_channel (:51-62) and the
// stage loop of Chain.apply (chain.py:66-71).
//
// Work decomposition
//   tile      = one CTA-iteration: a contiguous region of NT*L samples of one
//               channel; the first H samples are the FIR halo, the remaining
//               Lout = NT*L - H are this tile's outputs. Tiles are claimed from
//               a global counter in k-major order (k = tile index within the
//               channel, channels interleaved) by persistent CTAs.
//   chunk     = L consecutive samples owned by one thread.
// IIR scan ("re-run" formulation; D = 2S state = (w1,w2) per DF2T section)
//   pass 1   e_t = sum_n K[n] x_n          end state of chunk t from zero state
//   warp     Kogge-Stone over lanes with P[i] = M^(2^i), M = A^L (chunk transfer)
//   CTA      sequential combine of NW warp aggregates with W = M^32
//   grid     decoupled look-back over tiles with MT = M^(NT - H/L); lanes of
//            warp 0 inspect 32 predecessors at once and reduce MT^j * value_j
//   pass 2   exact DF2T recurrence from each chunk's true carry-in state
// All transfer matrices are block lower triangular (section s only sees
// sections <= s); the matvecs skip the zero blocks at compile time.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace wpk {

constexpr int NT = 128;          // threads per CTA
constexpr int NW = NT / 32;      // warps per CTA
constexpr int L = 64;            // samples per thread chunk
constexpr int CQ = L / 4;        // float4 per chunk
constexpr int REGION = NT * L;   // samples per tile region
constexpr int MAXS = 4;          // sections per fused IIR block
constexpr int MAXPOST = 4;

struct FusedArgs {
    const float *x;
    float *y;
    long long C, N, ldx, ldy;
    long long total_tiles;
    int Lout, H;        // outputs per tile, FIR halo (multiple of L)
    int Tpad;           // FIR taps rounded up to 8 (0 = no FIR)
    int vec_x, vec_y;   // 16-byte vector paths allowed
    const float *taps;  // [Tpad] zero padded, reversed order not needed
    float pre_gain;
    int n_post;
    float post[MAXPOST];
    const void *G;      // [D][D][33] scan dtype: M^l, l = 0..32 (lane-minor)
    const void *TP;     // [33][D][D] scan dtype: MT^j, j = 0..32
    unsigned int *counter;
    void *recs;
    unsigned long long epoch;
};

template <typename TS, int S>
struct IirTables {
    static constexpr int D = S > 0 ? 2 * S : 1;
    TS sos[S > 0 ? S : 1][5];
    TS K[L][D];
    TS P[5][D][D];
    TS W[NW][D][D];
    TS MT[D][D];
};

template <typename TS, int D>
struct alignas(16) TileRec {
    unsigned long long flag;
    unsigned long long pad;
    TS agg[D];
    TS incl[D];
};

__device__ __forceinline__ int swz(int q4) {
    const int t = q4 / CQ;
    const int j = q4 % CQ;
    return t * CQ + (j ^ (t & 7));
}

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <typename T>
__device__ __forceinline__ T shfl_up(T v, int d) {
    return __shfl_up_sync(0xffffffffu, v, d);
}

template <typename T>
__device__ __forceinline__ T shfl_xor(T v, int d) {
    return __shfl_xor_sync(0xffffffffu, v, d);
}

__device__ __forceinline__ float ldcg(const float *p) { return __ldcg(p); }
__device__ __forceinline__ double ldcg(const double *p) { return __ldcg(p); }

// out += M v for a block-lower-triangular M given by accessor m(i, j)
template <int D, typename TS, typename F>
__device__ __forceinline__ void matvec_acc(TS (&out)[D], const TS (&v)[D], F m) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
#pragma unroll
        for (int j = 0; j < D; ++j) {
            if ((j >> 1) > (i >> 1)) continue;
            out[i] = fma(m(i, j), v[j], out[i]);
        }
    }
}

__device__ __forceinline__ float4 load_region4(const float *row, long long pos, long long N, int vec) {
    float4 v;
    if (vec && pos >= 0 && pos + 4 <= N) {
        v = __ldcs(reinterpret_cast<const float4 *>(row + pos));
    } else {
        v.x = (pos + 0 >= 0 && pos + 0 < N) ? row[pos + 0] : 0.f;
        v.y = (pos + 1 >= 0 && pos + 1 < N) ? row[pos + 1] : 0.f;
        v.z = (pos + 2 >= 0 && pos + 2 < N) ? row[pos + 2] : 0.f;
        v.w = (pos + 3 >= 0 && pos + 3 < N) ? row[pos + 3] : 0.f;
    }
    return v;
}

__device__ __forceinline__ void store4(float *row, long long pos, long long N, int vec, float4 v) {
    if (vec && pos + 4 <= N) {
        __stcs(reinterpret_cast<float4 *>(row + pos), v);
    } else {
        if (pos + 0 < N) row[pos + 0] = v.x;
        if (pos + 1 < N) row[pos + 1] = v.y;
        if (pos + 2 < N) row[pos + 2] = v.z;
        if (pos + 3 < N) row[pos + 3] = v.w;
    }
}

__device__ __forceinline__ float apply_post(float v, const FusedArgs &a) {
    for (int i = 0; i < a.n_post; ++i) v *= a.post[i];
    return v;
}

// dynamic shared memory layout
template <typename TS, int S>
struct SmemLayout {
    static constexpr int D = S > 0 ? 2 * S : 1;
    static constexpr size_t region = 0;
    static constexpr size_t region_bytes = sizeof(float) * REGION;
    static constexpr size_t g = region + region_bytes;
    static constexpr size_t g_bytes = S > 0 ? sizeof(TS) * D * D * 33 : 0;
    static constexpr size_t tp = (g + g_bytes + 15) & ~size_t(15);
    static constexpr size_t tp_bytes = S > 0 ? sizeof(TS) * 33 * D * D : 0;  // look-back powers (M^T)^j
    static constexpr size_t misc = (tp + tp_bytes + 15) & ~size_t(15);
    // warp_incl[NW][D], wc[NW][D], WC[NW][D], agg[D], sin[D], agg_incl[D]
    static constexpr size_t misc_bytes = sizeof(TS) * (3 * NW * D + 3 * D) + 16;
    static constexpr size_t taps = (misc + misc_bytes + 15) & ~size_t(15);
    static size_t total(int tpad) { return taps + sizeof(float) * (size_t)tpad; }
};

template <typename TS, int S, bool FIR>
__global__ void __launch_bounds__(NT, 3) fused_chain_kernel(const FusedArgs a, const IirTables<TS, S> tb) {
    constexpr int D = IirTables<TS, S>::D;
    using Lay = SmemLayout<TS, S>;
    extern __shared__ __align__(16) unsigned char smem[];
    float *region = reinterpret_cast<float *>(smem + Lay::region);
    float4 *reg4 = reinterpret_cast<float4 *>(region);
    TS *gsm = reinterpret_cast<TS *>(smem + Lay::g);
    TS *tpsm = reinterpret_cast<TS *>(smem + Lay::tp);
    long long *tile_s = reinterpret_cast<long long *>(smem + Lay::misc);
    TS *warp_incl = reinterpret_cast<TS *>(smem + Lay::misc + 16);
    TS *wc_s = warp_incl + NW * D;
    TS *WC_s = wc_s + NW * D;
    TS *agg_s = WC_s + NW * D;
    TS *sin_s = agg_s + D;
    TS *aggin_s = sin_s + D;
    float *taps_s = reinterpret_cast<float *>(smem + Lay::taps);

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;

    // one-time staging of per-plan tables
    if constexpr (S > 0) {
        const TS *G = reinterpret_cast<const TS *>(a.G);
        for (int i = tid; i < D * D * 33; i += NT) gsm[i] = G[i];
        const TS *TPg = reinterpret_cast<const TS *>(a.TP);
        for (int i = tid; i < 33 * D * D; i += NT) tpsm[i] = TPg[i];
    }
    if constexpr (FIR) {
        for (int i = tid; i < a.Tpad; i += NT) taps_s[i] = a.taps[i];
    }

    const int tagg = NT - a.H / L - 1;  // chunk whose end is the next tile's region start
    const int lt_agg = tagg & 31, wt_agg = tagg >> 5;

    for (;;) {
        __syncthreads();  // previous tile fully consumed (region, misc)
        if (tid == 0) *tile_s = (long long)atomicAdd(a.counter, 1u);
        __syncthreads();
        const long long tile = *tile_s;
        if (tile >= a.total_tiles) break;
        const long long c = tile % a.C;
        const long long k = tile / a.C;
        const long long out0 = k * (long long)a.Lout;
        const long long r0 = out0 - a.H;
        const float *xr = a.x + c * a.ldx;
        float *yr = a.y + c * a.ldy;

        // ---- load region (coalesced) into the swizzled chunk layout ----
        {
            constexpr int NB = 8;  // float4 loads in flight per thread
            const bool interior = a.vec_x && r0 >= 0 && r0 + REGION <= a.N;
#pragma unroll 1
            for (int q0 = 0; q0 < REGION / 4; q0 += NB * NT) {
                float4 v[NB];
                if (interior) {
#pragma unroll
                    for (int j = 0; j < NB; ++j)
                        v[j] = __ldcs(reinterpret_cast<const float4 *>(xr + r0) + q0 + tid + j * NT);
                } else {
#pragma unroll
                    for (int j = 0; j < NB; ++j) v[j] = load_region4(xr, r0 + 4 * (q0 + tid + j * NT), a.N, a.vec_x);
                }
#pragma unroll
                for (int j = 0; j < NB; ++j) {
                    if (a.pre_gain != 1.f) {
                        v[j].x *= a.pre_gain;
                        v[j].y *= a.pre_gain;
                        v[j].z *= a.pre_gain;
                        v[j].w *= a.pre_gain;
                    }
                    reg4[swz(q0 + tid + j * NT)] = v[j];
                }
            }
        }
        __syncthreads();

        if constexpr (S > 0) {
            float4 *my4 = reg4 + tid * CQ;
            const int sw = tid & 7;
            // ---- pass 1: zero-state end state of my chunk ----
            TS e[D];
#pragma unroll
            for (int i = 0; i < D; ++i) e[i] = TS(0);
#pragma unroll
            for (int j = 0; j < CQ; ++j) {
                const float4 v = my4[j ^ sw];
                const TS xs[4] = {TS(v.x), TS(v.y), TS(v.z), TS(v.w)};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
#pragma unroll
                    for (int i = 0; i < D; ++i) e[i] = fma(tb.K[4 * j + u][i], xs[u], e[i]);
                }
            }
            // ---- warp inclusive scan: incl_t = e_t + M incl_{t-1} ----
            TS incl[D];
#pragma unroll
            for (int i = 0; i < D; ++i) incl[i] = e[i];
#pragma unroll
            for (int st = 0; st < 5; ++st) {
                const int off = 1 << st;
                TS prev[D];
#pragma unroll
                for (int i = 0; i < D; ++i) prev[i] = shfl_up(incl[i], off);
                if (lane >= off) {
                    matvec_acc<D, TS>(incl, prev, [&](int i, int j) { return tb.P[st][i][j]; });
                }
            }
            TS excl[D];
#pragma unroll
            for (int i = 0; i < D; ++i) {
                const TS v = shfl_up(incl[i], 1);
                excl[i] = lane == 0 ? TS(0) : v;
            }
            if (lane == 31) {
#pragma unroll
                for (int i = 0; i < D; ++i) warp_incl[warp * D + i] = incl[i];
            }
            if (tid == tagg) {
#pragma unroll
                for (int i = 0; i < D; ++i) aggin_s[i] = incl[i];
            }
            __syncthreads();

            // ---- CTA combine + tile aggregate (thread 0) ----
            if (tid == 0) {
                TS cur[D];
#pragma unroll
                for (int i = 0; i < D; ++i) cur[i] = TS(0);
                for (int w = 0; w < NW; ++w) {
#pragma unroll
                    for (int i = 0; i < D; ++i) wc_s[w * D + i] = cur[i];
                    if (w + 1 < NW) {
                        TS nxt[D];
#pragma unroll
                        for (int i = 0; i < D; ++i) nxt[i] = warp_incl[w * D + i];
                        matvec_acc<D, TS>(nxt, cur, [&](int i, int j) { return tb.W[1][i][j]; });
#pragma unroll
                        for (int i = 0; i < D; ++i) cur[i] = nxt[i];
                    }
                }
                // agg = incl(tagg) + M^(lt+1) wc[wt]
                TS agg[D], wcv[D];
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    agg[i] = aggin_s[i];
                    wcv[i] = wc_s[wt_agg * D + i];
                }
                matvec_acc<D, TS>(agg, wcv, [&](int i, int j) { return gsm[(i * D + j) * 33 + lt_agg + 1]; });
#pragma unroll
                for (int i = 0; i < D; ++i) agg_s[i] = agg[i];
            }
            __syncthreads();

            // ---- deterministic blocked look-back (warp 0) ----
            // Tiles of a channel form blocks of 32. carry_k (state at this
            // tile's region start) = sum_{j=1..kb} MT^(j-1) agg_{k-j}
            //                        + MT^kb * P_{base-1},
            // with kb = k mod 32 and P_{base-1} the inclusive prefix published
            // by the last tile of the previous block. Lane j owns term j and
            // the terms are summed by a fixed butterfly, so the result never
            // depends on scheduling (bit-reproducible, like the reference's
            // thread-count invariance, engine.py:1-8).
            if (warp == 0) {
                TileRec<TS, D> *recs = reinterpret_cast<TileRec<TS, D> *>(a.recs);
                TileRec<TS, D> *mine = recs + tile;
                const TS *TP = tpsm;  // staged in shared memory: one L2 round trip less per look-back
                TS agg[D], carry[D];
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    agg[i] = agg_s[i];
                    carry[i] = TS(0);
                }
                const int kb = (int)(k & 31);
                const long long base = k - kb;
                if (lane == 0 && kb < 31) {
#pragma unroll
                    for (int i = 0; i < D; ++i) mine->agg[i] = agg[i];
                    __threadfence();
                    st_release(&mine->flag, (a.epoch << 2) | 1ull);
                }
                const TileRec<TS, D> *src = nullptr;
                int need = 0, pw = 0;
                if (lane >= 1 && lane <= kb) {
                    src = recs + ((k - lane) * a.C + c);
                    need = 1;
                    pw = lane - 1;
                } else if (lane == 0 && base > 0) {
                    src = recs + ((base - 1) * a.C + c);
                    need = 2;
                    pw = kb;
                }
                if (src) {
                    const unsigned long long want = (a.epoch << 2) | (unsigned long long)need;
                    unsigned long long f = ld_acquire(&src->flag);
                    int spins = 0;
                    while ((f >> 2) != a.epoch || (f & 3ull) < (unsigned long long)need || f < want) {
                        if (++spins > 4) __nanosleep(spins < 64 ? 32 : 256);
                        if ((spins & 0x3FFFFFF) == 0) __trap();  // watchdog: ~64M polls (> 15 s) without progress
                        f = ld_acquire(&src->flag);
                    }
                    const TS *sv = need == 2 ? src->incl : src->agg;
                    TS val[D];
#pragma unroll
                    for (int i = 0; i < D; ++i) val[i] = ldcg(sv + i);
                    const TS *Mj = TP + (size_t)pw * D * D;
                    matvec_acc<D, TS>(carry, val, [&](int i, int j) { return Mj[i * D + j]; });
                }
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    TS v = carry[i];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v += shfl_xor(v, o);
                    carry[i] = v;
                }
                // the last tile of a block publishes its inclusive prefix
                // P = MT carry + agg for the next block
                if (lane == 0) {
                    if (kb == 31) {
                        TS P[D];
#pragma unroll
                        for (int i = 0; i < D; ++i) P[i] = agg[i];
                        matvec_acc<D, TS>(P, carry, [&](int i, int j) { return tb.MT[i][j]; });
#pragma unroll
                        for (int i = 0; i < D; ++i) mine->incl[i] = P[i];
                        __threadfence();
                        st_release(&mine->flag, (a.epoch << 2) | 2ull);
                    }
                    // warp carries with the region carry-in: WC[w] = M^(32w) carry + wc[w]
                    for (int w = 0; w < NW; ++w) {
                        TS v[D];
#pragma unroll
                        for (int i = 0; i < D; ++i) v[i] = wc_s[w * D + i];
                        if (w == 0) {
#pragma unroll
                            for (int i = 0; i < D; ++i) v[i] += carry[i];
                        } else {
                            matvec_acc<D, TS>(v, carry, [&](int i, int j) { return tb.W[w < NW ? w : 0][i][j]; });
                        }
#pragma unroll
                        for (int i = 0; i < D; ++i) WC_s[w * D + i] = v[i];
                    }
                }
            }
            __syncthreads();

            // ---- my chunk's true carry-in: excl + M^lane WC[warp] ----
            TS stt[D];
            {
                TS wcv[D];
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    stt[i] = excl[i];
                    wcv[i] = WC_s[warp * D + i];
                }
                matvec_acc<D, TS>(stt, wcv, [&](int i, int j) { return gsm[(i * D + j) * 33 + lane]; });
            }

            // ---- pass 2: exact DF2T recurrence, in place ----
#pragma unroll 2
            for (int j = 0; j < CQ; ++j) {
                const float4 v = my4[j ^ sw];
                TS xs[4] = {TS(v.x), TS(v.y), TS(v.z), TS(v.w)};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    TS val = xs[u];
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        const TS b0 = tb.sos[s][0], b1 = tb.sos[s][1], b2 = tb.sos[s][2];
                        const TS a1 = tb.sos[s][3], a2 = tb.sos[s][4];
                        const TS w1 = stt[2 * s], w2 = stt[2 * s + 1];
                        const TS yv = fma(b0, val, w1);
                        stt[2 * s] = fma(-a1, yv, fma(b1, val, w2));
                        stt[2 * s + 1] = fma(-a2, yv, b2 * val);
                        val = yv;
                    }
                    xs[u] = val;
                }
                my4[j ^ sw] = make_float4(float(xs[0]), float(xs[1]), float(xs[2]), float(xs[3]));
            }
            __syncthreads();
        }

        if constexpr (FIR) {
            // ---- direct FIR over the region: outputs at region positions [H, REGION) ----
            const int ngroups = a.Lout / 8;
            for (int g = tid; g < ngroups; g += NT) {
                const int p = a.H + 8 * g;
                float acc[8];
#pragma unroll
                for (int r = 0; r < 8; ++r) acc[r] = 0.f;
                float buf[16];
                {
                    const float4 h0 = reg4[swz((p - 8) >> 2)], h1 = reg4[swz((p - 4) >> 2)];
                    const float4 c0 = reg4[swz(p >> 2)], c1 = reg4[swz((p + 4) >> 2)];
                    buf[0] = h0.x; buf[1] = h0.y; buf[2] = h0.z; buf[3] = h0.w;
                    buf[4] = h1.x; buf[5] = h1.y; buf[6] = h1.z; buf[7] = h1.w;
                    buf[8] = c0.x; buf[9] = c0.y; buf[10] = c0.z; buf[11] = c0.w;
                    buf[12] = c1.x; buf[13] = c1.y; buf[14] = c1.z; buf[15] = c1.w;
                }
                for (int kb = 0; kb < a.Tpad; kb += 8) {
                    const float4 t0 = *reinterpret_cast<const float4 *>(taps_s + kb);
                    const float4 t1 = *reinterpret_cast<const float4 *>(taps_s + kb + 4);
                    const float h[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) {
#pragma unroll
                        for (int r = 0; r < 8; ++r) acc[r] = fmaf(h[jj], buf[8 + r - jj], acc[r]);
                    }
                    if (kb + 8 < a.Tpad) {
#pragma unroll
                        for (int i = 0; i < 8; ++i) buf[8 + i] = buf[i];
                        const int q = p - kb - 16;
                        const float4 n0 = reg4[swz(q >> 2)], n1 = reg4[swz((q + 4) >> 2)];
                        buf[0] = n0.x; buf[1] = n0.y; buf[2] = n0.z; buf[3] = n0.w;
                        buf[4] = n1.x; buf[5] = n1.y; buf[6] = n1.z; buf[7] = n1.w;
                    }
                }
                const long long o = out0 + 8 * g;
                if (o < a.N) {
                    float4 v0 = make_float4(apply_post(acc[0], a), apply_post(acc[1], a), apply_post(acc[2], a),
                                            apply_post(acc[3], a));
                    float4 v1 = make_float4(apply_post(acc[4], a), apply_post(acc[5], a), apply_post(acc[6], a),
                                            apply_post(acc[7], a));
                    store4(yr, o, a.N, a.vec_y, v0);
                    store4(yr, o + 4, a.N, a.vec_y, v1);
                }
            }
        } else {
            // ---- copy-out (H == 0, Lout == REGION) ----
            for (int q4 = tid; q4 < REGION / 4; q4 += NT) {
                const long long o = out0 + 4 * q4;
                if (o >= a.N) break;
                float4 v = reg4[swz(q4)];
                v.x = apply_post(v.x, a);
                v.y = apply_post(v.y, a);
                v.z = apply_post(v.z, a);
                v.w = apply_post(v.w, a);
                store4(yr, o, a.N, a.vec_y, v);
            }
        }
    }
}

}  // namespace wpk
