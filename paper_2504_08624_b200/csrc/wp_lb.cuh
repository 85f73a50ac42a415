// Single-pass tensor-core chain for sm_100a: any run of LTI stages (pre-gain,
// IIR SOS cascade of up to 8 sections, FIR, post-gains) in ONE kernel that
// reads every input sample from HBM once and writes every output once.
//
// Replaces the reference's per-stage passes (_iir_channel, _kernels_jit.py:
// 14-32; _fir_channel, :51-62; Chain.apply's stage loop, chain.py:66-71).
//
// Formulation. A pass is one LTI system: the cascade in a
// per-section BALANCED state basis s (D = 2S states; s' = A s + B u, y = C s
// + d u after the similarity transform of each section's DF2T realization),
// impulse response h, FIR f, gain G. For tile rows m = 0..127 of 64 outputs
// (n = n0 + 64 m + p), window start w_m = n0 - H + 64 m, H >= taps - 1:
//
//   y[n] = sum_{k < H+64} g[p + H - k] x[w_m + k]   main GEMM (tcgen05 f16x3)
//        + sum_i E[p][i] s_{w_m}[i]                  state term (fp32, epilogue)
//   s_{w_{m+1}} = M s_{w_m} + e_m,  M = A^64,  e_m = sum_{j<64} Ke[j] x[w_m + j]
//   g = G (f * h),  E[p] = G sum_t f[t] C A^(H+p-t),  Ke[j] = A^(63-j) B
//
// e_m comes out of the SAME MMAs as the main GEMM: the first K atom's B
// operand carries 2 * DE extra columns (Ke hi / lo parts), so the e GEMM
// shares every A-operand read. In the balanced basis the scan, the
// carries and the state term are well conditioned and run in fp32 (the DF2T
// basis needs fp64 there: tools/balance_probe.py).
//
// Cross-tile state: deterministic blocked decoupled look-back. Tile (c, k)
// publishes its zero-carry aggregate; its carry-in is
//   c_k = sum_{l < j} MT^l agg(k-1-l) + MT^j incl(kb - 1),  kb = k & ~31, j = k - kb,
// MT = M^128, and tiles with k % 32 == 31 publish incl(k) = MT c_k + agg(k).
// The formula does not depend on timing, so results are bit-reproducible and
// independent of the channel count / sharding (time-major tile order: tile t
// = k * C + c; predecessors are processed concurrently by other SMs).
//
// Warp roles (persistent, one CTA per SM, static tile schedule):
//   warp 0       TMEM allocation; lane 0 issues the main GEMM (2 MMAs per K step)
//   warp 1       bulk-copy producer of the fp32 window, L2 prefetch ahead
//   warps 2-6    converters: fp32 window -> SW128 fp16 hi / lo (Hankel rows)
//   warp 7       look-back: carry-in c of each tile (the only role that waits
//                on other SMs), inclusive state of block-end tiles
//   warps 8-15   two row groups (even / odd local tiles), one TMEM lane per
//                thread: scan (e from TMEM, Kogge-Stone over rows, aggregate ->
//                global), then the epilogue once the carry is known:
//                s_m = L_m + M^m (Z_w + M^(32 w) c), TMEM -> (hi + lo) * scale
//                + E s_m -> coalesced stores
//
// Published states are 64-bit words {fp32 value, valid flag} written and
// polled with relaxed gpu-scope accesses (no fences, no L1 invalidation);
// the host zeroes them before every launch (graph-safe).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "wp_chain3.cuh"

namespace wpk {

constexpr int LB_THREADS = 512;
constexpr int LB_CONV = 160;   // converter threads (warps 2..6)
constexpr int LB_QMAX = 14;    // float4 of the window per converter thread (W <= 8960)
constexpr int LB_NA = 3;       // TMEM accumulator stages
constexpr int LB_NC = 4;       // carry ring (look-back warps -> epilogue)
constexpr int LB_MAX_H = 256;  // FIR halo limit (W <= 8448)
constexpr int LB_TRACE_EV = 12;
constexpr int LB_BLK = 32;     // look-back block (tiles of one channel)

struct LbArgs {
    const float *x;
    float *y;
    long long C, N, ldx, ldy;
    long long total_tiles;
    int H, K, W;
    const unsigned char *Bimg;  // SW128 K-major fp16: atom 0 [g_hi | g_lo | Ke_hi | Ke_lo], atoms >= 1 [g_hi | g_lo]
    const float *stabs;         // tables copied to shared memory (LbTabs layout)
    const float *MTl;           // [D * D][32] lane-minor: (M^128)^l, l < 32; then [D][D] M^128
    float out_scale;            // 2^-fB of the g image
    float escale[16];           // 2^-fK_i of the Ke columns
    unsigned long long *aggw;   // [tiles][D] {value, 1}: zero-carry tile aggregates (zeroed before the launch)
    unsigned long long *inclw;  // [blocks][C][D] {value, 1}: state after block-end tiles (k % 32 == 31)
    int vec_x, vec_y;
    unsigned long long *trace;  // optional: [tiles][LB_TRACE_EV] globaltimer stamps
};

// ---- table layout shared by host and device (floats) ----
// Es[64][D] | Mp[7][LT] (M^(2^b)) | Wt[4][LT] (M^(32 w)) | Gl[LT][32] (M^l, lane-minor; D <= 8 only)
__host__ __device__ constexpr int lb_de(int D) { return D <= 8 ? 8 : 16; }
__host__ __device__ constexpr int lb_ns(int D) { return 128 + 2 * lb_de(D); }  // TMEM columns per stage
__host__ __device__ constexpr int lb_has_gl(int D) { return D <= 8; }
__host__ __device__ constexpr int lb_tab_floats(int D) {
    return 64 * D + 11 * lt_size(D) + (lb_has_gl(D) ? 32 * lt_size(D) : 0);
}
__host__ __device__ constexpr int lb_off_mp(int D) { return 64 * D; }
__host__ __device__ constexpr int lb_off_wt(int D) { return 64 * D + 7 * lt_size(D); }
__host__ __device__ constexpr int lb_off_gl(int D) { return 64 * D + 11 * lt_size(D); }

struct LbLayout {
    uint32_t opBytes, b0Bytes, bBytes;
    uint32_t bimg, op, raw, tabs, sbuf, stg, misc, bars;
    uint32_t total;
    __host__ __device__ LbLayout(int W, int K, int D, int nop) {
        opBytes = ((uint32_t)W * 2u + 1023u) & ~1023u;
        b0Bytes = (uint32_t)lb_ns(D) * 128u;                       // atom 0: NS rows of 128 B
        bBytes = b0Bytes + (uint32_t)((K + 63) / 64 - 1) * 16384u;  // atoms >= 1: 128 rows
        bimg = 0;
        op = bimg + bBytes;
        raw = op + 2u * (uint32_t)nop * opBytes;
        const uint32_t rawBytes = ((uint32_t)W * 4u + 1023u) & ~1023u;
        tabs = raw + rawBytes;
        sbuf = (tabs + 4u * (uint32_t)lb_tab_floats(D) + 15u) & ~15u;
        stg = sbuf;  // (no per-row buffers: scan and epilogue of a tile run in the same threads)
        misc = stg + 8u * 32u * CT_STG_PITCH;
        // misc: Tw[2][4][D], zb[NA][4][D], cb[NC][D] f32; scl[8] f32, red[8] f32, stag[8] i32
        bars = (misc + 4u * (uint32_t)((8 + 4 * LB_NA + LB_NC) * D) + 96u + 15u) & ~15u;
        total = bars + 32 * 8 + 16 + 1024;  // + alignment slack
    }
};

namespace lbd {

__device__ __forceinline__ unsigned long long ld_word(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_word(unsigned long long *p, float v) {
    const unsigned long long w = (1ull << 32) | (unsigned long long)__float_as_uint(v);
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}

// out += M v, M block lower triangular (2x2 blocks) stored compactly (lt_off)
template <int D>
__device__ __forceinline__ void lt_mv(float (&out)[D], const float *m, const float (&v)[D]) {
#pragma unroll
    for (int r = 0; r < D; ++r) {
        float acc = out[r];
#pragma unroll
        for (int q = 0; q < lt_nj(r); ++q) acc = fmaf(m[lt_off(r) + q], v[q], acc);
        out[r] = acc;
    }
}

// D published words at once (one round trip when they are valid), re-polled
// with back-off until every word is valid
template <int D>
__device__ __forceinline__ void wait_words(const unsigned long long *p, float (&v)[D]) {
    unsigned long long w[D];
    const unsigned long long t0 = ctd::gtimer();
    unsigned ns = 32;
    for (;;) {
#pragma unroll
        for (int d = 0; d < D; ++d) w[d] = ld_word(p + d);
        bool ok = true;
#pragma unroll
        for (int d = 0; d < D; ++d) ok = ok && (w[d] >> 32) != 0;
        if (ok) break;
        __nanosleep(ns);
        ns = ns < 256 ? 2 * ns : 256;
        if (ctd::gtimer() - t0 > 10000000000ull) __trap();
    }
#pragma unroll
    for (int d = 0; d < D; ++d) v[d] = __uint_as_float((unsigned)w[d]);
}

// value of a published word, waiting until it is valid (back-off, watchdog)
__device__ __forceinline__ float wait_word(const unsigned long long *p) {
    unsigned long long w = ld_word(p);
    if (w >> 32) return __uint_as_float((unsigned)w);
    const unsigned long long t0 = ctd::gtimer();
    unsigned ns = 32;
    while (!((w = ld_word(p)) >> 32)) {
        __nanosleep(ns);
        ns = ns < 256 ? 2 * ns : 256;
        if (ctd::gtimer() - t0 > 10000000000ull) __trap();
    }
    return __uint_as_float((unsigned)w);
}

}  // namespace lbd

template <int D, int NOP>
__global__ void __launch_bounds__(LB_THREADS, 1) chain_lb_kernel(const LbArgs a) {
    static_assert(D >= 2 && D <= 16 && (D % 2) == 0, "2..8 sections");
    static_assert(NOP == 2 || NOP == 3, "two or three fp16 operand stages");
    constexpr int DE = lb_de(D);
    constexpr int NS = lb_ns(D);
    constexpr int LT = lt_size(D);
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024u - (wptc::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nk = a.K / 16;
    const LbLayout lay(a.W, a.K, D, NOP);
    unsigned char *bimg = smem + lay.bimg;
    unsigned char *op = smem + lay.op;
    float *tabs = reinterpret_cast<float *>(smem + lay.tabs);
    const float *Es = tabs;
    const float *Mp = tabs + lb_off_mp(D);
    const float *Wt = tabs + lb_off_wt(D);
    const float *Gl = tabs + lb_off_gl(D);
    float *sbuf = reinterpret_cast<float *>(smem + lay.sbuf);  // [NA][128][D]: zero-carry row prefixes L_m
    unsigned char *stg = smem + lay.stg;
    float *Tw = reinterpret_cast<float *>(smem + lay.misc);  // [2][4][D] warp totals
    float *zb = Tw + 8 * D;                                  // [NA][4][D] warp starts Z_w
    float *cb = zb + 4 * LB_NA * D;                          // [NC][D] carry-in ring
    float *scl = cb + LB_NC * D;                             // [8] ring by local tile
    float *red = scl + 8;                                    // [8]
    int *stag = reinterpret_cast<int *>(red + 8);            // [8] local tile index of scl[]
    unsigned long long *bars = reinterpret_cast<unsigned long long *>(smem + lay.bars);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 32);
    static_assert(LB_NA == 3, "barrier map");
    const uint32_t bar0 = wptc::smem_u32(bars);
#define LBTR(tile, ev)                                                                \
    do {                                                                              \
        if (a.trace) a.trace[(long long)(tile) * LB_TRACE_EV + (ev)] = ctd::gtimer(); \
    } while (0)
    // barriers: OP_FULL / OP_EMPTY x 3, ACC_FULL / ACC_EMPTY / L_READY / C_READY x 3, RAW full / empty
#define OPF(s) (bar0 + 8u * (uint32_t)(0 + (s)))
#define OPE(s) (bar0 + 8u * (uint32_t)(3 + (s)))
#define ACF(s) (bar0 + 8u * (uint32_t)(6 + (s)))
#define ACE(s) (bar0 + 8u * (uint32_t)(9 + (s)))
#define SRD(s) (bar0 + 8u * (uint32_t)(12 + (s)))
#define CRD(s) (bar0 + 8u * (uint32_t)(15 + (s)))
#define CEM(s) (bar0 + 8u * (uint32_t)(19 + (s)))
#define RWF (bar0 + 8u * 23u)
#define RWE (bar0 + 8u * 24u)

    if (warp == 0) wptc::tmem_alloc(wptc::smem_u32(tmem_slot), 512);
    if (tid == 32) {
        for (int s = 0; s < NOP; ++s) {
            wptc::mbar_init(OPF(s), 1);
            wptc::mbar_init(OPE(s), 1);
        }
        for (int s = 0; s < LB_NA; ++s) {
            wptc::mbar_init(ACF(s), 1);
            wptc::mbar_init(ACE(s), CT_ROWS);
            wptc::mbar_init(SRD(s), CT_ROWS);
        }
        for (int s = 0; s < LB_NC; ++s) {
            wptc::mbar_init(CRD(s), 1);
            wptc::mbar_init(CEM(s), CT_ROWS);
        }
        wptc::mbar_init(RWF, 1);
        wptc::mbar_init(RWE, 1);
        wptc::mbar_fence_init();
    }
    for (int i = tid; i < (int)(lay.bBytes / 16); i += LB_THREADS)
        reinterpret_cast<uint4 *>(bimg)[i] = reinterpret_cast<const uint4 *>(a.Bimg)[i];
    for (int i = tid; i < lb_tab_floats(D); i += LB_THREADS) tabs[i] = a.stabs[i];
    if (tid < 8) stag[tid] = -1;
    wptc::fence_proxy_async_smem();
    wptc::fence_before_sync();
    __syncthreads();
    wptc::fence_after_sync();
    const uint32_t tmem = *tmem_slot;
    const long long first = blockIdx.x, stride = gridDim.x;
    const int ntiles = first < a.total_tiles ? (int)((a.total_tiles - 1 - first) / stride + 1) : 0;

    if (warp == 0) {
        // ================= MMA issuer =================
        if (lane == 0) {
            const uint32_t id_e = wptc::idesc_f16(128, NS);    // first K atom: g_hi | g_lo | Ke_hi | Ke_lo
            const uint32_t id_hl = wptc::idesc_f16(128, 128);  // x_hi [g_hi | g_lo]
            const uint32_t id_h = wptc::idesc_f16(128, 64);    // x_lo g_hi
            const uint32_t op0 = wptc::smem_u32(op), b0 = wptc::smem_u32(bimg);
            for (int i = 0; i < ntiles; ++i) {
                const int so = i % NOP;
                const uint32_t paro = (uint32_t)((i / NOP) & 1);
                const int sa = i % LB_NA;
                const uint32_t para = (uint32_t)((i / LB_NA) & 1);
                wptc::mbar_wait(OPF(so), paro);
                wptc::mbar_wait(ACE(sa), para ^ 1u);
                wptc::fence_after_sync();
                LBTR(first + (long long)i * stride, 2);
                const uint32_t dm = tmem + (uint32_t)NS * sa;
                const uint32_t ahi = op0 + (2u * so) * lay.opBytes, alo = ahi + lay.opBytes;
                const uint64_t ah0 = ctd::desc_sw128(ahi), al0 = ctd::desc_sw128(alo);
#pragma unroll 1
                for (int kk = 0; kk < nk; ++kk) {
                    const uint64_t ka = 2u * kk;  // +32 B per K step, across rows (Hankel)
                    if (kk < 4) {
                        // x_hi and x_lo against [g_hi | g_lo | Ke_hi | Ke_lo]; the x_lo g_lo
                        // (and x_lo Ke_lo) terms it adds are part of the exact product
                        const uint64_t bb = ctd::desc_sw128(b0 + 32u * kk);
                        wptc::mma_f16(dm, ah0 + ka, bb, id_e, kk > 0);
                        wptc::mma_f16(dm, al0 + ka, bb, id_e, 1u);
                    } else {
                        const uint64_t bb = ctd::desc_sw128(b0 + lay.b0Bytes + 16384u * ((kk >> 2) - 1) + 32u * (kk & 3));
                        wptc::mma_f16(dm, ah0 + ka, bb, id_hl, 1u);
                        wptc::mma_f16(dm, al0 + ka, bb, id_h, 1u);
                    }
                }
                wptc::mma_commit(OPE(so));
                wptc::mma_commit(ACF(sa));
                LBTR(first + (long long)i * stride, 3);
            }
        }
    } else if (warp == 1) {
        // ================= bulk-copy producer: fp32 window -> smem =================
        if (lane == 0) {
            const uint32_t raw0 = wptc::smem_u32(smem + lay.raw);
            for (int i = 0; i < ntiles; ++i) {
                wptc::mbar_wait(RWE, (uint32_t)(i & 1) ^ 1u);
                const c3d::Win g = c3d::win(first + (long long)i * stride, a.C, a.N, a.H, a.W, a.vec_x);
                const uint32_t bytes = (uint32_t)(4 * (g.hi - g.lo));
                if (bytes > 0) {
                    c3d::arrive_tx(RWF, bytes);
                    const float *src = a.x + g.c * a.ldx + g.lo;
                    const uint32_t dst = raw0 + 4u * (uint32_t)(g.lo - g.start);
                    for (uint32_t o = 0; o < bytes; o += 16384u) {
                        const uint32_t nb = bytes - o < 16384u ? bytes - o : 16384u;
                        c3d::bulk_g2s(dst + o, reinterpret_cast<const unsigned char *>(src) + o, nb, RWF);
                    }
                } else {
                    ctd::arrive(RWF);
                }
                const long long nt = first + (long long)(i + 2) * stride;
                if (i + 2 < ntiles) {
                    const c3d::Win g2 = c3d::win(nt, a.C, a.N, a.H, a.W, a.vec_x);
                    const uint32_t b2 = (uint32_t)(4 * (g2.hi - g2.lo));
                    if (b2 > 0) ctd::prefetch_l2(a.x + g2.c * a.ldx + g2.lo, b2);
                }
            }
        }
    } else if (warp >= 2 && warp < 2 + LB_CONV / 32) {
        // ================= converters: fp32 window -> SW128 fp16 hi / lo =================
        const int ct = tid - 64;
        const int cw = ct >> 5;
        const int nq = a.W / 4;
        const float4 *raw4 = reinterpret_cast<const float4 *>(smem + lay.raw);
        for (int i = 0; i < ntiles; ++i) {
            const int s = i % NOP;
            const uint32_t par = (uint32_t)((i / NOP) & 1);
            const c3d::Win g = c3d::win(first + (long long)i * stride, a.C, a.N, a.H, a.W, a.vec_x);
            const float *xr = a.x + g.c * a.ldx;
            const bool interior = g.start >= g.lo && g.start + a.W <= g.hi;
            wptc::mbar_wait(RWF, (uint32_t)(i & 1));
            if (ct == 0) LBTR(first + (long long)i * stride, 0);
            float4 v[LB_QMAX];
            float m = 0.f;
            if (interior) {
#pragma unroll
                for (int j = 0; j < LB_QMAX; ++j)
                    v[j] = (ct + j * LB_CONV < nq) ? raw4[ct + j * LB_CONV] : make_float4(0.f, 0.f, 0.f, 0.f);
            } else {
#pragma unroll 1
                for (int j = 0; j < LB_QMAX; ++j) {
                    const int q = ct + j * LB_CONV;
                    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (q < nq) {
                        const long long p0 = g.start + 4LL * q;
                        if (p0 >= g.lo && p0 + 4 <= g.hi) {
                            t = raw4[q];
                        } else {
                            t.x = (p0 + 0 >= 0 && p0 + 0 < a.N) ? __ldg(xr + p0 + 0) : 0.f;
                            t.y = (p0 + 1 >= 0 && p0 + 1 < a.N) ? __ldg(xr + p0 + 1) : 0.f;
                            t.z = (p0 + 2 >= 0 && p0 + 2 < a.N) ? __ldg(xr + p0 + 2) : 0.f;
                            t.w = (p0 + 3 >= 0 && p0 + 3 < a.N) ? __ldg(xr + p0 + 3) : 0.f;
                        }
                    }
#pragma unroll
                    for (int jj = 0; jj < LB_QMAX; ++jj)
                        if (jj == j) v[jj] = t;
                }
            }
#pragma unroll
            for (int j = 0; j < LB_QMAX; ++j)
                m = fmaxf(m, fmaxf(fmaxf(fabsf(v[j].x), fabsf(v[j].y)), fmaxf(fabsf(v[j].z), fabsf(v[j].w))));
            const unsigned mb = __reduce_max_sync(0xffffffffu, __float_as_uint(m));
            if (lane == 0) red[cw] = __uint_as_float(mb);
            ctd::named_sync(1, LB_CONV);
            if (ct == 0) ctd::arrive(RWE);  // the window is in registers: free it
            float tmax = red[0];
#pragma unroll
            for (int w = 1; w < LB_CONV / 32; ++w) tmax = fmaxf(tmax, red[w]);
            int ex = 0;
            if (tmax > 0.f) frexpf(tmax, &ex);
            const float sc = ldexpf(1.f, tmax > 0.f ? 14 - ex : 0);
            wptc::mbar_wait(OPE(s), par ^ 1u);
            unsigned char *ohi = op + (2 * s) * lay.opBytes, *olo = ohi + lay.opBytes;
#pragma unroll
            for (int j = 0; j < LB_QMAX; ++j) {
                const int q = ct + j * LB_CONV;
                if (q < nq) {
                    const float2 f01 = make_float2(v[j].x * sc, v[j].y * sc);
                    const float2 f23 = make_float2(v[j].z * sc, v[j].w * sc);
                    const __half2 h01 = __float22half2_rn(f01), h23 = __float22half2_rn(f23);
                    const float2 b01 = __half22float2(h01), b23 = __half22float2(h23);
                    const __half2 l01 = __floats2half2_rn(f01.x - b01.x, f01.y - b01.y);
                    const __half2 l23 = __floats2half2_rn(f23.x - b23.x, f23.y - b23.y);
                    uint2 hv, lv;
                    hv.x = *reinterpret_cast<const uint32_t *>(&h01);
                    hv.y = *reinterpret_cast<const uint32_t *>(&h23);
                    lv.x = *reinterpret_cast<const uint32_t *>(&l01);
                    lv.y = *reinterpret_cast<const uint32_t *>(&l23);
                    const uint32_t off = ctd::swz128(8u * (uint32_t)q);
                    *reinterpret_cast<uint2 *>(ohi + off) = hv;
                    *reinterpret_cast<uint2 *>(olo + off) = lv;
                }
            }
            if (ct == 0) {
                scl[i & 7] = sc;
                __threadfence_block();
                *reinterpret_cast<volatile int *>(stag + (i & 7)) = i;
            }
            wptc::fence_proxy_async_smem();
            ctd::named_sync(2, LB_CONV);
            if (ct == 0) {
                ctd::arrive(OPF(s));
                LBTR(first + (long long)i * stride, 1);
            }
        }
    } else if (warp == 7) {
        // ================= look-back: carry-in of each tile =================
        for (int i = 0; i < ntiles; ++i) {
            const int sc4 = i % LB_NC;
            const long long tile = first + (long long)i * stride;
            const long long c = (long long)((unsigned long long)tile % (unsigned long long)a.C);
            const long long k = (long long)((unsigned long long)tile / (unsigned long long)a.C);
            wptc::mbar_wait(CEM(sc4), (uint32_t)((i / LB_NC) & 1) ^ 1u);  // cb slot read by the epilogue
            if (lane == 0) LBTR(tile, 4);
            // c_k = sum_{l < j} MT^l agg(k-1-l) + MT^j incl(kb - 1)
            const long long kb = k & ~(long long)(LB_BLK - 1);
            const int j = (int)(k - kb);
            float w[D];
#pragma unroll
            for (int d = 0; d < D; ++d) w[d] = 0.f;
            // predecessors publish roughly in tile order: the nearest one first
            if (lane == 0 && j > 0) (void)lbd::wait_word(a.aggw + ((k - 1) * a.C + c) * D + (D - 1));
            __syncwarp();
            if (lane < j || (lane == j && kb > 0)) {
                const unsigned long long *src = lane < j ? a.aggw + ((k - 1 - lane) * a.C + c) * D
                                                         : a.inclw + ((kb / LB_BLK - 1) * a.C + c) * D;
                float v[D];
                lbd::wait_words<D>(src, v);
#pragma unroll
                for (int r = 0; r < D; ++r) {
                    float acc = 0.f;
#pragma unroll
                    for (int q = 0; q < D; ++q) acc = fmaf(__ldg(a.MTl + (r * D + q) * 32 + lane), v[q], acc);
                    w[r] = acc;
                }
            }
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
                for (int d = 0; d < D; ++d) w[d] += __shfl_xor_sync(0xffffffffu, w[d], off);
            if (lane == 0) {
#pragma unroll
                for (int d = 0; d < D; ++d) cb[sc4 * D + d] = w[d];
                ctd::arrive(CRD(sc4));
                LBTR(tile, 5);
            }
            if ((k & (LB_BLK - 1)) == LB_BLK - 1 && lane == 0) {
                // block end: incl = MT c_k + agg(k) for the next block's tiles
                float inc[D];
                lbd::wait_words<D>(a.aggw + tile * D, inc);
                const float *m = a.MTl + (size_t)D * D * 32;
#pragma unroll
                for (int r = 0; r < D; ++r) {
                    float acc = inc[r];
#pragma unroll
                    for (int q = 0; q < D; ++q) acc = fmaf(__ldg(m + r * D + q), w[q], acc);
                    inc[r] = acc;
                }
                unsigned long long *dst = a.inclw + ((k / LB_BLK) * a.C + c) * D;
#pragma unroll
                for (int d = 0; d < D; ++d) lbd::st_word(dst + d, inc[d]);
            }
            __syncwarp();
        }
    } else {
        // ================= row groups (warps 8-11: even, 12-15: odd local tiles) =================
        // scan: e from TMEM -> Kogge-Stone over the rows -> zero-carry prefix L_m,
        // warp start Z_w, tile aggregate -> global; then, once the look-back has
        // the carry: s_m = L_m + M^m (Z_w + M^(32 w) c), TMEM main -> (hi + lo) *
        // scale + E s_m -> coalesced stores. Two groups interleave tiles so every
        // SM sub-partition has two warps of this work.
        const int grp = (warp - 8) >> 2;
        const int wq = warp & 3;
        const int row = 32 * wq + lane;
        const uint32_t trow = (uint32_t)(32 * wq) << 16;
        unsigned char *mystg = stg + (size_t)(grp * 4 + wq) * 32 * CT_STG_PITCH;
        float *Tg = Tw + grp * 4 * D;  // this group's warp totals
        for (int i = grp; i < ntiles; i += 2) {
            const int sa = i % LB_NA;
            const uint32_t para = (uint32_t)((i / LB_NA) & 1);
            const int sc4 = i % LB_NC;
            const long long tile = first + (long long)i * stride;
            const long long c = (long long)((unsigned long long)tile % (unsigned long long)a.C);
            const long long n0 = (long long)((unsigned long long)tile / (unsigned long long)a.C) * (long long)CT_TOUT;
            wptc::mbar_wait(ACF(sa), para);
            wptc::fence_after_sync();
            float ev[2 * DE];
            {
                const uint32_t te = tmem + (uint32_t)NS * sa + 128u + trow;
                float t16[16];
                ctd::tmem_ld16(te, t16);
#pragma unroll
                for (int j = 0; j < 16; ++j) ev[j] = t16[j];
                if constexpr (DE == 16) {
                    ctd::tmem_ld16(te + 16u, t16);
#pragma unroll
                    for (int j = 0; j < 16; ++j) ev[16 + j] = t16[j];
                }
                wptc::tmem_wait_ld();
            }
            for (int spins = 0; *reinterpret_cast<volatile int *>(stag + (i & 7)) != i; ++spins) {
                __nanosleep(32);
                if (spins > (1 << 28)) __trap();
            }
            __threadfence_block();
            const float sci = scl[i & 7];
            const float inv_sc = 1.f / sci;
            float P[D];
#pragma unroll
            for (int d = 0; d < D; ++d) P[d] = (ev[d] + ev[DE + d]) * (a.escale[d] * inv_sc);
            // inclusive prefix over the warp's 32 rows: P_r = sum_{j <= r} M^(r-j) e_j
#pragma unroll
            for (int b = 0; b < 5; ++b) {
                const int off = 1 << b;
                float prev[D];
#pragma unroll
                for (int d = 0; d < D; ++d) prev[d] = __shfl_up_sync(0xffffffffu, P[d], off);
                if (lane >= off) lbd::lt_mv<D>(P, Mp + b * LT, prev);
            }
            // exclusive: state entering the row from the warp start (zero carry)
            float s[D];
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const float u = __shfl_up_sync(0xffffffffu, P[d], 1);
                s[d] = lane == 0 ? 0.f : u;
            }
            if (lane == 31) {
#pragma unroll
                for (int d = 0; d < D; ++d) Tg[wq * D + d] = P[d];
            }
            ctd::named_sync(3 + grp, 128);
            // Z_w: state at the warp start (zero carry at the tile start)
            float V[D];
#pragma unroll
            for (int d = 0; d < D; ++d) V[d] = 0.f;
#pragma unroll 1
            for (int u = 0; u < wq; ++u) {
                float t[D];
#pragma unroll
                for (int d = 0; d < D; ++d) t[d] = Tg[u * D + d];
                lbd::lt_mv<D>(t, Mp + 5 * LT, V);
#pragma unroll
                for (int d = 0; d < D; ++d) V[d] = t[d];
            }
            if (wq == 3 && lane == 0) {
                // tile aggregate (state at the next tile's start, zero carry) -> global
                float agg[D];
#pragma unroll
                for (int d = 0; d < D; ++d) agg[d] = Tg[3 * D + d];
                lbd::lt_mv<D>(agg, Mp + 5 * LT, V);
#pragma unroll
                for (int d = 0; d < D; ++d) lbd::st_word(a.aggw + tile * D + d, agg[d]);
            }
            ctd::named_sync(3 + grp, 128);  // Tg is rewritten by the group's next tile
            if (row == 0) LBTR(tile, 6);
            wptc::mbar_wait(CRD(sc4), (uint32_t)((i / LB_NC) & 1));
            if (row == 0) LBTR(tile, 9);
            {
                // s_m = L_m + M^lane (Z_w + M^(32 w) c)
                float cin[D];
#pragma unroll
                for (int d = 0; d < D; ++d) cin[d] = cb[sc4 * D + d];
                ctd::arrive(CEM(sc4));
                lbd::lt_mv<D>(V, Wt + wq * LT, cin);
                if constexpr (lb_has_gl(D)) {
#pragma unroll
                    for (int r = 0; r < D; ++r) {
                        float acc = s[r];
#pragma unroll
                        for (int q = 0; q < lt_nj(r); ++q) acc = fmaf(Gl[(lt_off(r) + q) * 32 + lane], V[q], acc);
                        s[r] = acc;
                    }
                } else {
#pragma unroll
                    for (int b = 0; b < 5; ++b) {
                        float t[D];
#pragma unroll
                        for (int d = 0; d < D; ++d) t[d] = 0.f;
                        lbd::lt_mv<D>(t, Mp + b * LT, V);
                        if ((lane >> b) & 1) {
#pragma unroll
                            for (int d = 0; d < D; ++d) V[d] = t[d];
                        }
                    }
#pragma unroll
                    for (int d = 0; d < D; ++d) s[d] += V[d];
                }
            }
            if (row == 0) LBTR(tile, 10);
            const float osc = a.out_scale / sci;
            const uint32_t tbase = tmem + (uint32_t)NS * sa + trow;
            float *yr = a.y + c * a.ldy + n0;
            const long long tleft = a.N - n0;
            const bool full = a.vec_y && tleft >= CT_TOUT;
#pragma unroll 1
            for (int ch = 0; ch < 4; ++ch) {
                const int h = ch >> 1, hh = ch & 1;
                float t16[16], u16[16];
                ctd::tmem_ld16(tbase + 16u * ch, t16);
                ctd::tmem_ld16(tbase + 64u + 16u * ch, u16);
                wptc::tmem_wait_ld();
                if (ch == 3) {
                    wptc::fence_before_sync();
                    ctd::arrive(ACE(sa));
                }
                float o16[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const float *e = Es + (16 * ch + j) * D;
                    float acc = (t16[j] + u16[j]) * osc;
#pragma unroll
                    for (int d = 0; d < D; ++d) acc = fmaf(e[d], s[d], acc);
                    o16[j] = acc;
                }
                float4 *dst = reinterpret_cast<float4 *>(mystg + lane * CT_STG_PITCH + 64 * hh);
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4)
                    dst[q4] = make_float4(o16[4 * q4], o16[4 * q4 + 1], o16[4 * q4 + 2], o16[4 * q4 + 3]);
                if (hh == 1) {
                    __syncwarp();
                    if (full) {
#pragma unroll
                        for (int r = 0; r < 8; ++r) {
                            const int q = lane + 32 * r;
                            const int rr = q >> 3, c4 = q & 7;
                            const float4 v = *reinterpret_cast<const float4 *>(mystg + rr * CT_STG_PITCH + 16 * c4);
                            __stcs(reinterpret_cast<float4 *>(yr + 64 * (32 * wq + rr) + 32 * h + 4 * c4), v);
                        }
                    } else {
#pragma unroll 1
                        for (int r = 0; r < 8; ++r) {
                            const int q = lane + 32 * r;
                            const int rr = q >> 3, c4 = q & 7;
                            const float4 v = *reinterpret_cast<const float4 *>(mystg + rr * CT_STG_PITCH + 16 * c4);
                            const int oo = 64 * (32 * wq + rr) + 32 * h + 4 * c4;
                            const long long left = tleft - oo;
                            if (a.vec_y && left >= 4) {
                                __stcs(reinterpret_cast<float4 *>(yr + oo), v);
                            } else {
                                if (left > 0) yr[oo + 0] = v.x;
                                if (left > 1) yr[oo + 1] = v.y;
                                if (left > 2) yr[oo + 2] = v.z;
                                if (left > 3) yr[oo + 3] = v.w;
                            }
                        }
                    }
                    __syncwarp();
                }
            }
            if (row == 0) LBTR(tile, 7);
        }
    }
#undef LBTR
#undef OPF
#undef OPE
#undef ACF
#undef ACE
#undef SRD
#undef CRD
#undef CEM
#undef RWF
#undef RWE
    wptc::fence_before_sync();
    __syncthreads();
    wptc::fence_after_sync();
    if (warp == 0) wptc::tmem_dealloc(tmem, 512);
}

}  // namespace wpk
