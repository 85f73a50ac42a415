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
//   y[n] = sum_{k < H+64} g[p + H - k] x[w_m + k]   main GEMM (tcgen05, f16x3)
//        + sum_i E[p][i] s_{w_m}[i]                  state term (CUDA cores, fp32)
//   s_{w_{m+1}} = M s_{w_m} + e_m,  M = A^64,  e_m = sum_{j<64} Ke[j] x[w_m + j]
//   g = G (f * h),  E[p] = G sum_t f[t] C A^(H+p-t),  Ke[j] = A^(63-j) B
//
// f16x3: every product is x_hi g_hi + x_hi g_lo + x_lo g_hi (fp16 parts, fp32
// accumulation), issued as three MMAs into ONE accumulator of 64 columns
// (the lo parts concatenated along K: same A operand, second B image), so a
// TMEM stage is only 80 columns and six stages fit. e_m comes out of the SAME
// MMAs: the first K atom's B images carry the Ke columns (64..64+D), so the e
// GEMM shares every A-operand read. In the balanced basis the scan and the
// carries are well conditioned in fp32 (the DF2T basis needs fp64 there:
// tools/balance_probe.py). The state term E s (D FMAs per output, packed
// fma.rn.f32x2) is added by the epilogue threads in fp32 straight from the
// TMEM read: no second MMA round trip through the tensor pipe (where it would
// queue behind main GEMMs), so an accumulator stage is released as soon as
// the tile's carry is known. Measured against the f16x3 state GEMM issued
// between main-GEMM K steps: 0.583 vs 0.618 ms for cfg3.
//
// Cross-tile state: deterministic blocked decoupled look-back. Tile (c, k)
// publishes its zero-carry aggregate; its carry-in is
//   c_k = sum_{l < j} MT^l agg(k-1-l) + MT^j incl(kb - 1),  kb = k & ~31, j = k - kb,
// MT = M^128, and tiles with k % 32 == 31 publish incl(k) = MT c_k + agg(k).
// The formula does not depend on timing, so results are bit-reproducible and
// independent of the channel count / sharding (time-major tile order: tile t
// = k * C + c; predecessors are processed concurrently by other SMs).
// Published states are 64-bit words {fp32 value, valid flag} written and
// polled with relaxed gpu-scope accesses (no fences, no L1 invalidation); the
// host zeroes them before every launch (graph-safe).
//
// Warp roles (persistent, one CTA per SM, static tile schedule):
//   warp 0       TMEM allocation; lane 0 issues the main GEMM of every tile
//                (3 MMAs per K step) into a ring of six accumulator stages
//   warps 2-6    converters: fp32 window -> SW128 fp16 hi / lo (Hankel rows);
//                thread 0 bulk-copies the next fp32 window, L2 prefetch ahead
//   warps 1, 7   look-back (even / odd local tiles, so two tiles' polls are in
//                flight): carry-in c of each tile (the only role that waits on
//                other SMs), inclusive state of block-end tiles
//   warps 8-11   scan, one TMEM lane per thread: e from TMEM as soon as the
//                MMAs complete, Kogge-Stone over rows, aggregate -> global
//                (early, so other SMs' look-backs see it), row prefixes at
//                zero carry -> shared ring
//   warps 12-15  epilogue: once the carry is known s_m = L_m + M^m c, TMEM ->
//                scale + E s_m -> padded staging -> coalesced stores
#pragma once

#include <cuda.h>  // CUtensorMap
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "wp_common.cuh"

namespace wpk {

#ifndef LB_TMA_Y
#define LB_TMA_Y 1  // epilogue: full tiles leave through TMA tensor stores from swizzled staging
#endif
#ifndef LB_UB_NOES
#define LB_UB_NOES 0  // upper bound (wrong output): epilogue without the E s state term
#endif
#ifndef LB_GL_MAXD
#define LB_GL_MAXD 16  // lane-minor M^l table for every state size (8: only up to 4 sections)
#endif
constexpr int LB_THREADS = 512;
constexpr int LB_CONV = 160;   // converter threads (warps 2..6)
constexpr int LB_QMAX = 14;    // float4 of the window per converter thread (W <= 8960)
constexpr int LB_NA = 6;       // TMEM accumulator stages (80 columns each)
constexpr int LB_NS = 80;      // TMEM columns per stage: main [0, 64), e [64, 80)
constexpr int LB_NC = 4;       // carry ring (look-back warp -> epilogue)
constexpr int LB_NL = 4;       // row-prefix ring (scan -> epilogue)
constexpr int LB_RING = 16;    // tile-scale ring (converters -> scan)
constexpr int LB_MAX_H = 256;  // FIR halo limit (W <= 8448)
constexpr int LB_TRACE_EV = 16;
constexpr int LB_BLK = 32;     // look-back block (tiles of one channel)

struct LbArgs {
    const float *x;
    float *y;
    long long C, N, ldx, ldy;
    long long total_tiles;
    int H, K, W;
    const unsigned char *Bimg;   // SW128 K-major fp16 per K atom: [hi image | lo image], atom 0 with Ke rows
    const float *stabs;          // tables copied to shared memory (layout below)
    const float *MTl;            // [D * D][32] lane-minor: (M^128)^l, l < 32; then [D][D] M^128
    float out_scale;             // 2^-fB of the g image
    // warp-uniform tables read from the constant bank (kernel parameters), so they stay off
    // the shared-memory pipe that the MMA operand reads saturate:
    float4 Ep[256];              // [32][D / 2] E pairs (= tabs[0, 64 D))
    float Mpw[11 * 16 * 16];     // Mp[7][D][DP] | Wt[4][D][DP] (= tabs[64 D, 64 D + 11 D DP))
    float escale[16];            // 2^-fK_i of the Ke columns
    unsigned long long *aggw;    // [tiles][D] {value, 1}: zero-carry tile aggregates (zeroed before the launch)
    unsigned long long *inclw;   // [blocks][C][D] {value, 1}: state after block-end tiles (k % 32 == 31)
    int vec_x, vec_y;
    int tma_stage;  // the plan's layout has TMA staging (LbLayout tma)
    int tma_y;      // and the y tensor map is valid (aligned output, N >= 64): full tiles use TMA stores
    unsigned long long *trace;   // optional: [tiles][LB_TRACE_EV] globaltimer stamps
};

// ---- table layout shared by host and device (floats) ----
// Ep[32][D][2] (E[2q][d], E[2q+1][d] pairs) | Mp[7][D][DP] (M^(2^b)) | Wt[4][D][DP] (M^(32 w)) | Gl[LT][32] (M^l, lane-minor; D <= 8 only)
__host__ __device__ constexpr int lb_de(int D) { return D <= 8 ? 8 : 16; }
__host__ __device__ constexpr int lb_dp(int D) { return (D + 3) & ~3; }
__host__ __device__ constexpr int lb_has_gl(int D) { return D <= LB_GL_MAXD; }
__host__ __device__ constexpr int lb_tab_floats(int D, bool dense) {
    return 64 * D + 11 * D * lb_dp(D) + (lb_has_gl(D) ? 32 * lt_size(D, dense) : 0);
}
__host__ __device__ constexpr int lb_off_mp(int D) { return 64 * D; }
__host__ __device__ constexpr int lb_off_wt(int D) { return 64 * D + 7 * D * lb_dp(D); }
__host__ __device__ constexpr int lb_off_gl(int D) { return 64 * D + 11 * D * lb_dp(D); }
// main-GEMM B images: atom 0 has 80 rows (g, Ke, zero pad), atoms >= 1 64 rows; hi then lo image per atom
__host__ __device__ constexpr uint32_t lb_bhi(int a) { return a == 0 ? 0u : 20480u + (uint32_t)(a - 1) * 16384u; }
__host__ __device__ constexpr uint32_t lb_blo(int a) { return lb_bhi(a) + (a == 0 ? 10240u : 8192u); }
__host__ __device__ constexpr uint32_t lb_bbytes(int K) { return lb_bhi((K + 63) / 64); }

struct LbLayout {
    uint32_t opBytes, bBytes;
    uint32_t bimg, op, raw, tabs, ring, stg, misc, bars;
    uint32_t total;
    // tma: 8 KB of staging per epilogue warp (two 32 x 32 TMA boxes) instead of 32 padded
    // half rows; chosen per plan only where it still fits (fusion reach is unchanged)
    __host__ __device__ LbLayout(int W, int K, int D, int nop, bool tma, bool dense) {
        opBytes = ((uint32_t)W * 2u + 1023u) & ~1023u;
        bBytes = lb_bbytes(K);
        bimg = 0;
        op = bimg + bBytes;
        raw = op + 2u * (uint32_t)nop * opBytes;
        const uint32_t rawBytes = ((uint32_t)W * 4u + 1023u) & ~1023u;
        tabs = raw + rawBytes;
        ring = (tabs + 4u * (uint32_t)lb_tab_floats(D, dense) + 127u) & ~127u;  // [NL][D][128] row prefixes
        // [4 warps][32 rows] staging, 1024-aligned (TMA SWIZZLE_128B boxes: 2 x 4 KB per warp)
        stg = (ring + 4u * (uint32_t)(LB_NL * D * CT_ROWS) + 1023u) & ~1023u;
        misc = stg + (tma ? 4u * 8192u : 4u * 32u * CT_STG_PITCH);
        // misc: Tw[2][4][D], cb[NC][D] f32; scl[RING] f32, rsc[NL] f32, red[8] f32, stag[RING] i32
        bars = (misc + 4u * (uint32_t)((8 + LB_NC) * D) + 4u * (2 * LB_RING + LB_NL + 8) + 15u) & ~15u;
        total = bars + 48 * 8 + 16 + 1024;  // + alignment slack (35 barriers + TMEM slot)
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

// D published words at once (one round trip when they are valid), re-polled
// with back-off until every word is valid
template <int D>
__device__ __forceinline__ void wait_words(const unsigned long long *p, float (&v)[D]) {
    unsigned long long w[D];
    unsigned long long t0 = 0;
    unsigned ns = 32, it = 0;
    for (;;) {
#pragma unroll
        for (int d = 0; d < D; ++d) w[d] = ld_word(p + d);
        bool ok = true;
#pragma unroll
        for (int d = 0; d < D; ++d) ok = ok && (w[d] >> 32) != 0;
        if (ok) break;
        __nanosleep(ns);
        ns = ns < 128 ? 2 * ns : 128;
        if ((++it & 63u) == 0) {
            const unsigned long long t = ctd::gtimer();
            if (t0 == 0) t0 = t;
            else if (t - t0 > 10000000000ull) __trap();
        }
    }
#pragma unroll
    for (int d = 0; d < D; ++d) v[d] = __uint_as_float((unsigned)w[d]);
}

// wait until one published word is valid (back-off, watchdog)
__device__ __forceinline__ void wait_word(const unsigned long long *p) {
    if (ld_word(p) >> 32) return;
    const unsigned long long t0 = ctd::gtimer();
    unsigned ns = 32;
    while (!(ld_word(p) >> 32)) {
        __nanosleep(ns);
        ns = ns < 256 ? 2 * ns : 256;
        if (ctd::gtimer() - t0 > 10000000000ull) __trap();
    }
}

// out += M v for a block-lower-triangular M stored dense ([D][DP], 16-B
// aligned rows): row r needs columns < lt_nj(D, r, DN), read as float4
template <int D, bool DN>
__device__ __forceinline__ void lt_mv4(float (&out)[D], const float *m, const float (&v)[D]) {
    constexpr int DP = lb_dp(D);
#pragma unroll
    for (int r = 0; r < D; ++r) {
        float acc = out[r];
#pragma unroll
        for (int q4 = 0; q4 < (lt_nj(D, r, DN) + 3) / 4; ++q4) {
            const float4 mm = *reinterpret_cast<const float4 *>(m + r * DP + 4 * q4);
            acc = fmaf(mm.x, v[4 * q4], acc);
            if (4 * q4 + 1 < D) acc = fmaf(mm.y, v[(4 * q4 + 1) % D], acc);
            if (4 * q4 + 2 < D) acc = fmaf(mm.z, v[(4 * q4 + 2) % D], acc);
            if (4 * q4 + 3 < D) acc = fmaf(mm.w, v[(4 * q4 + 3) % D], acc);
        }
        out[r] = acc;
    }
}


// Wait for an mbarrier phase: non-blocking probes with a nanosleep back-off
// from 32 ns up to MAXNS, the watchdog clock read every 64 probes only. Every
// probe costs issue slots the working warps need (try_wait's suspend returns
// whenever any barrier of the CTA changes), so each role has ONE waiting
// thread and fans out through a named barrier (blocked in hardware).
template <unsigned MAXNS>
__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t parity) {
    if (wptc::mbar_test(bar, parity)) return;
    unsigned ns = 32, it = 0;
    unsigned long long t0 = 0;
    while (!wptc::mbar_test(bar, parity)) {
        __nanosleep(ns);
        ns = ns < MAXNS ? 2 * ns : MAXNS;
        if ((++it & 63u) == 0) {
            const unsigned long long t = ctd::gtimer();
            if (t0 == 0) t0 = t;
            else if (t - t0 > 10000000000ull) __trap();
        }
    }
}

// epilogue, last tile of a channel (out of line): staged half rows, stores guarded by the signal end
static __device__ __noinline__ void store_partial(const unsigned char *stg, float *yr, long long tleft, int vec_y,
                                                  int wq, int h, int lane) {
    for (int r = 0; r < 8; ++r) {
        const int q = lane + 32 * r;
        const int rr = q >> 3, c4 = q & 7;
        const float4 v = *reinterpret_cast<const float4 *>(stg + rr * CT_STG_PITCH + 16 * c4);
        const int oo = 64 * (32 * wq + rr) + 32 * h + 4 * c4;
        const long long left = tleft - oo;
        if (vec_y && left >= 4) {
            __stcs(reinterpret_cast<float4 *>(yr + oo), v);
        } else {
            if (left > 0) yr[oo + 0] = v.x;
            if (left > 1) yr[oo + 1] = v.y;
            if (left > 2) yr[oo + 2] = v.z;
            if (left > 3) yr[oo + 3] = v.w;
        }
    }
}

// (a0, a1) += (e0, e1) * s as one packed fp32x2 FMA (FFMA2)
__device__ __forceinline__ void ffma2(float &a0, float &a1, float e0, float e1, float s) {
    unsigned long long acc = (unsigned long long)__float_as_uint(a0) | ((unsigned long long)__float_as_uint(a1) << 32);
    const unsigned long long ev = (unsigned long long)__float_as_uint(e0) | ((unsigned long long)__float_as_uint(e1) << 32);
    const unsigned long long sv = (unsigned long long)__float_as_uint(s) | ((unsigned long long)__float_as_uint(s) << 32);
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(ev), "l"(sv));
    a0 = __uint_as_float((unsigned)acc);
    a1 = __uint_as_float((unsigned)(acc >> 32));
}

// s += M^lane V (M^l for l = lane < 32): lane-minor table Gl for D <= 8, else
// five conditional squarings-table steps (Mp[b] = M^(2^b))
template <int D, bool DN>
__device__ __forceinline__ void add_mlane(float (&s)[D], float (&V)[D], const float *Mp, const float *Gl, int lane) {
    constexpr int DP = lb_dp(D);
    if constexpr (lb_has_gl(D)) {
#pragma unroll
        for (int r = 0; r < D; ++r) {
            float acc = s[r];
#pragma unroll
            for (int q = 0; q < lt_nj(D, r, DN); ++q) acc = fmaf(Gl[(lt_off(D, r, DN) + q) * 32 + lane], V[q], acc);
            s[r] = acc;
        }
    } else {
#pragma unroll
        for (int b = 0; b < 5; ++b) {
            float t[D];
#pragma unroll
            for (int d = 0; d < D; ++d) t[d] = 0.f;
            lt_mv4<D, DN>(t, Mp + b * D * DP, V);
            if ((lane >> b) & 1) {
#pragma unroll
                for (int d = 0; d < D; ++d) V[d] = t[d];
            }
        }
#pragma unroll
        for (int d = 0; d < D; ++d) s[d] += V[d];
    }
}
// Warp reduce-scatter of D values (padded to a power of two DP): recursive halving
// over lane bits 4, 3, ... then an all-reduce over the remaining bits. Returns this
// lane's total for index idx (out); lanes whose remaining low bits are zero own it.
// DP + 5 - log2(DP) shuffles instead of 5 D for a butterfly all-reduce.
template <int D>
__device__ __forceinline__ float reduce_scatter(const float (&w)[D], int lane, int &idx, bool &owner) {
    constexpr int DP = D <= 2 ? 2 : D <= 4 ? 4 : D <= 8 ? 8 : 16;
    float cur[DP];
#pragma unroll
    for (int d = 0; d < DP; ++d) cur[d] = d < D ? w[d] : 0.f;
    int id = 0;
    int low = 0;  // lane bits reduced by all-reduce rounds
#pragma unroll
    for (int r = 0, off = 16, n = DP; r < 5; ++r, off >>= 1) {
        if (n > 1) {
            const int h = n / 2;
            const bool up = (lane & off) != 0;
#pragma unroll
            for (int k = 0; k < h; ++k) {
                const float send = up ? cur[k] : cur[k + h];
                const float keep = up ? cur[k + h] : cur[k];
                cur[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
            }
            id = 2 * id + (up ? 1 : 0);
            n = h;
        } else {
            cur[0] += __shfl_xor_sync(0xffffffffu, cur[0], off);
            low |= off;
        }
    }
    idx = id;
    owner = (lane & low) == 0 && id < D;
    return cur[0];
}

}  // namespace lbd

// DN: the plan's state basis is globally balanced (dense transfer matrices) instead of
// per-section balanced (block lower triangular) - chosen at plan time for cascades
// whose block basis is ill-conditioned in fp32
template <int D, int NOP, bool DN>
__global__ void __launch_bounds__(LB_THREADS, 1) chain_lb_kernel(const LbArgs a, const __grid_constant__ CUtensorMap ymap) {
    static_assert(D >= 2 && D <= 16 && (D % 2) == 0, "2..8 sections");
    static_assert(NOP == 2 || NOP == 3, "two or three fp16 operand stages");
    static_assert(LB_NA * LB_NS <= 512, "TMEM columns");
    static_assert(28 + 2 * LB_NL <= 48, "barrier slots");
    constexpr int DP = lb_dp(D);
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024u - (wptc::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nk = a.K / 16;
    const LbLayout lay(a.W, a.K, D, NOP, a.tma_stage != 0, DN);
    unsigned char *bimg = smem + lay.bimg;
    unsigned char *op = smem + lay.op;
    float *tabs = reinterpret_cast<float *>(smem + lay.tabs);
    const float *Mp = a.Mpw;
    const float *Wt = a.Mpw + 7 * D * DP;
    const float4 *Ep = reinterpret_cast<const float4 *>(tabs);  // [32][D / 2]: E pairs of two states
    const float *Gl = tabs + lb_off_gl(D);
    float *ring = reinterpret_cast<float *>(smem + lay.ring);  // [NL][D][128] row prefixes (zero carry)
    unsigned char *stg = smem + lay.stg;
    float *Tw = reinterpret_cast<float *>(smem + lay.misc);  // [2 parities][4][D] scan warp totals
    float *cb = Tw + 8 * D;                                  // [NC][D] carry-in ring
    float *scl = cb + LB_NC * D;                             // [RING] tile scales
    float *rsc = scl + LB_RING;                              // [NL] tile scales of the ring slots
    float *red = rsc + LB_NL;                                // [8]
    int *stag = reinterpret_cast<int *>(red + 8);            // [RING] local tile index of scl[]
    unsigned long long *bars = reinterpret_cast<unsigned long long *>(smem + lay.bars);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 48);
    const uint32_t bar0 = wptc::smem_u32(bars);
    // per-tile role stamps (tools/trace_lb.py) only in -DLB_TRACE builds: the checks and
    // stores cost 3 % (cfg3) to 10 % (cfg5) of the pass through the instruction cache
#ifdef LB_TRACE
#define LBTR(tile, ev)                                                                \
    do {                                                                              \
        if (a.trace) a.trace[(long long)(tile) * LB_TRACE_EV + (ev)] = ctd::gtimer(); \
    } while (0)
#else
#define LBTR(tile, ev) \
    do {               \
    } while (0)
#endif
    // barriers: OP_FULL / OP_EMPTY x 3; E_READY / ACC_EMPTY x 6; C_READY / C_EMPTY x 4;
    // RAW full; L_FULL / L_EMPTY x 4
#define OPF(s) (bar0 + 8u * (uint32_t)(0 + (s)))
#define OPE(s) (bar0 + 8u * (uint32_t)(3 + (s)))
#define EFL(s) (bar0 + 8u * (uint32_t)(6 + (s)))
#define ACE(s) (bar0 + 8u * (uint32_t)(12 + (s)))
#define CRD(s) (bar0 + 8u * (uint32_t)(18 + (s)))
#define CEM(s) (bar0 + 8u * (uint32_t)(22 + (s)))
#define RWF (bar0 + 8u * 26u)
#define LFL(s) (bar0 + 8u * (uint32_t)(28 + (s)))
#define LEM(s) (bar0 + 8u * (uint32_t)(28 + LB_NL + (s)))

    if (warp == 0) wptc::tmem_alloc(wptc::smem_u32(tmem_slot), 512);
    if (tid == 32) {
        for (int s = 0; s < NOP; ++s) {
            wptc::mbar_init(OPF(s), 1);
            wptc::mbar_init(OPE(s), 1);
        }
        for (int s = 0; s < LB_NA; ++s) {
            wptc::mbar_init(EFL(s), 1);
            wptc::mbar_init(ACE(s), CT_ROWS);

        }
        for (int s = 0; s < LB_NC; ++s) {
            wptc::mbar_init(CRD(s), 1);
            wptc::mbar_init(CEM(s), CT_ROWS);
        }
        for (int s = 0; s < LB_NL; ++s) {
            wptc::mbar_init(LFL(s), CT_ROWS);
            wptc::mbar_init(LEM(s), CT_ROWS);
        }
        wptc::mbar_init(RWF, 1);
        wptc::mbar_fence_init();
    }
    for (int i = tid; i < (int)(lay.bBytes / 16); i += LB_THREADS)
        reinterpret_cast<uint4 *>(bimg)[i] = reinterpret_cast<const uint4 *>(a.Bimg)[i];
    for (int i = tid; i < lb_tab_floats(D, DN); i += LB_THREADS) tabs[i] = a.stabs[i];
    if (tid < LB_RING) stag[tid] = -1;
    wptc::fence_proxy_async_smem();
    wptc::fence_before_sync();
    __syncthreads();
    wptc::fence_after_sync();
    const uint32_t tmem = *tmem_slot;
    const long long first = blockIdx.x, stride = gridDim.x;
    const int ntiles = first < a.total_tiles ? (int)((a.total_tiles - 1 - first) / stride + 1) : 0;

    if (warp == 0) {
        // ================= MMA issuer: the main GEMM of every tile, in tile order =================
        if (lane == 0) {
            const uint32_t id_e = wptc::idesc_f16(128, LB_NS);  // first K atom: [g | Ke | 0]
            const uint32_t id_g = wptc::idesc_f16(128, 64);     // other atoms
            const uint32_t op0 = wptc::smem_u32(op), b0 = wptc::smem_u32(bimg);
            for (int im = 0; im < ntiles; ++im) {
                const int so = im % NOP;
                const int sa = im % LB_NA;
                wptc::mbar_wait(OPF(so), (uint32_t)((im / NOP) & 1));
                wptc::mbar_wait(ACE(sa), (uint32_t)((im / LB_NA) & 1) ^ 1u);
                wptc::fence_after_sync();
                LBTR(first + (long long)im * stride, 2);
                const uint32_t dm = tmem + (uint32_t)LB_NS * sa;
                const uint32_t ahi = op0 + (2u * so) * lay.opBytes, alo = ahi + lay.opBytes;
                const uint64_t ah0 = ctd::desc_sw128(ahi), al0 = ctd::desc_sw128(alo);
#pragma unroll 1
                for (int kk = 0; kk < nk; ++kk) {
                    const uint64_t ka = 2u * kk;  // +32 B per K step, across rows (Hankel)
                    const int at = kk >> 2;
                    const uint32_t sub = 32u * (uint32_t)(kk & 3);
                    const uint64_t bh = ctd::desc_sw128(b0 + lb_bhi(at) + sub);
                    const uint64_t bl = ctd::desc_sw128(b0 + lb_blo(at) + sub);
                    const uint32_t id = at == 0 ? id_e : id_g;
                    wptc::mma_f16(dm, ah0 + ka, bh, id, kk > 0);  // x_hi g_hi
                    wptc::mma_f16(dm, ah0 + ka, bl, id, 1u);      // x_hi g_lo
                    wptc::mma_f16(dm, al0 + ka, bh, id, 1u);      // x_lo g_hi
                }
                wptc::mma_commit(OPE(so));
                wptc::mma_commit(EFL(sa));
                LBTR(first + (long long)im * stride, 3);
            }
        }
    } else if (warp >= 2 && warp < 2 + LB_CONV / 32) {
        // ================= converters: fp32 window -> SW128 fp16 hi / lo =================
        const int ct = tid - 64;
        const int cw = ct >> 5;
        const int nq = a.W / 4;
        const float4 *raw4 = reinterpret_cast<const float4 *>(smem + lay.raw);
        const uint32_t raw0 = wptc::smem_u32(smem + lay.raw);
        // thread 0 is also the bulk-copy producer of the (single) fp32 window buffer:
        // tile i + 1 is requested as soon as every converter holds tile i in registers
        auto issue_window = [&](int i) {
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
            if (i + 2 < ntiles) {
                const c3d::Win g2 = c3d::win(first + (long long)(i + 2) * stride, a.C, a.N, a.H, a.W, a.vec_x);
                const uint32_t b2 = (uint32_t)(4 * (g2.hi - g2.lo));
                if (b2 > 0) ctd::prefetch_l2(a.x + g2.c * a.ldx + g2.lo, b2);
            }
        };
        if (ct == 0 && ntiles > 0) issue_window(0);
        for (int i = 0; i < ntiles; ++i) {
            const int s = i % NOP;
            const uint32_t par = (uint32_t)((i / NOP) & 1);
            const c3d::Win g = c3d::win(first + (long long)i * stride, a.C, a.N, a.H, a.W, a.vec_x);
            wptc::mbar_wait_sleep<256>(RWF, (uint32_t)(i & 1));
            if (ct == 0) LBTR(first + (long long)i * stride, 0);
            if (!(g.start >= g.lo && g.start + a.W <= g.hi)) {
                c3d::fill_window(reinterpret_cast<float *>(smem + lay.raw), a.x + g.c * a.ldx, g.start, g.lo, g.hi, a.N,
                                 a.W, ct, LB_CONV);
                ctd::named_sync(1, LB_CONV);
            }
            float4 v[LB_QMAX];
            float m = 0.f;
#pragma unroll
            for (int j = 0; j < LB_QMAX; ++j)
                v[j] = (ct + j * LB_CONV < nq) ? raw4[ct + j * LB_CONV] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int j = 0; j < LB_QMAX; ++j)
                m = fmaxf(m, fmaxf(fmaxf(fabsf(v[j].x), fabsf(v[j].y)), fmaxf(fabsf(v[j].z), fabsf(v[j].w))));
            const unsigned mb = __reduce_max_sync(0xffffffffu, __float_as_uint(m));
            if (lane == 0) red[cw] = __uint_as_float(mb);
            ctd::named_sync(1, LB_CONV);
            if (ct == 0 && i + 1 < ntiles) issue_window(i + 1);  // the window is in registers: refill it
            float tmax = red[0];
#pragma unroll
            for (int w = 1; w < LB_CONV / 32; ++w) tmax = fmaxf(tmax, red[w]);
            int ex = 0;
            if (tmax > 0.f) frexpf(tmax, &ex);
            const float sc = ldexpf(1.f, tmax > 0.f ? 14 - ex : 0);
            wptc::mbar_wait_sleep<1024>(OPE(s), par ^ 1u);
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
                scl[i % LB_RING] = sc;
                __threadfence_block();
                *reinterpret_cast<volatile int *>(stag + (i % LB_RING)) = i;
            }
            wptc::fence_proxy_async_smem();
            ctd::named_sync(2, LB_CONV);
            if (ct == 0) {
                ctd::arrive(OPF(s));
                LBTR(first + (long long)i * stride, 1);
            }
        }
    } else if (warp == 1 || warp == 7) {
        // ================= look-back (warp 1: even, warp 7: odd local tiles): carry-in of each tile =================
        for (int i = warp == 1 ? 0 : 1; i < ntiles; i += 2) {
            const int sc4 = i % LB_NC;
            const long long tile = first + (long long)i * stride;
            const long long c = (long long)((unsigned)tile % (unsigned)a.C);  // tiles < 2^31 (host check)
            const long long k = (long long)((unsigned)tile / (unsigned)a.C);
            wptc::mbar_wait_sleep<512>(CEM(sc4), (uint32_t)((i / LB_NC) & 1) ^ 1u);  // slot read by the epilogue
            if (lane == 0) LBTR(tile, 4);
            // c_k = sum_{l < j} MT^l agg(k-1-l) + MT^j incl(kb - 1)
            const long long kb = k & ~(long long)(LB_BLK - 1);
            const int j = (int)(k - kb);
            float w[D];
#pragma unroll
            for (int d = 0; d < D; ++d) w[d] = 0.f;
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
            {
                int di;
                bool own;
                const float tot = lbd::reduce_scatter<D>(w, lane, di, own);
                if (own) cb[sc4 * D + di] = tot;
                __syncwarp();
            }
            if (lane == 0) {
                ctd::arrive(CRD(sc4));
                LBTR(tile, 5);
            }
            if ((k & (LB_BLK - 1)) == LB_BLK - 1 && lane == 0) {
#pragma unroll
                for (int d = 0; d < D; ++d) w[d] = cb[sc4 * D + d];
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
    } else if (warp < 12) {
        // ================= scan (warps 8-11): row prefixes at zero carry, tile aggregates =================
        const int wq = warp & 3;
        const int row = 32 * wq + lane;
        const uint32_t trow = (uint32_t)(32 * wq) << 16;
#pragma unroll 1
        for (int i = 0; i < ntiles; ++i) {
            const int sa = i % LB_NA;
            const long long tile = first + (long long)i * stride;
            const int sl = i % LB_NL;
            wptc::mbar_wait_sleep<128>(EFL(sa), (uint32_t)((i / LB_NA) & 1));
            for (int spins = 0; *reinterpret_cast<volatile int *>(stag + (i % LB_RING)) != i; ++spins) {
                __nanosleep(32);
                if (spins > (1 << 28)) __trap();
            }
            __threadfence_block();
            wptc::fence_after_sync();
            if (row == 0) LBTR(tile, 8);
            float ev[16];
            ctd::tmem_ld16(tmem + (uint32_t)LB_NS * sa + 64u + trow, ev);
            wptc::tmem_wait_ld();
            const float sci = scl[i % LB_RING];
            const float inv_sc = 1.f / sci;
            float P[D];
#pragma unroll
            for (int d = 0; d < D; ++d) P[d] = ev[d] * (a.escale[d] * inv_sc);
            // inclusive prefix over the warp's 32 rows: P_r = sum_{j <= r} M^(r-j) e_j
#pragma unroll 1
            for (int b = 0; b < 5; ++b) {
                const int off = 1 << b;
                float prev[D];
#pragma unroll
                for (int d = 0; d < D; ++d) prev[d] = __shfl_up_sync(0xffffffffu, P[d], off);
                if (lane >= off) lbd::lt_mv4<D, DN>(P, Mp + b * D * DP, prev);
            }
            // exclusive: state entering the row from the warp start (zero carry)
            float s[D];
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const float u = __shfl_up_sync(0xffffffffu, P[d], 1);
                s[d] = lane == 0 ? 0.f : u;
            }
            float *Tg = Tw + (i & 1) * 4 * D;  // double-buffered: one barrier per tile
            if (lane == 31) {
#pragma unroll
                for (int d = 0; d < D; ++d) Tg[wq * D + d] = P[d];
            }
            ctd::named_sync(3, 128);
            // Z_w: state at the warp start (zero carry at the tile start)
            float V[D];
#pragma unroll
            for (int d = 0; d < D; ++d) V[d] = 0.f;
#pragma unroll 1
            for (int u = 0; u < wq; ++u) {
                float t[D];
#pragma unroll
                for (int d = 0; d < D; ++d) t[d] = Tg[u * D + d];
                lbd::lt_mv4<D, DN>(t, Mp + 5 * D * DP, V);
#pragma unroll
                for (int d = 0; d < D; ++d) V[d] = t[d];
            }
            if (wq == 3 && lane == 0) {
                // tile aggregate (state at the next tile's start, zero carry) -> global
                float agg[D];
#pragma unroll
                for (int d = 0; d < D; ++d) agg[d] = Tg[3 * D + d];
                lbd::lt_mv4<D, DN>(agg, Mp + 5 * D * DP, V);
#pragma unroll
                for (int d = 0; d < D; ++d) lbd::st_word(a.aggw + tile * D + d, agg[d]);
            }
            // L_m = s + M^lane Z_w: the state entering row m at zero carry from the tile start
            lbd::add_mlane<D, DN>(s, V, Mp, Gl, lane);
            if (row == 0) LBTR(tile, 12);
            // only now (the aggregate is out) wait for the ring slot
            wptc::mbar_wait_sleep<256>(LEM(sl), (uint32_t)((i / LB_NL) & 1) ^ 1u);
#pragma unroll
            for (int d = 0; d < D; ++d) ring[(sl * D + d) * CT_ROWS + row] = s[d];
            if (row == 0) rsc[sl] = sci;
            ctd::arrive(LFL(sl));
            if (row == 0) LBTR(tile, 6);
        }
    } else {
        // ================= epilogue (warps 12-15) =================
        // s_m = L_m + M^m c, TMEM + E s_m -> y
        const int wq = warp & 3;
        const int row = 32 * wq + lane;
        const uint32_t trow = (uint32_t)(32 * wq) << 16;
        // each warp owns its staging (TMA: 8 KB, the padded half-row path reuses it)
        unsigned char *mystg = stg + (size_t)wq * (a.tma_stage ? 8192 : 32 * CT_STG_PITCH);
#pragma unroll 1
        for (int i = 0; i < ntiles; ++i) {
            const int sa = i % LB_NA, sl = i % LB_NL, sc4 = i % LB_NC;
            const long long tile = first + (long long)i * stride;
            const long long c = (long long)((unsigned)tile % (unsigned)a.C);
            const long long n0 = (long long)((unsigned)tile / (unsigned)a.C) * (long long)CT_TOUT;
            wptc::mbar_wait_sleep<128>(LFL(sl), (uint32_t)((i / LB_NL) & 1));
            wptc::mbar_wait_sleep<128>(CRD(sc4), (uint32_t)((i / LB_NC) & 1));
            float s[D];
#pragma unroll
            for (int d = 0; d < D; ++d) s[d] = ring[(sl * D + d) * CT_ROWS + row];
            const float sci = rsc[sl];
            ctd::arrive(LEM(sl));
            if (row == 0) LBTR(tile, 10);
            if (row == 0) LBTR(tile, 9);
            {
                // s_m = L_m + M^lane (M^(32 w) c)
                float cin[D], V[D];
#pragma unroll
                for (int d = 0; d < D; ++d) cin[d] = cb[sc4 * D + d], V[d] = 0.f;
                ctd::arrive(CEM(sc4));
                lbd::lt_mv4<D, DN>(V, Wt + wq * D * DP, cin);
                lbd::add_mlane<D, DN>(s, V, Mp, Gl, lane);
            }
            if (row == 0) LBTR(tile, 11);
            wptc::mbar_wait(EFL(sa), (uint32_t)((i / LB_NA) & 1));  // completed before the scan: ordering only
            wptc::fence_after_sync();
            const float osc = a.out_scale / sci;
            const uint32_t tbase = tmem + (uint32_t)LB_NS * sa + trow;
            float *yr = a.y + c * a.ldy + n0;
            const long long tleft = a.N - n0;
            const bool full = a.vec_y && tleft >= CT_TOUT;
#if LB_TMA_Y
            const bool tma = full && a.tma_y;
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // staging free again
            __syncwarp();
#endif
#pragma unroll 1
            for (int ch = 0; ch < 4; ++ch) {
                const int h = ch >> 1, hh = ch & 1;
                float o16[16];
                ctd::tmem_ld16(tbase + 16u * ch, o16);
                wptc::tmem_wait_ld();
                if (ch == 0 && row == 0) LBTR(tile, 13);
                if (ch == 3) {
                    wptc::fence_before_sync();
                    ctd::arrive(ACE(sa));  // the accumulator has been read: free it
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) o16[j] *= osc;
#pragma unroll
                for (int pp = 0; pp < (LB_UB_NOES ? 0 : 8); ++pp)
#pragma unroll
                    for (int d2 = 0; d2 < D / 2; ++d2) {
                        const float4 e = Ep[(8 * ch + pp) * (D / 2) + d2];
                        lbd::ffma2(o16[2 * pp], o16[2 * pp + 1], e.x, e.y, s[2 * d2]);
                        lbd::ffma2(o16[2 * pp], o16[2 * pp + 1], e.z, e.w, s[2 * d2 + 1]);
                    }
#if LB_TMA_Y
                if (tma) {
                    // this warp's 32 rows x columns [32 h, 32 h + 32) -> box h, in the 128-B swizzle
                    // the tensor map un-swizzles (conflict-free: 8 rows hit 8 different 16-B slots)
                    unsigned char *box = mystg + 4096 * h;
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        const int j = 4 * hh + q4;
                        *reinterpret_cast<float4 *>(box + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                            make_float4(o16[4 * q4], o16[4 * q4 + 1], o16[4 * q4 + 2], o16[4 * q4 + 3]);
                    }
                    if (ch == 3) {  // one proxy fence per tile, then both boxes
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        __syncwarp();
                        if (lane == 0) {
                            const int row0 = (int)(n0 >> 6) + 32 * wq;
#pragma unroll
                            for (int b = 0; b < 2; ++b)
                                asm volatile(
                                    "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                                        reinterpret_cast<uint64_t>(&ymap)),
                                    "r"(wptc::smem_u32(mystg + 4096 * b)), "r"(32 * b), "r"(row0), "r"((int)c)
                                    : "memory");
                            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                        }
                    }
                    continue;
                }
#endif
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
                        lbd::store_partial(mystg, yr, tleft, a.vec_y, wq, h, lane);
                    }
                    __syncwarp();
                }
            }
            if (row == 0) LBTR(tile, 7);
        }
#if LB_TMA_Y
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#endif
    }
#undef LBTR
#undef OPF
#undef OPE
#undef EFL
#undef ACE
#undef CRD
#undef CEM
#undef RWF
#undef LFL
#undef LEM
    wptc::fence_before_sync();
    __syncthreads();
    wptc::fence_after_sync();
    if (warp == 0) wptc::tmem_dealloc(tmem, 512);
}

}  // namespace wpk
