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
//        + sum_i E[p][i] s_{w_m}[i]                  state GEMM (tcgen05, f16x3)
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
// tools/balance_probe.py). The state term is one more f16x3 GEMM into the
// same accumulator: A = [s_hi | s_lo | s_hi] x (tile scale), B = [E_hi; E_hi;
// E_lo]. A row whose scaled state would overflow fp16 (a silent tile after a
// loud one) sends zeros to it and adds E s on the CUDA cores instead.
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
//   warp 0       TMEM allocation; lane 0 issues main(i) (3 MMAs per K step),
//                then state(i - LAG), so a tile's scan / look-back latency
//                overlaps the following tiles' main GEMMs
//   warp 1       bulk-copy producer of the fp32 window, L2 prefetch ahead
//   warps 2-6    converters: fp32 window -> SW128 fp16 hi / lo (Hankel rows)
//   warp 7       look-back: carry-in c of each tile (the only role that waits
//                on other SMs), inclusive state of block-end tiles
//   warps 8-15   two row groups (even / odd local tiles), one TMEM lane per
//                thread: scan (e from TMEM, Kogge-Stone over rows, aggregate ->
//                global); once the carry is known s_m = L_m + M^m (Z_w +
//                M^(32 w) c) -> state operand; after the state MMA the
//                epilogue: TMEM -> scale -> coalesced stores
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "wp_chain3.cuh"

namespace wpk {

constexpr int LB_THREADS = 512;
constexpr int LB_CONV = 160;   // converter threads (warps 2..6)
constexpr int LB_QMAX = 14;    // float4 of the window per converter thread (W <= 8960)
constexpr int LB_NA = 6;       // TMEM accumulator stages (80 columns each)
constexpr int LB_NS = 80;      // TMEM columns per stage: main [0, 64), e [64, 80)
constexpr int LB_LAG = 4;      // main(i) is issued before state(i - LB_LAG)
constexpr int LB_NC = 4;       // carry ring (look-back warp -> row groups)
constexpr int LB_RING = 16;    // tile-scale ring (converters -> row groups)
constexpr int LB_MAX_H = 256;  // FIR halo limit (W <= 8448)
constexpr int LB_TRACE_EV = 12;
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
    const unsigned char *Bsimg;  // [64 rows][KS] fp16, no-swizzle K-major: state-term B operand
    float st_mul;                // 2^(fB - fE): state operand = s * tile scale * st_mul
    float out_scale;             // 2^-fB of the g image
    float escale[16];            // 2^-fK_i of the Ke columns
    unsigned long long *aggw;    // [tiles][D] {value, 1}: zero-carry tile aggregates (zeroed before the launch)
    unsigned long long *inclw;   // [blocks][C][D] {value, 1}: state after block-end tiles (k % 32 == 31)
    int vec_x, vec_y;
    unsigned long long *trace;   // optional: [tiles][LB_TRACE_EV] globaltimer stamps
};

// ---- table layout shared by host and device (floats) ----
// Es[64][D] | Mp[7][D][DP] (M^(2^b)) | Wt[4][D][DP] (M^(32 w)) | Gl[LT][32] (M^l, lane-minor; D <= 8 only)
__host__ __device__ constexpr int lb_de(int D) { return D <= 8 ? 8 : 16; }
__host__ __device__ constexpr int lb_dp(int D) { return (D + 3) & ~3; }
__host__ __device__ constexpr int lb_has_gl(int D) { return D <= 8; }
__host__ __device__ constexpr int lb_tab_floats(int D) {
    return 64 * D + 11 * D * lb_dp(D) + (lb_has_gl(D) ? 32 * lt_size(D) : 0);
}
__host__ __device__ constexpr int lb_off_mp(int D) { return 64 * D; }
__host__ __device__ constexpr int lb_off_wt(int D) { return 64 * D + 7 * D * lb_dp(D); }
__host__ __device__ constexpr int lb_off_gl(int D) { return 64 * D + 11 * D * lb_dp(D); }
// main-GEMM B images: atom 0 has 80 rows (g, Ke, zero pad), atoms >= 1 64 rows; hi then lo image per atom
__host__ __device__ constexpr uint32_t lb_bhi(int a) { return a == 0 ? 0u : 20480u + (uint32_t)(a - 1) * 16384u; }
__host__ __device__ constexpr uint32_t lb_blo(int a) { return lb_bhi(a) + (a == 0 ? 10240u : 8192u); }
__host__ __device__ constexpr uint32_t lb_bbytes(int K) { return lb_bhi((K + 63) / 64); }
// state-term operands: K = 3 DE fp16 per row ([s_hi | s_lo | s_hi]), padded to 16; no-swizzle K-major
__host__ __device__ constexpr int lb_ks(int D) { return (3 * lb_de(D) + 15) / 16 * 16; }
__host__ __device__ constexpr uint32_t lb_sbo(int D) { return (uint32_t)lb_ks(D) / 8u * 128u; }
__host__ __device__ constexpr uint32_t lb_s_off(int D, int r, int k) {
    return (uint32_t)(r >> 3) * lb_sbo(D) + (uint32_t)(k >> 3) * 128u + (uint32_t)(r & 7) * 16u + (uint32_t)(k & 7) * 2u;
}

struct LbLayout {
    uint32_t opBytes, bBytes, sopBytes;
    uint32_t bimg, op, raw, tabs, sop, bs, stg, misc, bars;
    uint32_t total;
    __host__ __device__ LbLayout(int W, int K, int D, int nop) {
        opBytes = ((uint32_t)W * 2u + 1023u) & ~1023u;
        bBytes = lb_bbytes(K);
        sopBytes = 128u * (uint32_t)lb_ks(D) * 2u;
        bimg = 0;
        op = bimg + bBytes;
        raw = op + 2u * (uint32_t)nop * opBytes;
        const uint32_t rawBytes = ((uint32_t)W * 4u + 1023u) & ~1023u;
        tabs = raw + rawBytes;
        sop = (tabs + 4u * (uint32_t)lb_tab_floats(D) + 127u) & ~127u;  // [2 groups] state operands
        bs = sop + 2u * sopBytes;                                         // state-term B
        stg = bs + 64u * (uint32_t)lb_ks(D) * 2u;
        misc = stg + 8u * 32u * CT_STG_PITCH;
        // misc: Tw[2][4][D], cb[NC][D] f32; scl[RING] f32, red[8] f32, stag[RING] i32
        bars = (misc + 4u * (uint32_t)((8 + LB_NC) * D) + 4u * (2 * LB_RING + 8) + 15u) & ~15u;
        total = bars + 48 * 8 + 16 + 1024;  // + alignment slack (42 barriers + TMEM slot)
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
// aligned rows): row r needs columns < lt_nj(r), read as float4
template <int D>
__device__ __forceinline__ void lt_mv4(float (&out)[D], const float *m, const float (&v)[D]) {
    constexpr int DP = lb_dp(D);
#pragma unroll
    for (int r = 0; r < D; ++r) {
        float acc = out[r];
#pragma unroll
        for (int q4 = 0; q4 < (lt_nj(r) + 3) / 4; ++q4) {
            const float4 mm = *reinterpret_cast<const float4 *>(m + r * DP + 4 * q4);
            acc = fmaf(mm.x, v[4 * q4], acc);
            if (4 * q4 + 1 < D) acc = fmaf(mm.y, v[(4 * q4 + 1) % D], acc);
            if (4 * q4 + 2 < D) acc = fmaf(mm.z, v[(4 * q4 + 2) % D], acc);
            if (4 * q4 + 3 < D) acc = fmaf(mm.w, v[(4 * q4 + 3) % D], acc);
        }
        out[r] = acc;
    }
}

}  // namespace lbd

template <int D, int NOP>
__global__ void __launch_bounds__(LB_THREADS, 1) chain_lb_kernel(const LbArgs a) {
    static_assert(D >= 2 && D <= 16 && (D % 2) == 0, "2..8 sections");
    static_assert(NOP == 2 || NOP == 3, "two or three fp16 operand stages");
    static_assert(LB_NA * LB_NS <= 512, "TMEM columns");
    constexpr int DE = lb_de(D);
    constexpr int DP = lb_dp(D);
    constexpr int KS = lb_ks(D);
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
    unsigned char *sop = smem + lay.sop;  // [2 groups][128 rows][KS] fp16 state operands
    unsigned char *bsi = smem + lay.bs;   // [64 rows][KS] fp16 state-term B
    unsigned char *stg = smem + lay.stg;
    float *Tw = reinterpret_cast<float *>(smem + lay.misc);  // [2 groups][4][D] warp totals
    float *cb = Tw + 8 * D;                                  // [NC][D] carry-in ring
    float *scl = cb + LB_NC * D;                             // [RING] tile scales
    float *red = scl + LB_RING;                              // [8]
    int *stag = reinterpret_cast<int *>(red + 8);            // [RING] local tile index of scl[]
    unsigned long long *bars = reinterpret_cast<unsigned long long *>(smem + lay.bars);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 48);
    const uint32_t bar0 = wptc::smem_u32(bars);
#define LBTR(tile, ev)                                                                \
    do {                                                                              \
        if (a.trace) a.trace[(long long)(tile) * LB_TRACE_EV + (ev)] = ctd::gtimer(); \
    } while (0)
    // barriers: OP_FULL / OP_EMPTY x 3; E_READY / S_READY / ACC_FULL / ACC_EMPTY x 6;
    // C_READY / C_EMPTY x 4; RAW full / empty
#define OPF(s) (bar0 + 8u * (uint32_t)(0 + (s)))
#define OPE(s) (bar0 + 8u * (uint32_t)(3 + (s)))
#define EFL(s) (bar0 + 8u * (uint32_t)(6 + (s)))
#define SRD(s) (bar0 + 8u * (uint32_t)(12 + (s)))
#define ACF(s) (bar0 + 8u * (uint32_t)(18 + (s)))
#define ACE(s) (bar0 + 8u * (uint32_t)(24 + (s)))
#define CRD(s) (bar0 + 8u * (uint32_t)(30 + (s)))
#define CEM(s) (bar0 + 8u * (uint32_t)(34 + (s)))
#define RWF (bar0 + 8u * 38u)
#define RWE (bar0 + 8u * 39u)

    if (warp == 0) wptc::tmem_alloc(wptc::smem_u32(tmem_slot), 512);
    if (tid == 32) {
        for (int s = 0; s < NOP; ++s) {
            wptc::mbar_init(OPF(s), 1);
            wptc::mbar_init(OPE(s), 1);
        }
        for (int s = 0; s < LB_NA; ++s) {
            wptc::mbar_init(EFL(s), 1);
            wptc::mbar_init(SRD(s), CT_ROWS);
            wptc::mbar_init(ACF(s), 1);
            wptc::mbar_init(ACE(s), CT_ROWS);
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
    for (int i = tid; i < 64 * KS * 2 / 16; i += LB_THREADS)
        reinterpret_cast<uint4 *>(bsi)[i] = reinterpret_cast<const uint4 *>(a.Bsimg)[i];
    if (tid < LB_RING) stag[tid] = -1;
    wptc::fence_proxy_async_smem();
    wptc::fence_before_sync();
    __syncthreads();
    wptc::fence_after_sync();
    const uint32_t tmem = *tmem_slot;
    const long long first = blockIdx.x, stride = gridDim.x;
    const int ntiles = first < a.total_tiles ? (int)((a.total_tiles - 1 - first) / stride + 1) : 0;

    if (warp == 0) {
        // ================= MMA issuer: main(i), then state(i - LAG) =================
        if (lane == 0) {
            const uint32_t id_e = wptc::idesc_f16(128, LB_NS);  // first K atom: [g | Ke | 0]
            const uint32_t id_g = wptc::idesc_f16(128, 64);     // other atoms, state term
            const uint32_t op0 = wptc::smem_u32(op), b0 = wptc::smem_u32(bimg);
            const uint32_t sop0 = wptc::smem_u32(sop), bs0 = wptc::smem_u32(bsi);
            // issue whichever is ready: the next main GEMM (operands converted, a
            // free accumulator stage) or the next state GEMM (state operand
            // written); each kind in tile order
            int im = 0, is = 0;
            unsigned idle = 0;
            const unsigned long long t0 = ctd::gtimer();
            while (is < ntiles) {
                bool done = false;
                if (im < ntiles && im - is < LB_NA) {
                    const int so = im % NOP;
                    const int sa = im % LB_NA;
                    if (wptc::mbar_test(OPF(so), (uint32_t)((im / NOP) & 1)) &&
                        wptc::mbar_test(ACE(sa), (uint32_t)((im / LB_NA) & 1) ^ 1u)) {
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
                        ++im;
                        done = true;
                    }
                }
                if (is < im) {
                    const int sa = is % LB_NA;
                    if (wptc::mbar_test(SRD(sa), (uint32_t)((is / LB_NA) & 1))) {
                        // state term of tile is: [s_hi | s_lo | s_hi] x [E_hi; E_hi; E_lo]
                        wptc::fence_after_sync();
                        const uint32_t dm = tmem + (uint32_t)LB_NS * sa;
                        const uint32_t sa0 = sop0 + (uint32_t)(is & 1) * lay.sopBytes;
#pragma unroll
                        for (int kk = 0; kk < KS / 16; ++kk)
                            wptc::mma_f16(dm, c3d::desc_sbo(sa0 + 256u * kk, lb_sbo(D)),
                                          c3d::desc_sbo(bs0 + 256u * kk, lb_sbo(D)), id_g, 1u);
                        wptc::mma_commit(ACF(sa));
                        ++is;
                        done = true;
                    }
                }
                if (!done) {
                    __nanosleep(20);
                    if ((++idle & 1023u) == 0 && ctd::gtimer() - t0 > 10000000000ull) __trap();
                }
            }
        }
    } else if (warp == 1) {
        // ================= bulk-copy producer: fp32 window -> smem =================
        if (lane == 0) {
            const uint32_t raw0 = wptc::smem_u32(smem + lay.raw);
            for (int i = 0; i < ntiles; ++i) {
                wptc::mbar_wait_sleep<256>(RWE, (uint32_t)(i & 1) ^ 1u);
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
            wptc::mbar_wait_sleep<256>(RWF, (uint32_t)(i & 1));
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
    } else if (warp == 7) {
        // ================= look-back: carry-in of each tile =================
        for (int i = 0; i < ntiles; ++i) {
            const int sc4 = i % LB_NC;
            const long long tile = first + (long long)i * stride;
            const long long c = (long long)((unsigned long long)tile % (unsigned long long)a.C);
            const long long k = (long long)((unsigned long long)tile / (unsigned long long)a.C);
            wptc::mbar_wait_sleep<512>(CEM(sc4), (uint32_t)((i / LB_NC) & 1) ^ 1u);  // slot read by the row group
            if (lane == 0) LBTR(tile, 4);
            // c_k = sum_{l < j} MT^l agg(k-1-l) + MT^j incl(kb - 1)
            const long long kb = k & ~(long long)(LB_BLK - 1);
            const int j = (int)(k - kb);
            float w[D];
#pragma unroll
            for (int d = 0; d < D; ++d) w[d] = 0.f;
            // predecessors publish roughly in tile order: the nearest one first
            if (lane == 0 && j > 0) lbd::wait_word(a.aggw + ((k - 1) * a.C + c) * D + (D - 1));
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
        const int grp = (warp - 8) >> 2;
        const int wq = warp & 3;
        const int row = 32 * wq + lane;
        const uint32_t trow = (uint32_t)(32 * wq) << 16;
        unsigned char *mystg = stg + (size_t)(grp * 4 + wq) * 32 * CT_STG_PITCH;
        unsigned char *mysop = sop + (size_t)grp * lay.sopBytes;
        float *Tg = Tw + grp * 4 * D;  // this group's warp totals
        // scan of local tile i: zero-carry prefix s (row), warp start V, tile scale;
        // publishes the tile aggregate
        auto scan_tile = [&](int i, float (&s)[D], float (&V)[D], float &sci) {
            const int sa = i % LB_NA;
            const uint32_t para = (uint32_t)((i / LB_NA) & 1);
            const long long tile = first + (long long)i * stride;
            wptc::mbar_wait_sleep<256>(EFL(sa), para);
            wptc::fence_after_sync();
            float ev[16];
            ctd::tmem_ld16(tmem + (uint32_t)LB_NS * sa + 64u + trow, ev);
            wptc::tmem_wait_ld();
            for (int spins = 0; *reinterpret_cast<volatile int *>(stag + (i % LB_RING)) != i; ++spins) {
                __nanosleep(32);
                if (spins > (1 << 28)) __trap();
            }
            __threadfence_block();
            sci = scl[i % LB_RING];
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
                if (lane >= off) lbd::lt_mv4<D>(P, Mp + b * D * DP, prev);
            }
            // exclusive: state entering the row from the warp start (zero carry)
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
#pragma unroll
            for (int d = 0; d < D; ++d) V[d] = 0.f;
#pragma unroll 1
            for (int u = 0; u < wq; ++u) {
                float t[D];
#pragma unroll
                for (int d = 0; d < D; ++d) t[d] = Tg[u * D + d];
                lbd::lt_mv4<D>(t, Mp + 5 * D * DP, V);
#pragma unroll
                for (int d = 0; d < D; ++d) V[d] = t[d];
            }
            if (wq == 3 && lane == 0) {
                // tile aggregate (state at the next tile's start, zero carry) -> global
                float agg[D];
#pragma unroll
                for (int d = 0; d < D; ++d) agg[d] = Tg[3 * D + d];
                lbd::lt_mv4<D>(agg, Mp + 5 * D * DP, V);
#pragma unroll
                for (int d = 0; d < D; ++d) lbd::st_word(a.aggw + tile * D + d, agg[d]);
            }
            ctd::named_sync(3 + grp, 128);  // Tg is rewritten by the group's next tile
            if (row == 0) LBTR(tile, 6);
        };
        // software pipeline: the scan of the group's next tile runs before this
        // tile waits for its carry, so aggregates are published early and the
        // look-back latency overlaps a scan
        float sN[D], VN[D], sciN = 1.f;
#pragma unroll 1
        for (int it = grp; it < ntiles + 2; it += 2) {
            float s[D], V[D];
#pragma unroll
            for (int d = 0; d < D; ++d) s[d] = sN[d], V[d] = VN[d];
            const float sci = sciN;
            if (it < ntiles) scan_tile(it, sN, VN, sciN);
            const int i = it - 2;
            if (i < grp) continue;
            const int sa = i % LB_NA;
            const uint32_t para = (uint32_t)((i / LB_NA) & 1);
            const int sc4 = i % LB_NC;
            const long long tile = first + (long long)i * stride;
            const long long c = (long long)((unsigned long long)tile % (unsigned long long)a.C);
            const long long n0 = (long long)((unsigned long long)tile / (unsigned long long)a.C) * (long long)CT_TOUT;
            wptc::mbar_wait_sleep<256>(CRD(sc4), (uint32_t)((i / LB_NC) & 1));
            if (row == 0) LBTR(tile, 9);
            {
                // s_m = L_m + M^lane (Z_w + M^(32 w) c)
                float cin[D];
#pragma unroll
                for (int d = 0; d < D; ++d) cin[d] = cb[sc4 * D + d];
                ctd::arrive(CEM(sc4));
                lbd::lt_mv4<D>(V, Wt + wq * D * DP, cin);
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
                        lbd::lt_mv4<D>(t, Mp + b * D * DP, V);
                        if ((lane >> b) & 1) {
#pragma unroll
                            for (int d = 0; d < D; ++d) V[d] = t[d];
                        }
                    }
#pragma unroll
                    for (int d = 0; d < D; ++d) s[d] += V[d];
                }
            }
            // state operand [s_hi | s_lo | s_hi] x tile scale x 2^(fB - fE); a row that
            // would overflow fp16 sends zeros and takes the CUDA-core path below
            bool ovf = false;
            {
                const float f = sci * a.st_mul;
                float v[D];
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    v[d] = s[d] * f;
                    ovf = ovf || !(fabsf(v[d]) < 32768.f);
                }
#pragma unroll
                for (int k8 = 0; k8 < KS / 8; ++k8) {
                    uint32_t hw[4];
#pragma unroll
                    for (int t2 = 0; t2 < 4; ++t2) {
                        __half pr[2];
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            const int k = 8 * k8 + 2 * t2 + u;
                            const int part = k / DE, d = k % DE;  // 0: hi, 1: lo, 2: hi, 3: pad
                            const float val = (d < D && part < 3 && !ovf) ? v[d < D ? d : 0] : 0.f;
                            const __half hi = __float2half_rn(val);
                            pr[u] = part == 1 ? __float2half_rn(val - __half2float(hi)) : hi;
                        }
                        hw[t2] = (uint32_t)__half_as_ushort(pr[0]) | ((uint32_t)__half_as_ushort(pr[1]) << 16);
                    }
                    *reinterpret_cast<uint4 *>(mysop + lb_s_off(D, row, 8 * k8)) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                }
            }
            wptc::fence_proxy_async_smem();
            ctd::arrive(SRD(sa));
            wptc::mbar_wait_sleep<256>(ACF(sa), para);
            wptc::fence_after_sync();
            if (row == 0) LBTR(tile, 10);
            const float osc = a.out_scale / sci;
            const uint32_t tbase = tmem + (uint32_t)LB_NS * sa + trow;
            float *yr = a.y + c * a.ldy + n0;
            const long long tleft = a.N - n0;
            const bool full = a.vec_y && tleft >= CT_TOUT;
#pragma unroll 1
            for (int ch = 0; ch < 4; ++ch) {
                const int h = ch >> 1, hh = ch & 1;
                float o16[16];
                ctd::tmem_ld16(tbase + 16u * ch, o16);
                wptc::tmem_wait_ld();
                if (ch == 3) {
                    wptc::fence_before_sync();
                    ctd::arrive(ACE(sa));  // the accumulator has been read: free it
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) o16[j] *= osc;
                if (__any_sync(0xffffffffu, ovf)) {
                    // rare: rows whose state operand would overflow fp16 add E s here
#pragma unroll 1
                    for (int j = 0; j < 16; ++j) {
                        const float *e = Es + (16 * ch + j) * D;
                        float acc = 0.f;
#pragma unroll
                        for (int d = 0; d < D; ++d) acc = fmaf(e[d], s[d], acc);
                        if (ovf) reinterpret_cast<float *>(mystg + lane * CT_STG_PITCH + 64 * hh)[j] = acc;
                        else reinterpret_cast<float *>(mystg + lane * CT_STG_PITCH + 64 * hh)[j] = 0.f;
                    }
                    float4 *add = reinterpret_cast<float4 *>(mystg + lane * CT_STG_PITCH + 64 * hh);
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        const float4 t = add[q4];
                        o16[4 * q4] += t.x, o16[4 * q4 + 1] += t.y, o16[4 * q4 + 2] += t.z, o16[4 * q4 + 3] += t.w;
                    }
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
#undef EFL
#undef SRD
#undef ACF
#undef ACE
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
