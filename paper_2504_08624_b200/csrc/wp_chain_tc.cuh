// Tensor-core fused chain for sm_100a: pre-gain -> IIR SOS cascade -> FIR ->
// post-gains in ONE pass, as GEMMs on tcgen05 plus a chunk-state scan.
//
// Replaces the reference's per-stage passes (_iir_channel, _kernels_jit.py:
// 14-32; _fir_channel, :51-62; Chain.apply's stage loop, chain.py:66-71).
//
// Formulation. The pass is one LTI system: cascade state s
// (D = 2S DF2T states), impulse response h, FIR f, gain G. For tile rows
// m = 0..127 of 64 outputs (n = n0 + 64 m + p), window start w_m = n0 - H + 64 m
// (H >= taps - 1):
//
//   y[n] = sum_{k < H+64} g[p + H - k] x[w_m + k]      main GEMM, fp16 x3 split,
//                                                      fp32 accumulation (TMEM)
//        + sum_i E[p][i] s_{w_m}[i]                     state term, TS (fp64/fp32)
//   g = G (f * h),  E[p] = G sum_t f[t] C A^(H+p-t)
//
// Row-start states come from a scan over the rows:
//   s_{w_{m+1}} = M s_{w_m} + e_m,  M = A^64,  e_m = sum_j A^(63-j) B x[w_m+j]
// e_m is an EXACT integer GEMM on the tensor cores (kind::i8): x as a 24-bit
// per-tile fixed-point number in 3 int8 digits, A^(63-j) B as 31-bit per-state
// fixed point in 4 digits, int32 accumulation per digit level. The chain's
// output is the small difference of the window term and the state term when
// the input sits in a stopband (cfg3's 100 Hz high-pass with low-frequency
// input), so e must be accurate far beyond fp32 (tools/emulate_tcchain.py).
// The scan runs in TS: Kogge-Stone over rows with M^(2^i), warp prefixes with
// M^32, and a deterministic blocked decoupled look-back across tiles with
// M^128 (as in wp_fused.cuh).
//
// Warp roles (persistent, one CTA per SM, static tile schedule, every hand-off
// double-buffered through mbarriers):
//   warp 0       TMEM allocation; lane 0 issues the int8 e-GEMM (24 MMAs) and
//                the fp16 main GEMM (3 x K/16 MMAs) per tile
//   warps 2-6    converters: coalesced loads of the fp32 window (the next
//                window is prefetched into L2 by a bulk prefetch) -> SW128 fp16
//                hi/lo operands + int8 digit planes
//   warps 8-11   scan: e from TMEM, row scan, zero-carry row prefixes L_m,
//                tile aggregate
//   warps 1, 7   look-back for even / odd local tiles: carry-in of the tile,
//                V_w = M^(32 w) carry
//   warps 12-15  epilogue: s_m = L_m + M^lane V_w, TMEM -> registers,
//                + E s_m, staging, coalesced stores
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "wp_fused.cuh"
#include "wp_tc.cuh"

namespace wpk {

constexpr int CT_THREADS = 512;
constexpr int CT_CONV = 160;            // warps 2..6
constexpr int CT_QMAX = 14;             // float4 of the window per converter thread (W <= 8960)
constexpr int CT_ROWS = 128;            // UMMA M
constexpr int CT_TOUT = CT_ROWS * 64;   // outputs per tile
constexpr int CT_MAX_H = 128;           // FIR halo limit (K <= 192, smem)
constexpr int CT_STG_PITCH = 144;       // staging row pitch: 32 floats + 16 B pad
constexpr int CT_TRACE_EV = 12;         // trace events per tile
constexpr int CT_XD = 3;                // int8 digits of x
constexpr int CT_KD = 4;                // int8 digits of the chunk-state weights

struct ChainTcArgs {
    const float *x;
    float *y;
    long long C, N, ldx, ldy;
    long long total_tiles;
    int H, K, W;
    const unsigned char *Bimg;   // [2][atoms][64 rows][128 B], SW128 K-major fp16 hi / lo of g
    const unsigned char *Bk;     // [CT_KD][16 rows][64 B] int8 digits of A^(63-j) B, no-swizzle K-major
    float out_scale;             // 2^-fB of the g image
    double kscale[8];            // 2^-kappa_d of the digit image, per state
    const void *G;               // [D][D][33] TS, M^l lane-minor
    const void *TP;              // [33][D][D] TS, (M^128)^j
    void *recs;
    unsigned long long epoch;
    int vec_x, vec_y;
    int dbg;                     // diagnostics: 1 = no look-back wait, 4 = no state term
    unsigned long long *trace;   // optional: [tiles][CT_TRACE_EV] globaltimer stamps
};

template <typename TS, int D>
struct ETable {
    TS E[64][D];
};

namespace ctd {

__device__ __forceinline__ uint32_t swz128(uint32_t byte) { return byte ^ (((byte >> 7) & 7u) << 4); }

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1u << 16;
    d |= (uint64_t)((1024u >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1u << 46;
    d |= (uint64_t)2u << 61;
    return d;
}

// K-major, no swizzle: core matrices of 8 rows x 16 B; LBO = 128 B (next core
// matrix along K), SBO = 512 B (next 8-row group); rows of 64 bytes
// (hardware-checked by tools/i8_probe.cu).
__device__ __forceinline__ uint64_t desc_none(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)(128u >> 4) << 16;
    d |= (uint64_t)(512u >> 4) << 32;
    d |= (uint64_t)1u << 46;
    return d;
}

__host__ __device__ __forceinline__ uint32_t dg_off(int r, int k) {
    return (uint32_t)((r >> 3) * 512 + (k >> 4) * 128 + (r & 7) * 16 + (k & 15));
}

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, int as, int bs) {
    return (2u << 4) | ((uint32_t)as << 7) | ((uint32_t)bs << 10) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld8i(uint32_t taddr, int (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr)
                 : "memory");
}

// out += M v, M block lower triangular (2x2 blocks), accessor m(i, j); the
// products of a row are summed as a balanced tree (short dependency chains)
template <int D, typename TS, typename F>
__device__ __forceinline__ void matvec_tree(TS (&out)[D], const TS (&v)[D], F m) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
        const int nj = 2 * ((i >> 1) + 1);  // columns 0 .. nj-1 can be nonzero
        TS part[D];
#pragma unroll
        for (int j = 0; j < D; ++j)
            if (j < nj) part[j] = m(i, j) * v[j];
#pragma unroll
        for (int w = 1; w < D; w <<= 1) {
#pragma unroll
            for (int j = 0; j + w < D; j += 2 * w)
                if (j + w < nj) part[j] += part[j + w];
        }
        out[i] += part[0];
    }
}

}  // namespace ctd

// shared memory carve-up (offsets from the 1024-aligned base)
// block-lower-triangular row r of a D x D transfer matrix has entries q < nj(r)
__host__ __device__ constexpr int lt_nj(int r) { return 2 * ((r >> 1) + 1); }
__host__ __device__ constexpr int lt_off(int r) {
    return (r & 1) ? 2 * ((r >> 1) + 1) * ((r >> 1) + 1) : 2 * (r >> 1) * ((r >> 1) + 1);
}
__host__ __device__ constexpr int lt_size(int D) { return lt_off(D); }

struct CtLayout {
    uint32_t opBytes, bBytes;
    uint32_t bimg, bk, op, dg, g, tabs, sbuf, stg, misc, bars;
    uint32_t total;
    __host__ __device__ CtLayout(int W, int K, int D, int ts) {
        opBytes = ((uint32_t)W * 2u + 1023u) & ~1023u;
        bBytes = (uint32_t)((K + 63) / 64) * 8192u;
        bimg = 0;
        bk = bimg + 2 * bBytes;
        op = bk + CT_KD * 1024u;
        dg = op + 4 * opBytes;
        g = dg + 2u * CT_XD * 8192u;
        // G: M^lane, lane < 32, compact lower-triangular entries, lane-minor
        tabs = (g + (uint32_t)(ts * lt_size(D) * 32) + 15u) & ~15u;
        // tabs: P[5][D][D], W[4][D][D], MT[D][D], E[64][D]
        sbuf = (tabs + (uint32_t)(ts * (10 * D * D + 64 * D)) + 15u) & ~15u;
        stg = sbuf + 2u * CT_ROWS * (uint32_t)(D * ts);
        misc = stg + 4u * 32u * CT_STG_PITCH;
        // misc: warp_incl[2][4][D], agg[2][D], cv[2][4][D] (TS); scl[8] f32, xex[8] i32, red[8] f32
        bars = (misc + (uint32_t)(ts * (8 * D + 2 * D + 8 * D)) + 96u + 15u) & ~15u;
        total = bars + 30 * 8 + 16 + 1024;  // + alignment slack
    }
};

template <typename TS, int S>
__global__ void __launch_bounds__(CT_THREADS, 1)
    chain_tc_kernel(const ChainTcArgs a, const IirTables<TS, S> tb, const ETable<TS, 2 * S> et) {
    constexpr int D = 2 * S;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // align by offsetting the __shared__ array itself (keeps the shared
    // address space visible to the compiler: LDS/STS, not generic LD/ST)
    unsigned char *smem = smem_raw + ((1024u - (wptc::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nk = a.K / 16;
    const CtLayout lay(a.W, a.K, D, (int)sizeof(TS));
    unsigned char *bimg = smem + lay.bimg;
    unsigned char *op = smem + lay.op;
    unsigned char *dg = smem + lay.dg;
    TS *gsm = reinterpret_cast<TS *>(smem + lay.g);
    TS *Ps = reinterpret_cast<TS *>(smem + lay.tabs);  // [5][D][D]
    TS *Ws = Ps + 5 * D * D;                           // [4][D][D]
    TS *MTs = Ws + 4 * D * D;                          // [D][D]
    // E transposed, split into fp32 hi / lo parts: Esh[D][64], Esl[D][64]
    float *Esh = reinterpret_cast<float *>(MTs + D * D);
    float *Esl = Esh + D * 64;
    TS *sbuf = reinterpret_cast<TS *>(smem + lay.sbuf);
    unsigned char *stg = smem + lay.stg;
    TS *warp_incl = reinterpret_cast<TS *>(smem + lay.misc);  // [2][4][D]
    TS *agg_s = warp_incl + 8 * D;                              // [2][D]
    TS *cv_s = agg_s + 2 * D;                                   // [2][4][D]
    float *scl = reinterpret_cast<float *>(cv_s + 8 * D);      // [8] ring by local tile
    int *xex = reinterpret_cast<int *>(scl + 8);                // [8]
    float *red = reinterpret_cast<float *>(xex + 8);            // [8]
    unsigned long long *bars = reinterpret_cast<unsigned long long *>(smem + lay.bars);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 30);
    const uint32_t bar0 = wptc::smem_u32(bars);
    enum {
        OP_FULL = 0, OP_EMPTY, EF_FULL, ACC_FULL, ACC_EMPTY, SB_FULL, SB_EMPTY, AG_FULL, CV_FULL, CV_EMPTY
    };
#define CBAR(kind, s) (bar0 + 8u * (uint32_t)(3 * (kind) + (s)))

    // ---- one-time setup ----
    if (warp == 0) wptc::tmem_alloc(wptc::smem_u32(tmem_slot), 512);
    if (tid == 32) {
        for (int s = 0; s < 3; ++s) {
            wptc::mbar_init(CBAR(OP_FULL, s), 1);
            wptc::mbar_init(CBAR(OP_EMPTY, s), 1);
            wptc::mbar_init(CBAR(EF_FULL, s), 1);
            wptc::mbar_init(CBAR(ACC_FULL, s), 1);
            wptc::mbar_init(CBAR(ACC_EMPTY, s), 256);
            wptc::mbar_init(CBAR(SB_FULL, s), 128);
            wptc::mbar_init(CBAR(SB_EMPTY, s), 128);
            wptc::mbar_init(CBAR(AG_FULL, s), 1);
            wptc::mbar_init(CBAR(CV_FULL, s), 1);
            wptc::mbar_init(CBAR(CV_EMPTY, s), 128);
        }
        wptc::mbar_fence_init();
    }
    for (int i = tid; i < (int)(2 * lay.bBytes / 16); i += CT_THREADS)
        reinterpret_cast<uint4 *>(bimg)[i] = reinterpret_cast<const uint4 *>(a.Bimg)[i];
    for (int i = tid; i < CT_KD * 1024 / 16; i += CT_THREADS)
        reinterpret_cast<uint4 *>(smem + lay.bk)[i] = reinterpret_cast<const uint4 *>(a.Bk)[i];
    {
        const TS *G = reinterpret_cast<const TS *>(a.G);
        for (int i = tid; i < D * D * 32; i += CT_THREADS) {
            const int r = i / (D * 32), q = (i / 32) % D, l = i % 32;
            if (q < lt_nj(r)) gsm[(lt_off(r) + q) * 32 + l] = G[(r * D + q) * 33 + l];
        }
        for (int i = tid; i < D * D; i += CT_THREADS) {
            const int r = i / D, q = i % D;
            for (int t = 0; t < 5; ++t) Ps[t * D * D + i] = tb.P[t][r][q];
            for (int t = 0; t < 4; ++t) Ws[t * D * D + i] = tb.W[t][r][q];
            MTs[i] = tb.MT[r][q];
        }
        for (int i = tid; i < 64 * D; i += CT_THREADS) {
            const double e = (double)et.E[i % 64][i / 64];
            Esh[i] = (float)e;
            Esl[i] = (float)(e - (double)(float)e);
        }
    }
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
            const uint32_t idesc = wptc::idesc_f16(128, 64);
            const uint32_t op0 = wptc::smem_u32(op), b0 = wptc::smem_u32(bimg);
            const uint32_t dg0 = wptc::smem_u32(dg), bk0 = wptc::smem_u32(smem + lay.bk);
            for (int i = 0; i < ntiles; ++i) {
                const int s = i & 1;
                const uint32_t par = (uint32_t)((i >> 1) & 1);
                const int s3 = i % 3;
                const uint32_t par3 = (uint32_t)((i / 3) & 1);
                wptc::mbar_wait(CBAR(OP_FULL, s), par);
                wptc::mbar_wait(CBAR(ACC_EMPTY, s3), par3 ^ 1u);
                wptc::fence_after_sync();
                if (a.trace) a.trace[(first + (long long)i * stride) * CT_TRACE_EV + 2] = ctd::gtimer();
                const uint32_t dm = tmem + 160u * s3;  // TMEM stage: main [0,64), e levels [64,160)
                // ---- exact e-GEMM: level l = xa + kb, digits xa < 3 (top signed), kb < 4 (top signed) ----
#pragma unroll
                for (int l = 0; l < CT_XD + CT_KD - 1; ++l) {
                    int nmma = 0;
#pragma unroll
                    for (int xa = 0; xa < CT_XD; ++xa) {
                        const int kb = l - xa;
                        if (kb < 0 || kb >= CT_KD) continue;
                        const uint32_t id = ctd::idesc_i8(128, 16, xa == CT_XD - 1, kb == CT_KD - 1);
#pragma unroll
                        for (int kh = 0; kh < 2; ++kh) {
                            const uint64_t da = ctd::desc_none(dg0 + (uint32_t)(s * CT_XD + xa) * 8192u + 256u * kh);
                            const uint64_t db = ctd::desc_none(bk0 + (uint32_t)kb * 1024u + 256u * kh);
                            ctd::mma_i8(dm + 64u + 16u * l, da, db, id, nmma > 0);
                            ++nmma;
                        }
                    }
                }
                wptc::mma_commit(CBAR(EF_FULL, s3));
                // ---- main GEMM: fp16 x3 (hi hi + lo hi + hi lo), one fp32 accumulator ----
                const uint32_t ahi = op0 + (2u * s) * lay.opBytes, alo = ahi + lay.opBytes;
                const uint64_t ah0 = ctd::desc_sw128(ahi), al0 = ctd::desc_sw128(alo);
#pragma unroll 1
                for (int kk = 0; kk < nk; ++kk) {
                    const uint64_t ka = 2u * kk;  // +32 B per K step, across rows (Hankel)
                    const uint32_t boff = 8192u * (kk >> 2) + 32u * (kk & 3);
                    const uint64_t bh = ctd::desc_sw128(b0 + boff), bl = ctd::desc_sw128(b0 + lay.bBytes + boff);
                    wptc::mma_f16(dm, ah0 + ka, bh, idesc, kk > 0);
                    wptc::mma_f16(dm, al0 + ka, bh, idesc, 1u);
                    wptc::mma_f16(dm, ah0 + ka, bl, idesc, 1u);
                }
                wptc::mma_commit(CBAR(OP_EMPTY, s));
                wptc::mma_commit(CBAR(ACC_FULL, s3));
            }
        }
    } else if (warp >= 2 && warp <= 6) {
        // ================= converters (warps 2..6) =================
        const int ct = tid - 64;
        const int cw = ct >> 5;
        const int nq = a.W / 4;
        for (int i = 0; i < ntiles; ++i) {
            const int s = i & 1;
            const uint32_t par = (uint32_t)((i >> 1) & 1);
            const long long tile = first + (long long)i * stride;
            const long long c = (long long)((unsigned)tile % (unsigned)a.C);
            const long long n0 = (long long)((unsigned)tile / (unsigned)a.C) * (long long)CT_TOUT;
            const long long start = n0 - a.H;
            const float *xr = a.x + c * a.ldx;
            if (ct == 0) {
                if (a.trace) a.trace[tile * CT_TRACE_EV + 0] = ctd::gtimer();
                // warm L2 with the next tile's window while this one is converted
                const long long nt = tile + stride;
                if (nt < a.total_tiles && a.vec_x) {
                    const long long c2 = (long long)((unsigned)nt % (unsigned)a.C);
                    const long long s2 = (long long)((unsigned)nt / (unsigned)a.C) * (long long)CT_TOUT - a.H;
                    long long lo = s2 > 0 ? s2 : 0, hi = s2 + a.W;
                    if (hi > (a.N & ~3LL)) hi = a.N & ~3LL;
                    lo &= ~3LL;
                    const uint32_t bytes = (uint32_t)(4 * (hi - lo)) & ~15u;
                    if (hi > lo && bytes > 0) ctd::prefetch_l2(a.x + c2 * a.ldx + lo, bytes);
                }
            }
            float4 v[CT_QMAX];
            float m = 0.f;
            const bool interior = a.vec_x && start >= 0 && start + a.W <= a.N;
#pragma unroll
            if (interior) {
                const float4 *src4 = reinterpret_cast<const float4 *>(xr + start) + ct;
#pragma unroll
                for (int j = 0; j < CT_QMAX; ++j)
                    v[j] = (ct + j * CT_CONV < nq) ? __ldcs(src4 + j * CT_CONV) : make_float4(0.f, 0.f, 0.f, 0.f);
            } else {
#pragma unroll 1
                for (int j = 0; j < CT_QMAX; ++j) {
                    const int q = ct + j * CT_CONV;
                    const float4 t = q < nq ? load_region4(xr, start + 4LL * q, a.N, a.vec_x) : make_float4(0.f, 0.f, 0.f, 0.f);
                    // register arrays need static indices: select into place
#pragma unroll
                    for (int jj = 0; jj < CT_QMAX; ++jj)
                        if (jj == j) v[jj] = t;
                }
            }
#pragma unroll
            for (int j = 0; j < CT_QMAX; ++j)
                m = fmaxf(m, fmaxf(fmaxf(fabsf(v[j].x), fabsf(v[j].y)), fmaxf(fabsf(v[j].z), fabsf(v[j].w))));
            const unsigned mb = __reduce_max_sync(0xffffffffu, __float_as_uint(m));
            if (lane == 0) red[cw] = __uint_as_float(mb);
            wptc::mbar_wait(CBAR(OP_EMPTY, s), par ^ 1u);
            ctd::named_sync(1, CT_CONV);
            float tmax = red[0];
#pragma unroll
            for (int w = 1; w < CT_CONV / 32; ++w) tmax = fmaxf(tmax, red[w]);
            int ex = 0;
            if (tmax > 0.f) frexpf(tmax, &ex);
            const float sc = ldexpf(1.f, tmax > 0.f ? 14 - ex : 0);
            const float xs = ldexpf(1.f, tmax > 0.f ? 22 - ex : 0);  // |X| < 2^22: no overflow
            unsigned char *ohi = op + (2 * s) * lay.opBytes, *olo = ohi + lay.opBytes;
            unsigned char *dgs = dg + (size_t)s * CT_XD * 8192;
#pragma unroll
            for (int j = 0; j < CT_QMAX; ++j) {
                const int q = ct + j * CT_CONV;
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
                    if (q < CT_TOUT / 4) {
                        // 23-bit fixed point in 3 int8 digits (top digit signed): bytes
                        // 0/1/2 of the four int32 values, gathered with byte permutes
                        const uint32_t X0 = (uint32_t)__float2int_rn(v[j].x * xs), X1 = (uint32_t)__float2int_rn(v[j].y * xs);
                        const uint32_t X2 = (uint32_t)__float2int_rn(v[j].z * xs), X3 = (uint32_t)__float2int_rn(v[j].w * xs);
                        const uint32_t a01 = __byte_perm(X0, X1, 0x5140), a23 = __byte_perm(X2, X3, 0x5140);  // b0 b0' b1 b1'
                        const uint32_t c01 = __byte_perm(X0, X1, 0x0062), c23 = __byte_perm(X2, X3, 0x0062);  // b2 b2'
                        const uint32_t d0 = __byte_perm(a01, a23, 0x5410);
                        const uint32_t d1 = __byte_perm(a01, a23, 0x7632);
                        const uint32_t d2 = __byte_perm(c01, c23, 0x5410);
                        const uint32_t o = ctd::dg_off(q >> 4, (q & 15) * 4);
                        *reinterpret_cast<uint32_t *>(dgs + o) = d0;
                        *reinterpret_cast<uint32_t *>(dgs + 8192 + o) = d1;
                        *reinterpret_cast<uint32_t *>(dgs + 16384 + o) = d2;
                    }
                }
            }
            if (ct == 0) {
                scl[i & 7] = sc;
                xex[i & 7] = tmax > 0.f ? 22 - ex : 0;
            }
            wptc::fence_proxy_async_smem();
            ctd::named_sync(2, CT_CONV);
            if (ct == 0) {
                ctd::arrive(CBAR(OP_FULL, s));
                if (a.trace) a.trace[tile * CT_TRACE_EV + 1] = ctd::gtimer();
            }
        }
    } else if (warp == 1 || warp == 7) {
        // ================= look-back (warp 1: even local tiles, warp 7: odd) =================
        const int s = warp == 1 ? 0 : 1;
        const TS *TP = reinterpret_cast<const TS *>(a.TP);
        TileRec<TS, D> *recs = reinterpret_cast<TileRec<TS, D> *>(a.recs);
        for (int i = s; i < ntiles; i += 2) {
            const uint32_t par = (uint32_t)((i >> 1) & 1);
            const long long tile = first + (long long)i * stride;
            const long long c = (long long)((unsigned)tile % (unsigned)a.C);
            const long long k = (long long)((unsigned)tile / (unsigned)a.C);
            wptc::mbar_wait(CBAR(AG_FULL, s), par);
            if (lane == 0 && a.trace) a.trace[tile * CT_TRACE_EV + 5] = ctd::gtimer();
            TS agg[D], carry[D];
#pragma unroll
            for (int d = 0; d < D; ++d) {
                agg[d] = agg_s[s * D + d];
                carry[d] = TS(0);
            }
            TileRec<TS, D> *mine = recs + tile;
            const int kb = (int)(k & 31);
            const long long base = k - kb;
            if (lane == 0 && kb < 31) {
#pragma unroll
                for (int d = 0; d < D; ++d) mine->agg[d] = agg[d];
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
            if (src && !(a.dbg & 1)) {
                const unsigned long long want = (a.epoch << 2) | (unsigned long long)need;
                unsigned long long f = ld_acquire(&src->flag);
                int spins = 0;
                while ((f >> 2) != a.epoch || (f & 3ull) < (unsigned long long)need || f < want) {
                    if (++spins > 8) __nanosleep(spins < 64 ? 20 : 100);
                    if ((spins & 0x3FFFFFF) == 0) __trap();  // watchdog: ~64M polls without progress
                    f = ld_acquire(&src->flag);
                }
                const TS *sv = need == 2 ? src->incl : src->agg;
                TS val[D];
#pragma unroll
                for (int d = 0; d < D; ++d) val[d] = ldcg(sv + d);
                const TS *Mj = TP + (size_t)pw * D * D;
                ctd::matvec_tree<D, TS>(carry, val, [&](int r, int q) { return ldcg(Mj + r * D + q); });
            }
#pragma unroll
            for (int d = 0; d < D; ++d) {
                TS v = carry[d];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += shfl_xor(v, o);
                carry[d] = v;
            }
            if (lane == 0 && a.trace) a.trace[tile * CT_TRACE_EV + 11] = ctd::gtimer();
            if (lane == 0 && kb == 31) {
                TS P[D];
#pragma unroll
                for (int d = 0; d < D; ++d) P[d] = agg[d];
                ctd::matvec_tree<D, TS>(P, carry, [&](int r, int q) { return MTs[r * D + q]; });
#pragma unroll
                for (int d = 0; d < D; ++d) mine->incl[d] = P[d];
                __threadfence();
                st_release(&mine->flag, (a.epoch << 2) | 2ull);
            }
            // V_w = M^(32 w) carry for the four row blocks: lane = 8 w + d
            wptc::mbar_wait(CBAR(CV_EMPTY, s), par ^ 1u);
            {
                const int w = lane >> 3, d = lane & 7;
                if (d < D) {
                    TS acc = TS(0);
#pragma unroll
                    for (int j = 0; j < D; ++j) {
                        acc = fma(Ws[(w * D + d) * D + j], carry[j], acc);
                    }
                    cv_s[(s * 4 + w) * D + d] = acc;
                }
            }
            __syncwarp();
            if (lane == 0) {
                ctd::arrive(CBAR(CV_FULL, s));
                if (a.trace) a.trace[tile * CT_TRACE_EV + 6] = ctd::gtimer();
            }
        }
    } else if (warp >= 8 && warp <= 11) {
        // ================= scan (warps 8..11), one tile row per thread =================
        const int wq = warp & 3;
        const int row = 32 * wq + lane;
        const uint32_t trow = (uint32_t)(32 * wq) << 16;
        for (int i = 0; i < ntiles; ++i) {
            const int s = i & 1;
            const uint32_t par = (uint32_t)((i >> 1) & 1);
            const long long tile = first + (long long)i * stride;
            const int s3 = i % 3;
            wptc::mbar_wait(CBAR(EF_FULL, s3), (uint32_t)((i / 3) & 1));
            wptc::fence_after_sync();
            if (row == 0 && a.trace) a.trace[tile * CT_TRACE_EV + 3] = ctd::gtimer();
            int lv[CT_XD + CT_KD - 1][8];
#pragma unroll
            for (int l = 0; l < CT_XD + CT_KD - 1; ++l) ctd::tmem_ld8i(tmem + 160u * s3 + trow + 64u + 16u * l, lv[l]);
            wptc::tmem_wait_ld();
            const int xe = xex[i & 7];
            wptc::fence_before_sync();
            ctd::arrive(CBAR(ACC_EMPTY, s3));
            TS e[D];
            {
                const double xscale = ldexp(1.0, -xe);
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    double acc = 0.0;
#pragma unroll
                    for (int l = CT_XD + CT_KD - 2; l >= 0; --l) acc = acc * 256.0 + (double)lv[l][d];
                    e[d] = TS(acc * (xscale * a.kscale[d]));
                }
            }
            // warp inclusive scan over rows: incl_t = e_t + M incl_{t-1}
            TS incl[D];
#pragma unroll
            for (int d = 0; d < D; ++d) incl[d] = e[d];
#pragma unroll 1
            for (int stp = 0; stp < 5; ++stp) {
                const int off = 1 << stp;
                TS prev[D];
#pragma unroll
                for (int d = 0; d < D; ++d) prev[d] = shfl_up(incl[d], off);
                if (lane >= off) ctd::matvec_tree<D, TS>(incl, prev, [&](int r, int q) { return Ps[(stp * D + r) * D + q]; });
            }
            TS Lm[D];
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const TS v = shfl_up(incl[d], 1);
                Lm[d] = lane == 0 ? TS(0) : v;
            }
            TS *wi = warp_incl + s * 4 * D;
            if (lane == 31) {
#pragma unroll
                for (int d = 0; d < D; ++d) wi[wq * D + d] = incl[d];
            }
            ctd::named_sync(3, 128);
            // prefix entering this row block (zero carry): wc = sum_{u < wq} M^(32 (wq-1-u)) incl_u
            {
                TS wc[D];
#pragma unroll
                for (int d = 0; d < D; ++d) wc[d] = TS(0);
#pragma unroll 1
                for (int u = 0; u < wq; ++u) {
                    {
                        TS iu[D];
#pragma unroll
                        for (int d = 0; d < D; ++d) iu[d] = wi[u * D + d];
                        const int pw = wq - 1 - u;
                        ctd::matvec_tree<D, TS>(wc, iu, [&](int r, int q) { return Ws[(pw * D + r) * D + q]; });
                    }
                }
                ctd::matvec_tree<D, TS>(Lm, wc, [&](int r, int q) { return gsm[(lt_off(r) + q) * 32 + lane]; });
            }
            wptc::mbar_wait(CBAR(SB_EMPTY, s), par ^ 1u);
            if (row == 0 && a.trace) a.trace[tile * CT_TRACE_EV + 9] = ctd::gtimer();
            {
                TS *dst = sbuf + ((size_t)s * CT_ROWS + row) * D;
#pragma unroll
                for (int d = 0; d < D; ++d) dst[d] = Lm[d];
            }
            if (row == 0) {
                // tile aggregate: inclusive prefix after the last row, zero carry
                TS ag[D];
#pragma unroll
                for (int d = 0; d < D; ++d) ag[d] = wi[3 * D + d];
#pragma unroll 1
                for (int u = 0; u < 3; ++u) {
                    TS iu[D];
#pragma unroll
                    for (int d = 0; d < D; ++d) iu[d] = wi[u * D + d];
                    const int pw = 3 - u;
                    ctd::matvec_tree<D, TS>(ag, iu, [&](int r, int q) { return Ws[(pw * D + r) * D + q]; });
                }
#pragma unroll
                for (int d = 0; d < D; ++d) agg_s[s * D + d] = ag[d];
                ctd::arrive(CBAR(AG_FULL, s));
                if (a.trace) a.trace[tile * CT_TRACE_EV + 4] = ctd::gtimer();
            }
            ctd::arrive(CBAR(SB_FULL, s));
        }
    } else if (warp >= 12) {
        // ================= epilogue (warps 12..15), one tile row per thread =================
        // TMEM is triple-buffered, so the epilogue can read the accumulator
        // after the look-back's carry arrives without stalling the GEMM.
        const int wq = warp & 3;
        const int row = 32 * wq + lane;
        const uint32_t trow = (uint32_t)(32 * wq) << 16;
        unsigned char *mystg = stg + (size_t)wq * 32 * CT_STG_PITCH;
        for (int i = 0; i < ntiles; ++i) {
            const int s = i & 1, s3 = i % 3;
            const uint32_t par = (uint32_t)((i >> 1) & 1);
            const long long tile = first + (long long)i * stride;
            const long long c = (long long)((unsigned)tile % (unsigned)a.C);
            const long long n0 = (long long)((unsigned)tile / (unsigned)a.C) * (long long)CT_TOUT;
            TS sv[D], V[D];
            wptc::mbar_wait(CBAR(SB_FULL, s), par);
#pragma unroll
            for (int d = 0; d < D; ++d) sv[d] = sbuf[((size_t)s * CT_ROWS + row) * D + d];
            ctd::arrive(CBAR(SB_EMPTY, s));
            wptc::mbar_wait(CBAR(CV_FULL, s), par);
            if (row == 0 && a.trace) a.trace[tile * CT_TRACE_EV + 10] = ctd::gtimer();
#pragma unroll
            for (int d = 0; d < D; ++d) V[d] = cv_s[(s * 4 + wq) * D + d];
            ctd::arrive(CBAR(CV_EMPTY, s));
            ctd::matvec_tree<D, TS>(sv, V, [&](int r, int q) { return gsm[(lt_off(r) + q) * 32 + lane]; });
            float sh[D], sl[D];
#pragma unroll
            for (int d = 0; d < D; ++d) {
                sh[d] = (float)sv[d];
                sl[d] = (float)(sv[d] - (TS)sh[d]);
            }
            wptc::mbar_wait(CBAR(ACC_FULL, s3), (uint32_t)((i / 3) & 1));
            wptc::fence_after_sync();
            if (row == 0 && a.trace) a.trace[tile * CT_TRACE_EV + 7] = ctd::gtimer();
            const float osc = a.out_scale / scl[i & 7];
            const uint32_t tbase = tmem + 160u * s3 + trow;
            float *yr = a.y + c * a.ldy + n0;
#pragma unroll 1
            for (int ch = 0; ch < 4; ++ch) {
                const int h = ch >> 1, hh = ch & 1;
                float t16[16];
                ctd::tmem_ld16(tbase + 16u * ch, t16);
                wptc::tmem_wait_ld();
                if (ch == 3) {
                    wptc::fence_before_sync();
                    ctd::arrive(CBAR(ACC_EMPTY, s3));
                }
                // state term in fp32 double-single: E s = Eh sh + (El sh + Eh sl)
                // (no fp64 <-> fp32 conversions per output; error ~2^-24 |E s|)
                float acc[16], cor[16];
#pragma unroll
                for (int pp = 0; pp < 16; ++pp) {
                    acc[pp] = t16[pp] * osc;
                    cor[pp] = 0.f;
                }
                if (!(a.dbg & 4)) {
#pragma unroll
                    for (int d = 0; d < D; ++d) {
                        const float4 *eh = reinterpret_cast<const float4 *>(Esh + d * 64 + 16 * ch);  // uniform: broadcast
                        const float4 *el = reinterpret_cast<const float4 *>(Esl + d * 64 + 16 * ch);
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) {
                            const float4 h4 = eh[q4], l4 = el[q4];
                            const float hv[4] = {h4.x, h4.y, h4.z, h4.w}, lv4[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                acc[4 * q4 + u] = fmaf(hv[u], sh[d], acc[4 * q4 + u]);
                                if constexpr (sizeof(TS) == 8)
                                    cor[4 * q4 + u] = fmaf(lv4[u], sh[d], fmaf(hv[u], sl[d], cor[4 * q4 + u]));
                            }
                        }
                    }
                }
                float4 *dst = reinterpret_cast<float4 *>(mystg + lane * CT_STG_PITCH + 64 * hh);
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4)
                    dst[q4] = make_float4(acc[4 * q4] + cor[4 * q4], acc[4 * q4 + 1] + cor[4 * q4 + 1],
                                          acc[4 * q4 + 2] + cor[4 * q4 + 2], acc[4 * q4 + 3] + cor[4 * q4 + 3]);
                if (hh == 1) {
                    __syncwarp();
                    // 32 rows x 32 outputs of this half: 8 float4 per row, 4 rows per instruction
                    const long long tleft = a.N - n0;  // valid outputs in this tile
#pragma unroll 1
                    for (int r = 0; r < 8; ++r) {
                        const int q = lane + 32 * r;
                        const int rr = q >> 3, c4 = q & 7;
                        const float4 v = *reinterpret_cast<const float4 *>(mystg + rr * CT_STG_PITCH + 16 * c4);
                        const int o = 64 * (32 * wq + rr) + 32 * h + 4 * c4;  // offset from n0
                        const long long left = tleft - o;
                        if (a.vec_y && left >= 4) {
                            __stcs(reinterpret_cast<float4 *>(yr + o), v);
                        } else {
                            if (left > 0) yr[o + 0] = v.x;
                            if (left > 1) yr[o + 1] = v.y;
                            if (left > 2) yr[o + 2] = v.z;
                            if (left > 3) yr[o + 3] = v.w;
                        }
                    }
                    __syncwarp();
                }
            }
            if (row == 0 && a.trace) a.trace[tile * CT_TRACE_EV + 8] = ctd::gtimer();
        }
    }
#undef CBAR
    wptc::fence_before_sync();
    __syncthreads();
    wptc::fence_after_sync();
    if (warp == 0) wptc::tmem_dealloc(tmem, 512);
}

}  // namespace wpk
