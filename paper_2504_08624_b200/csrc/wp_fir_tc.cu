// Tensor-core FIR (tcgen05, kind::f16, split precision) for sm_100a.
//
// Direct-form convolution y[n] = sum_t h[t] x[n-t] (the reference's
// _fir_channel, _kernels_jit.py:51-62) as one GEMM per tile of 8192 outputs
// of one channel:
//
//   D[m, p] = y[n0 + 64 m + p]          m in [0,128) (M), p in [0,64) (N)
//   A[m, k] = xw[64 m + k]              Hankel view of the raw signal window
//   B[p, k] = h[p + Tp - k]             constant Toeplitz band of the taps
//
// The A operand is never materialised: stored linearly in shared memory with
// the 128-byte swizzle pre-applied, the 64-sample (128 B) row stride makes the
// Hankel matrix exactly a K-major SWIZZLE_128B UMMA operand whose start
// address advances 32 B per K step, across rows (the swizzle is a function of
// absolute smem address bits - verified on hardware by tools/umma_probe.cu).
//
// Precision: x = 2^-e (xh + 2^-11 xl), h = 2^-f (hh + 2^-11 hl), fp16 parts;
// y = 2^-(e+f) (xh hh + 2^-11 (xl hh + xh hl)) accumulated in fp32 in TMEM.
// e is chosen per tile, f per plan, so the maxima sit in [2^13, 2^14); the
// dropped xl hl term is 2^-22 relative.
//
// Pipeline (persistent, one CTA per SM, static tile schedule):
//   warp 0   bulk-copy producer: fp32 window -> smem (cp.async.bulk, mbarrier tx)
//   warp 1   MMA issuer (one thread): 3 x K/16 tcgen05.mma per tile
//   warps 2-9 convert window -> swizzled fp16 hi/lo operands
//   warps 10-13 epilogue: TMEM -> registers -> padded smem staging ->
//            coalesced stores (runs concurrently with the next conversion)
//   double buffers: fp32 window, fp16 operands, TMEM accumulators
//   (2 x 128 columns); one padded output staging tile.
#include <cuda_fp16.h>

#include "wp_internal.h"
#include "wp_tc.cuh"

namespace wpk {

namespace {

constexpr int kThreads = 448;     // 14 warps
constexpr int kConv = 256;        // converter threads (warps 2..9)
constexpr int kEpi = 128;         // epilogue threads (warps 10..13, one per TMEM lane quarter)
constexpr int kMaxQ = 10;         // float4 of the window per converter thread (W <= 10240)
constexpr int kStagePitch = 272;  // bytes per staged output row (256 + 16 pad)

__device__ __forceinline__ uint32_t swz128(uint32_t byte) { return byte ^ (((byte >> 7) & 7u) << 4); }

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1u << 16;                        // LBO (ignored for swizzled K-major)
    d |= (uint64_t)((1024u >> 4) & 0x3FFFu) << 32;  // SBO: 8 rows x 128 B
    d |= (uint64_t)1u << 46;                        // version
    d |= (uint64_t)2u << 61;                        // SWIZZLE_128B
    return d;
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct Geo {
    long long c, n0, start;  // channel, first output, window start sample
    long long lo, hi;        // bulk-copied sample range [lo, hi)
};

__device__ __forceinline__ Geo geo(const FirTcArgs &a, long long tile) {
    Geo g;
    g.c = tile % a.C;
    g.n0 = (tile / a.C) * (long long)TC_TOUT;
    g.start = g.n0 - a.Tp;
    g.lo = g.start > 0 ? g.start : 0;
    const long long nv = a.vec_x ? (a.N & ~3LL) : 0;  // vector-copyable prefix
    long long hi = g.start + a.W;
    if (hi > nv) hi = nv;
    g.hi = hi > g.lo ? hi : g.lo;
    return g;
}

}  // namespace

__global__ void __launch_bounds__(kThreads, 1) fir_tc_kernel(const FirTcArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment of the operand buffers (swizzle phase = address bits)
    // align by offsetting the __shared__ array itself (keeps the shared
    // address space visible to the compiler: LDS/STS, not generic LD/ST)
    unsigned char *smem = smem_raw + ((1024u - (wptc::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nk = a.K / 16;
    // ---- shared memory carve-up ----
    const uint32_t opBytes = ((uint32_t)a.W * 2u + 1023u) & ~1023u;  // one fp16 window
    const uint32_t inBytes = ((uint32_t)a.W * 4u + 1023u) & ~1023u;
    const uint32_t stgBytes = (128u * kStagePitch + 1023u) & ~1023u;
    const uint32_t bBytes = (uint32_t)((a.K + 63) / 64) * 8192u;  // one split of B
    // fp32 windows: double-buffered, or one buffer (a.nin == 1) when the taps' B image
    // needs the room (T > 129): the converters free it as soon as it is in registers
    unsigned char *inbuf0 = smem, *inbuf1 = smem + (a.nin > 1 ? inBytes : 0u);
    unsigned char *stg = smem + (uint32_t)a.nin * inBytes;  // output staging (padded rows)
    unsigned char *op = stg + stgBytes;       // [stage][hi, lo]
    unsigned char *bimg = op + 4 * opBytes;  // [hi, lo]
    unsigned long long *bars = reinterpret_cast<unsigned long long *>(bimg + 2 * bBytes);
    // bars: in_full[2], in_empty[2], op_full[2], op_empty[2], acc_full[2], acc_empty[2]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 12);
    float *red = reinterpret_cast<float *>(tmem_slot + 1);  // [8]
    float *scl = red + 8;                                    // per-stage scale [2]
    const uint32_t bar0 = wptc::smem_u32(bars);
    enum { IN_FULL = 0, IN_EMPTY = 1, OP_FULL = 2, OP_EMPTY = 3, ACC_FULL = 4, ACC_EMPTY = 5 };
#define BAR(kind, s) (bar0 + 8u * (uint32_t)(2 * (kind) + (s)))

    // ---- one-time setup ----
    if (warp == 0) wptc::tmem_alloc(wptc::smem_u32(tmem_slot), 256);
    if (tid == 32) {
        for (int s = 0; s < 2; ++s) {
            wptc::mbar_init(BAR(IN_FULL, s), 1);
            wptc::mbar_init(BAR(IN_EMPTY, s), 1);
            wptc::mbar_init(BAR(OP_FULL, s), 1);
            wptc::mbar_init(BAR(OP_EMPTY, s), 1);
            wptc::mbar_init(BAR(ACC_FULL, s), 1);
            wptc::mbar_init(BAR(ACC_EMPTY, s), kEpi);
        }
        wptc::mbar_fence_init();
    }
    for (int i = tid; i < (int)(2 * bBytes / 16); i += kThreads)
        reinterpret_cast<uint4 *>(bimg)[i] = reinterpret_cast<const uint4 *>(a.Bimg)[i];
    wptc::fence_proxy_async_smem();
    wptc::fence_before_sync();
    __syncthreads();
    wptc::fence_after_sync();
    const uint32_t tmem = *tmem_slot;
    const long long first = blockIdx.x, stride = gridDim.x;
    const int ntiles = first < a.total_tiles ? (int)((a.total_tiles - 1 - first) / stride + 1) : 0;

    if (warp == 0) {
        // ================= bulk-copy producer =================
        if (lane == 0) {
            for (int i = 0; i < ntiles; ++i) {
                const int s = a.nin > 1 ? (i & 1) : 0;
                const uint32_t par = (uint32_t)((a.nin > 1 ? (i >> 1) : i) & 1);
                wptc::mbar_wait(BAR(IN_EMPTY, s), par ^ 1u);
                const Geo g = geo(a, first + (long long)i * stride);
                const uint32_t bytes = (uint32_t)(4 * (g.hi - g.lo));
                unsigned char *dstb = s ? inbuf1 : inbuf0;
                if (bytes > 0) {
                    mbar_arrive_tx(BAR(IN_FULL, s), bytes);
                    const float *src = a.x + g.c * a.ldx + g.lo;
                    bulk_g2s(wptc::smem_u32(dstb) + 4u * (uint32_t)(g.lo - g.start), src, bytes, BAR(IN_FULL, s));
                } else {
                    mbar_arrive(BAR(IN_FULL, s));
                }
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer =================
        if (lane == 0) {
            const uint32_t idesc = wptc::idesc_f16(128, 64), idesc2 = wptc::idesc_f16(128, 128);
            const uint32_t op0 = wptc::smem_u32(op), b0 = wptc::smem_u32(bimg);
            for (int i = 0; i < ntiles; ++i) {
                const int s = i & 1;
                const uint32_t par = (uint32_t)((i >> 1) & 1);
                wptc::mbar_wait(BAR(OP_FULL, s), par);
                wptc::mbar_wait(BAR(ACC_EMPTY, s), par ^ 1u);
                wptc::fence_after_sync();
                const uint32_t dm = tmem + 128u * s, dc = dm + 64u;
                const uint32_t ahi = op0 + (2u * s) * opBytes, alo = ahi + opBytes;
                const uint64_t ah0 = desc_sw128(ahi), al0 = desc_sw128(alo);
#pragma unroll 1
                for (int kk = 0; kk < nk; ++kk) {
                    const uint64_t ka = 2u * kk;  // +32 B per K step (units of 16 B)
                    // B image [atom][hi rows | lo rows x 2^11]: one N = 128 MMA puts
                    // hi.hi into columns [0, 64) and hi.lo into [64, 128) = dc
                    const uint64_t bb = desc_sw128(b0 + 16384u * (kk >> 2) + 32u * (kk & 3));
                    wptc::mma_f16(dm, ah0 + ka, bb, idesc2, kk > 0);
                    wptc::mma_f16(dc, al0 + ka, bb, idesc, 1u);
                }
                wptc::mma_commit(BAR(OP_EMPTY, s));
                wptc::mma_commit(BAR(ACC_FULL, s));
            }
        }
    } else if (warp < 10) {
        // ================= converters (warps 2..9) =================
        const int ct = tid - 64;  // 0..255
        const int cw = ct >> 5;   // converter warp 0..7
        const int nq = a.W / 4;
        for (int i = 0; i < ntiles; ++i) {
            const int s = i & 1;
            const uint32_t par = (uint32_t)((i >> 1) & 1);
            const int si = a.nin > 1 ? s : 0;  // fp32 window buffer
            const uint32_t pari = (uint32_t)((a.nin > 1 ? (i >> 1) : i) & 1);
            const Geo g = geo(a, first + (long long)i * stride);
            const float *xr = a.x + g.c * a.ldx;
            wptc::mbar_wait(BAR(IN_FULL, si), pari);
            const float4 *in4 = reinterpret_cast<const float4 *>(si ? inbuf1 : inbuf0);
            float4 v[kMaxQ];
            float m = 0.f;
            const bool interior = g.start >= g.lo && g.start + a.W <= g.hi;
#pragma unroll
            for (int j = 0; j < kMaxQ; ++j) {
                const int q = ct + j * kConv;
                if (q < nq) {
                    const long long p0 = g.start + 4LL * q;
                    if (interior || (p0 >= g.lo && p0 + 4 <= g.hi)) {
                        v[j] = in4[q];
                    } else {
                        v[j].x = (p0 + 0 >= 0 && p0 + 0 < a.N) ? __ldg(xr + p0 + 0) : 0.f;
                        v[j].y = (p0 + 1 >= 0 && p0 + 1 < a.N) ? __ldg(xr + p0 + 1) : 0.f;
                        v[j].z = (p0 + 2 >= 0 && p0 + 2 < a.N) ? __ldg(xr + p0 + 2) : 0.f;
                        v[j].w = (p0 + 3 >= 0 && p0 + 3 < a.N) ? __ldg(xr + p0 + 3) : 0.f;
                    }
                    if (a.pre_gain != 1.f) {
                        v[j].x *= a.pre_gain; v[j].y *= a.pre_gain; v[j].z *= a.pre_gain; v[j].w *= a.pre_gain;
                    }
                    m = fmaxf(m, fmaxf(fmaxf(fabsf(v[j].x), fabsf(v[j].y)), fmaxf(fabsf(v[j].z), fabsf(v[j].w))));
                }
            }
            const unsigned mb = __reduce_max_sync(0xffffffffu, __float_as_uint(m));
            if (lane == 0) red[cw] = __uint_as_float(mb);
            named_sync(1, kConv);
            if (ct == 0) mbar_arrive(BAR(IN_EMPTY, si));  // window si is in registers: free it
            float tmax = red[0];
#pragma unroll
            for (int w = 1; w < 8; ++w) tmax = fmaxf(tmax, red[w]);
            int ex = 0;
            if (tmax > 0.f) frexpf(tmax, &ex);
            const float sc = ldexpf(1.f, tmax > 0.f ? 14 - ex : 0);
            if (ct == 0) scl[s] = sc;
            wptc::mbar_wait(BAR(OP_EMPTY, s), par ^ 1u);
            unsigned char *ohi = op + (2 * s) * opBytes, *olo = ohi + opBytes;
#pragma unroll
            for (int j = 0; j < kMaxQ; ++j) {
                const int q = ct + j * kConv;
                if (q < nq) {
                    const float2 f01 = make_float2(v[j].x * sc, v[j].y * sc);
                    const float2 f23 = make_float2(v[j].z * sc, v[j].w * sc);
                    const __half2 h01 = __float22half2_rn(f01), h23 = __float22half2_rn(f23);
                    const float2 b01 = __half22float2(h01), b23 = __half22float2(h23);
                    const __half2 l01 = __floats2half2_rn((f01.x - b01.x) * 2048.f, (f01.y - b01.y) * 2048.f);
                    const __half2 l23 = __floats2half2_rn((f23.x - b23.x) * 2048.f, (f23.y - b23.y) * 2048.f);
                    uint2 hv, lv;
                    hv.x = *reinterpret_cast<const uint32_t *>(&h01);
                    hv.y = *reinterpret_cast<const uint32_t *>(&h23);
                    lv.x = *reinterpret_cast<const uint32_t *>(&l01);
                    lv.y = *reinterpret_cast<const uint32_t *>(&l23);
                    const uint32_t off = swz128(8u * (uint32_t)q);
                    *reinterpret_cast<uint2 *>(ohi + off) = hv;
                    *reinterpret_cast<uint2 *>(olo + off) = lv;
                }
            }
            wptc::fence_proxy_async_smem();
            named_sync(1, kConv);
            if (ct == 0) mbar_arrive(BAR(OP_FULL, s));
        }
    } else {
        // ================= epilogue (warps 10..13) =================
        const int et = tid - 320;      // 0..127
        const int quarter = warp & 3;  // TMEM lane quarter this warp may access
        const int row = 32 * quarter + lane;
        for (int j = 0; j < ntiles; ++j) {
            const int s = j & 1;
            const uint32_t par = (uint32_t)((j >> 1) & 1);
            const Geo g = geo(a, first + (long long)j * stride);
            wptc::mbar_wait(BAR(ACC_FULL, s), par);
            wptc::fence_after_sync();
            const float osc = a.out_scale / scl[s];
            const uint32_t tbase = tmem + 128u * s + ((uint32_t)(32 * quarter) << 16);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float mn[4][8], cr[4][8];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    wptc::tmem_ld8(tbase + 32u * h + 8u * c, mn[c]);
                    wptc::tmem_ld8(tbase + 64u + 32u * h + 8u * c, cr[c]);
                }
                wptc::tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    float o[8];
#pragma unroll
                    for (int p = 0; p < 8; ++p) {
                        o[p] = fmaf(cr[c][p], 1.f / 2048.f, mn[c][p]) * osc;
#pragma unroll
                        for (int t = 0; t < MAXPOST; ++t)
                            if (t < a.n_post) o[p] *= a.post[t];
                    }
                    float4 *dst = reinterpret_cast<float4 *>(stg + row * kStagePitch + 4 * (32 * h + 8 * c));
                    dst[0] = make_float4(o[0], o[1], o[2], o[3]);
                    dst[1] = make_float4(o[4], o[5], o[6], o[7]);
                }
            }
            wptc::fence_before_sync();
            mbar_arrive(BAR(ACC_EMPTY, s));  // this thread's TMEM reads are done
            named_sync(2, kEpi);
            // coalesced copy-out of the 128 x 64 tile (contiguous outputs)
            float *yr = a.y + g.c * a.ldy + g.n0;
            const long long left = a.N - g.n0;
#pragma unroll 4
            for (int q = et; q < TC_TOUT / 4; q += kEpi) {
                const int r = q >> 4, c4 = q & 15;
                const float4 v = *reinterpret_cast<const float4 *>(stg + r * kStagePitch + 16 * c4);
                const long long p0 = 4LL * q;
                if (a.vec_y && p0 + 4 <= left) {
                    __stcs(reinterpret_cast<float4 *>(yr + p0), v);
                } else {
                    if (p0 + 0 < left) yr[p0 + 0] = v.x;
                    if (p0 + 1 < left) yr[p0 + 1] = v.y;
                    if (p0 + 2 < left) yr[p0 + 2] = v.z;
                    if (p0 + 3 < left) yr[p0 + 3] = v.w;
                }
            }
            named_sync(2, kEpi);  // staging consumed before the next tile writes it
        }
    }
#undef BAR
    wptc::fence_before_sync();
    __syncthreads();
    wptc::fence_after_sync();
    if (warp == 0) wptc::tmem_dealloc(tmem, 256);
}

}  // namespace wpk

namespace wp {

size_t fir_tc_smem_bytes(int W, int K, int nin) {
    const size_t opB = ((size_t)W * 2 + 1023) & ~size_t(1023);
    const size_t inB = ((size_t)W * 4 + 1023) & ~size_t(1023);
    const size_t stgB = ((size_t)128 * wpk::kStagePitch + 1023) & ~size_t(1023);
    const size_t bB = (size_t)((K + 63) / 64) * 8192;
    return (size_t)nin * inB + stgB + 4 * opB + 2 * bB + 12 * 8 + 64 + 1024;  // +1 KB alignment slack
}

cudaError_t launch_fir_tc(const wpk::FirTcArgs &a, int grid, size_t smem, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(wpk::fir_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    wpk::fir_tc_kernel<<<grid, wpk::kThreads, smem, st>>>(a);
    count_launch();
    return cudaGetLastError();
}

int fir_tc_occupancy(size_t smem) {
    if (cudaFuncSetAttribute(wpk::fir_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 0;
    return smem <= 227 * 1024 ? 1 : 0;  // persistent: one CTA per SM (256 TMEM columns)
}

}  // namespace wp
