// Device helpers shared by the tensor-core kernels (chain_lb): tile geometry,
// SW128 UMMA descriptors, mbarrier / bulk-copy / TMEM wrappers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "wp_tc.cuh"

namespace wpk {

constexpr int CT_ROWS = 128;           // UMMA M: rows of a tile
constexpr int CT_TOUT = CT_ROWS * 64;  // outputs per tile (rows of 64 samples)
constexpr int CT_STG_PITCH = 144;      // epilogue staging row pitch: 32 floats + 16 B pad

// block-lower-triangular row r of a D x D transfer matrix (2 x 2 section blocks,
// cascade order) has entries q < lt_nj(D, r, false); lt_off packs the rows. A
// dense (globally balanced) basis has full rows.
__host__ __device__ constexpr int lt_nj(int D, int r, bool dense) { return dense ? D : 2 * ((r >> 1) + 1); }
__host__ __device__ constexpr int lt_off(int D, int r, bool dense) {
    return dense ? r * D : ((r & 1) ? 2 * ((r >> 1) + 1) * ((r >> 1) + 1) : 2 * (r >> 1) * ((r >> 1) + 1));
}
__host__ __device__ constexpr int lt_size(int D, bool dense) { return lt_off(D, D, dense); }

namespace ctd {

__device__ __forceinline__ uint32_t swz128(uint32_t byte) { return byte ^ (((byte >> 7) & 7u) << 4); }

// K-major SWIZZLE_128B UMMA descriptor (8-row groups 1024 B apart)
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1u << 16;
    d |= (uint64_t)((1024u >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1u << 46;
    d |= (uint64_t)2u << 61;
    return d;
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

// 32 lanes x 32 bit, 16 consecutive columns per thread
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

}  // namespace ctd

namespace c3d {

__device__ __forceinline__ void arrive_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

// window of one tile: start sample and the bulk-copyable range [lo, hi)
struct Win {
    long long c, n0, start, lo, hi;
};
__device__ __forceinline__ Win win(long long tile, long long C, long long N, int H, int W, int vec_x) {
    Win g;
    g.c = (long long)((unsigned)tile % (unsigned)C);
    g.n0 = (long long)((unsigned)tile / (unsigned)C) * (long long)CT_TOUT;
    g.start = g.n0 - H;
    g.lo = g.start > 0 ? g.start : 0;
    const long long nv = vec_x ? (N & ~3LL) : 0;
    long long hi = g.start + W;
    if (hi > nv) hi = nv;
    g.hi = hi > g.lo ? hi : g.lo;
    return g;
}

// Edge tile (signal start/end, an unaligned channel, or the non-vector tail): complete
// a window of W fp32 samples starting at sample `start` in place - zeros outside
// [0, N), samples the bulk copy did not cover ([lo, hi)) read from global - so the
// converters' register loads need no per-element bounds. Out of line and called
// before the window is register-resident: rare, and off the instruction cache's hot path.
static __device__ __noinline__ void fill_window(float *win, const float *xr, long long start, long long lo,
                                                long long hi, long long N, int W, int t, int nthreads) {
    for (int k = t; k < W; k += nthreads) {
        const long long p = start + k;
        if (p >= lo && p < hi) continue;  // bulk-copied
        win[k] = (p >= 0 && p < N) ? __ldg(xr + p) : 0.f;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // before the next bulk copy overwrites it
}

}  // namespace c3d

}  // namespace wpk
