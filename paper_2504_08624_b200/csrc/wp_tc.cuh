// Thin inline-PTX wrappers for the sm_100a tensor-core path: tcgen05.mma /
// commit / ld, TMEM allocation, mbarriers and UMMA shared-memory descriptors.
// Field layouts follow the PTX ISA (tcgen05 "Shared memory descriptor" and
// "Instruction descriptor" for kind::f16).
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>

namespace wptc {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// UMMA smem descriptor, no swizzle ("interleave"), K-major canonical layout
// ((8,m),2):((16B,SBO),LBO): 8 rows of 16 bytes form a core matrix.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1u << 46;  // descriptor version for tcgen05
    // base offset 0, lbo mode 0, layout type 0 (SWIZZLE_NONE)
    return d;
}

// kind::f16 instruction descriptor: fp16 A/B, fp32 accumulate, both K-major.
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
    return (1u << 4)                       // D format F32
           | (0u << 7) | (0u << 10)        // A, B format F16
           | ((uint32_t)(N >> 3) << 17)    // N >> 3
           | ((uint32_t)(M >> 4) << 24);   // M >> 4
}

__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t mbar_saddr) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar_saddr)
                 : "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t dst_saddr, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_saddr), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

__device__ __forceinline__ void fence_before_sync() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after_sync() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// make generic-proxy st.shared visible to the tensor-core (async) proxy
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_init(uint32_t saddr, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// Blocking wait on an mbarrier phase. The suspend-time hint lets the waiting
// warp sleep in hardware until the phase completes instead of re-polling the
// barrier (spinning warps otherwise eat issue slots and shared-memory pipe
// bandwidth that the producer warps need). Watchdog: a wait that has not
// completed after 10 s traps, so a pipeline bug aborts the launch with an
// error instead of hanging the device.
__device__ __forceinline__ bool mbar_try(uint32_t saddr, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred done;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, done;\n\t}\n"
        : "=r"(ok)
        : "r"(saddr), "r"(parity), "r"(1000000u)
        : "memory");
    return ok != 0;
}
// non-blocking probe of an mbarrier phase
__device__ __forceinline__ bool mbar_test(uint32_t saddr, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred done;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 done, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, done;\n\t}\n"
        : "=r"(ok)
        : "r"(saddr), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ unsigned long long now_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void mbar_wait(uint32_t saddr, uint32_t parity) {
    if (mbar_try(saddr, parity)) return;
    const unsigned long long t0 = now_ns();
    while (!mbar_try(saddr, parity)) {
        if (now_ns() - t0 > 10000000000ull) asm volatile("trap;");
    }
}
// The same with an exponential nanosleep back-off (capped at MAXNS) between
// polls: the suspend hint above returns early whenever any barrier of the CTA
// changes, so a warp that is far ahead would otherwise spin and take issue
// slots from the warps it is waiting for.
template <unsigned MAXNS>
__device__ __forceinline__ void mbar_wait_sleep(uint32_t saddr, uint32_t parity) {
    if (mbar_try(saddr, parity)) return;
    const unsigned long long t0 = now_ns();
    unsigned ns = 32;
    while (!mbar_try(saddr, parity)) {
        __nanosleep(ns);
        ns = ns < MAXNS ? 2 * ns : MAXNS;
        if (now_ns() - t0 > 10000000000ull) asm volatile("trap;");
    }
}

// 32 lanes x 32 bit, 8 consecutive columns per thread
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

}  // namespace wptc
