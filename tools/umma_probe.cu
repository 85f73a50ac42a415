// Hardware probe (not part of the product): does a K-major SWIZZLE_128B UMMA
// descriptor over a *linear, pre-swizzled* fp16 signal give the Hankel matrix
// A[m,k] = x[64 m + k] when the start address is advanced by 2k bytes
// (crossing 128-byte rows), and which "base offset" setting is required?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_probe umma_probe.cu
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t sbo, uint32_t base_off) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;                       // LBO (unused for swizzled K-major), 16 B
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;                       // version
    d |= (uint64_t)(base_off & 7) << 49;
    d |= (uint64_t)2 << 61;                       // SWIZZLE_128B
    return d;
}

__device__ __forceinline__ uint32_t swz128(uint32_t byte) { return byte ^ (((byte >> 7) & 7) << 4); }

// x: 16384 fp16 values, B: [N=64][K=64*KA] taps image (row p, k) dense fp32 -> converted here
__global__ void probe(const float *x, const float *Bm, float *D, int K, int mode) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __half *xs = reinterpret_cast<__half *>(smem);            // 32 KB signal, 1024-aligned
    unsigned char *bs = smem + 32768;                           // B image
    __shared__ uint32_t tslot;
    __shared__ __align__(8) unsigned long long mbar;
    const int tid = threadIdx.x;
    // signal, pre-swizzled relative to the 1024-aligned base
    for (int s = tid; s < 16384; s += blockDim.x) {
        uint32_t b = swz128(2u * s);
        *reinterpret_cast<__half *>(smem + b) = __float2half_rn(x[s]);
    }
    // B: K atoms of 64; atom a holds rows p (64) x 128 B, swizzled per 1024 B group
    const int KA = K / 64;
    for (int i = tid; i < 64 * K; i += blockDim.x) {
        int p = i / K, k = i % K;
        int a = k / 64, kk = k % 64;
        uint32_t logical = a * 8192 + p * 128 + kk * 2;
        *reinterpret_cast<__half *>(bs + swz128(logical)) = __float2half_rn(Bm[p * K + k]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    const uint32_t idesc = (1u << 4) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
    if (tid == 0) {
        const uint32_t xa = smem_u32(xs), ba = smem_u32(bs);
        for (int k16 = 0; k16 < K / 16; ++k16) {
            const uint32_t a0 = xa + 32u * k16;
            const uint32_t b0 = ba + 8192u * (k16 / 4) + 32u * (k16 % 4);
            uint32_t boa = mode == 1 ? ((a0 >> 7) & 7) : 0;
            const uint64_t ad = desc_sw128(a0, 1024, boa);
            const uint64_t bd = desc_sw128(b0, 1024, 0);
            const uint32_t acc = k16 > 0;
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                         "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
    }
    asm volatile("{\n\t.reg .pred done;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 done, [%0], 0;\n\t@!done bra W;\n\t}\n" ::"r"(smem_u32(&mbar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int warp = tid / 32, lane = tid % 32;
    for (int c0 = 0; c0 < 64; c0 += 8) {
        uint32_t r[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(tmem + ((32u * warp) << 16) + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int i = 0; i < 8; ++i) D[(32 * warp + lane) * 64 + c0 + i] = __uint_as_float(r[i]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

int main() {
    const int K = 192;  // three 64-element K atoms -> start address crosses rows
    std::vector<float> x(16384), B(64 * K), D(128 * 64);
    srand(1);
    for (auto &v : x) v = (float)((rand() % 17) - 8);  // small integers: exact in fp16 and fp32 sums
    for (auto &v : B) v = (float)((rand() % 5) - 2);
    float *dx, *dB, *dD;
    cudaMalloc(&dx, x.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 64 * K * 2 + 1024);
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(dD, 0, D.size() * 4);
        probe<<<1, 128, 32768 + 64 * K * 2 + 1024>>>(dx, dB, dD, K, mode);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("mode %d: CUDA error %s\n", mode, cudaGetErrorString(e)); return 1; }
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double maxerr = 0; int bad = 0;
        for (int m = 0; m < 128; ++m)
            for (int p = 0; p < 64; ++p) {
                double ref = 0;
                for (int k = 0; k < K; ++k) ref += (double)x[64 * m + k] * B[p * K + k];
                double err = fabs(ref - D[m * 64 + p]);
                if (err > 0.5) ++bad;
                maxerr = fmax(maxerr, err);
            }
        printf("mode %d (base_offset %s): max err %g, bad %d / %d\n", mode, mode ? "=(addr>>7)&7" : "=0", maxerr, bad, 128 * 64);
    }
    return 0;
}
