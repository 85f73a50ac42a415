// Hardware probe (not product code): tcgen05.mma kind::f16 with A from TMEM
// ("ts") vs A from shared memory ("ss"), M=128 K=16.
// (1) layout: A[128][16] fp16 written to TMEM with tcgen05.st 32x32b.x8
//     (lane = row, column c holds elements 2c (low half) and 2c+1), B[N][16]
//     K-major no-swizzle in smem (32-B rows: LBO = 128, SBO = 256); compare
//     with a host GEMM.
// (2) throughput: 2048 back-to-back MMAs per mode and N, cycles per MMA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o ts_probe ts_probe.cu
#include <cuda_fp16.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2504_08624_b200/csrc/wp_tc.cuh"

__device__ __forceinline__ uint64_t desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1u << 46;
    return d;
}

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

__host__ __device__ inline int off32(int r, int k2) {  // byte offset of element (r, k) with k2 = 2k bytes
    return (r / 8) * 256 + (k2 / 16) * 128 + (r % 8) * 16 + (k2 % 16);
}

template <int N>
__global__ void probe(const __half *A, const __half *B, float *D, int mode, int reps, long long *cyc, int nacc = 1) {
    __shared__ __align__(1024) unsigned char sa[128 * 32];
    __shared__ __align__(1024) unsigned char sb[N * 32];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) unsigned long long bar;
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 128 * 16; i += blockDim.x) {
        const int r = i / 16, k = i % 16;
        *reinterpret_cast<__half *>(&sa[off32(r, 2 * k)]) = A[i];
    }
    for (int i = tid; i < N * 16; i += blockDim.x) {
        const int r = i / 16, k = i % 16;
        *reinterpret_cast<__half *>(&sb[off32(r, 2 * k)]) = B[i];
    }
    if (w == 0) wptc::tmem_alloc(wptc::smem_u32(&tslot), 256);
    if (tid == 0) {
        wptc::mbar_init(wptc::smem_u32(&bar), 1);
        wptc::mbar_fence_init();
    }
    wptc::fence_proxy_async_smem();
    wptc::fence_before_sync();
    __syncthreads();
    wptc::fence_after_sync();
    const uint32_t tmem = tslot;
    const uint32_t ta = tmem + 128;  // A at columns [128, 136)
    {
        // thread = row 32 w + lane: 16 halves -> 8 columns
        const int r = 32 * w + lane;
        uint32_t v[8];
        for (int c = 0; c < 8; ++c) {
            const __half lo = A[r * 16 + 2 * c], hi = A[r * 16 + 2 * c + 1];
            v[c] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
        }
        tmem_st8(ta + ((uint32_t)(32 * w) << 16), v);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    wptc::fence_before_sync();
    __syncthreads();
    wptc::fence_after_sync();
    if (tid == 0) {
        const uint32_t idesc = wptc::idesc_f16(128, N);
        const uint64_t da = desc_none(wptc::smem_u32(sa), 128, 256);
        const uint64_t db = desc_none(wptc::smem_u32(sb), 128, 256);
        const long long t0 = clock64();
        for (int i = 0; i < reps; ++i) {
            // nacc independent accumulators (columns N * (i % nacc)); A stays at column 128+ only
            // for nacc * N <= 128
            const uint32_t dacc = tmem + (uint32_t)(N * (i % nacc));
            if (mode == 0)
                wptc::mma_f16(dacc, da, db, idesc, i >= nacc);
            else
                mma_ts(dacc, ta, db, idesc, i >= nacc);
        }
        wptc::mma_commit(wptc::smem_u32(&bar));
        wptc::mbar_wait(wptc::smem_u32(&bar), 0);
        *cyc = clock64() - t0;
    }
    __syncthreads();
    wptc::fence_after_sync();
    for (int c = 0; c < N; c += 8) {
        float v[8];
        wptc::tmem_ld8(tmem + ((uint32_t)(32 * w) << 16) + (uint32_t)c, v);
        wptc::tmem_wait_ld();
        for (int j = 0; j < 8; ++j) D[(32 * w + lane) * N + c + j] = v[j];
    }
    wptc::fence_before_sync();
    __syncthreads();
    wptc::fence_after_sync();
    if (w == 0) wptc::tmem_dealloc(tmem, 256);
}

template <int N>
int run() {
    std::vector<__half> A(128 * 16), B(N * 16);
    std::vector<float> Af(128 * 16), Bf(N * 16);
    srand(3);
    for (int i = 0; i < 128 * 16; ++i) A[i] = __float2half((float)((rand() % 17) - 8) / 8.f), Af[i] = __half2float(A[i]);
    for (int i = 0; i < N * 16; ++i) B[i] = __float2half((float)((rand() % 17) - 8) / 8.f), Bf[i] = __half2float(B[i]);
    __half *dA, *dB;
    float *dD;
    long long *dc;
    cudaMalloc(&dA, A.size() * 2);
    cudaMalloc(&dB, B.size() * 2);
    cudaMalloc(&dD, 128 * N * 4);
    cudaMalloc(&dc, 8);
    cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
    int fails = 0;
    for (int mode = 0; mode < 2; ++mode) {
        // correctness with one MMA
        probe<N><<<1, 128>>>(dA, dB, dD, mode, 1, dc);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> D(128 * N);
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double worst = 0;
        for (int r = 0; r < 128; ++r)
            for (int n = 0; n < N; ++n) {
                double ref = 0;
                for (int k = 0; k < 16; ++k) ref += (double)Af[r * 16 + k] * Bf[n * 16 + k];
                worst = std::max(worst, std::fabs(ref - D[r * N + n]));
            }
        // throughput
        long long cyc = 0;
        const int reps = 2048;
        probe<N><<<1, 128>>>(dA, dB, dD, mode, reps, dc);
        cudaError_t e2 = cudaDeviceSynchronize();
        cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
        printf("N=%d mode=%s: max err %.3g (%s), %.1f cycles per MMA  %s %s\n", N, mode ? "ts (A in TMEM)" : "ss (A in smem)",
               worst, worst < 1e-3 ? "ok" : "FAIL", (double)cyc / reps, cudaGetErrorString(e), cudaGetErrorString(e2));
        fails += worst >= 1e-3;
    }
    return fails;
}

// SW128 K-major operands as in chain_gemm: A 128 rows x 128 B, B N rows x 128 B
// (one 64-element K atom), 4 K steps of +32 B, repeated; nacc accumulators
template <int N>
__global__ void probe_sw(int reps, int nacc, long long *cyc) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char *sa = sm + ((1024u - (wptc::smem_u32(sm) & 1023u)) & 1023u);
    unsigned char *sb = sa + 128 * 128;
    __shared__ uint32_t tslot;
    __shared__ __align__(8) unsigned long long bar;
    const int tid = threadIdx.x, w = tid >> 5;
    for (int i = tid; i < (128 + N) * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sa)[i] = 0x3c003c00u;
    if (w == 0) wptc::tmem_alloc(wptc::smem_u32(&tslot), 512);
    if (tid == 0) {
        wptc::mbar_init(wptc::smem_u32(&bar), 1);
        wptc::mbar_fence_init();
    }
    wptc::fence_proxy_async_smem();
    wptc::fence_before_sync();
    __syncthreads();
    wptc::fence_after_sync();
    const uint32_t tmem = tslot;
    if (tid == 0) {
        const uint32_t idesc = wptc::idesc_f16(128, N);
        const uint32_t a0 = wptc::smem_u32(sa), b0 = wptc::smem_u32(sb);
        const long long t0 = clock64();
#pragma unroll 1
        for (int i = 0; i < reps; i += 4) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const uint64_t da = wptc::umma_desc(a0, 16, 1024) | ((uint64_t)2 << 61);
                const uint64_t db = wptc::umma_desc(b0, 16, 1024) | ((uint64_t)2 << 61);
                const uint32_t acc = (uint32_t)(nacc > 1 ? (N * ((i / 4 + kk) & (nacc - 1))) : 0);
                wptc::mma_f16(tmem + acc, da + 2u * kk, db + 2u * kk, idesc, 1u);
            }
        }
        wptc::mma_commit(wptc::smem_u32(&bar));
        wptc::mbar_wait(wptc::smem_u32(&bar), 0);
        *cyc = clock64() - t0;
    }
    wptc::fence_before_sync();
    __syncthreads();
    wptc::fence_after_sync();
    if (w == 0) wptc::tmem_dealloc(tmem, 512);
}

template <int N>
void run_sw(int nacc) {
    long long *dc;
    cudaMalloc(&dc, 8);
    const int smem = (128 + N) * 128 + 1024;
    cudaFuncSetAttribute(probe_sw<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int reps = 4096;
    probe_sw<N><<<1, 128, smem>>>(reps, nacc, dc);
    cudaError_t e = cudaDeviceSynchronize();
    long long cyc = 0;
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    printf("SW128 N=%d, %d accumulators: %.1f cycles per MMA %s\n", N, nacc, (double)cyc / reps, cudaGetErrorString(e));
}

// tf32 K=8 MMAs (M=128, N=64): no-swizzle 32-B rows vs SWIZZLE_32B K-major
__device__ __forceinline__ void mma_tf32p(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(a), "l"(b), "r"(idesc) : "memory");
}
__global__ void probe_tf32(int reps, int swz, long long *cyc) {
    __shared__ __align__(1024) unsigned char sa[128 * 32];
    __shared__ __align__(1024) unsigned char sb[64 * 32];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) unsigned long long bar;
    const int tid = threadIdx.x, w = tid >> 5;
    for (int i = tid; i < 128 * 8; i += blockDim.x) reinterpret_cast<float *>(sa)[i] = 1.0f;
    for (int i = tid; i < 64 * 8; i += blockDim.x) reinterpret_cast<float *>(sb)[i] = 1.0f;
    if (w == 0) wptc::tmem_alloc(wptc::smem_u32(&tslot), 64);
    if (tid == 0) {
        wptc::mbar_init(wptc::smem_u32(&bar), 1);
        wptc::mbar_fence_init();
    }
    wptc::fence_proxy_async_smem();
    wptc::fence_before_sync();
    __syncthreads();
    wptc::fence_after_sync();
    const uint32_t tmem = tslot;
    if (tid == 0) {
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        uint64_t da, db;
        if (swz) {
            da = wptc::umma_desc(wptc::smem_u32(sa), 16, 256) | ((uint64_t)6 << 61);
            db = wptc::umma_desc(wptc::smem_u32(sb), 16, 256) | ((uint64_t)6 << 61);
        } else {
            da = desc_none(wptc::smem_u32(sa), 128, 256);
            db = desc_none(wptc::smem_u32(sb), 128, 256);
        }
        const long long t0 = clock64();
#pragma unroll 1
        for (int i = 0; i < reps; ++i) mma_tf32p(tmem, da, db, idesc);
        wptc::mma_commit(wptc::smem_u32(&bar));
        wptc::mbar_wait(wptc::smem_u32(&bar), 0);
        *cyc = clock64() - t0;
    }
    wptc::fence_before_sync();
    __syncthreads();
    wptc::fence_after_sync();
    if (w == 0) wptc::tmem_dealloc(tmem, 64);
}

void run_tf32(int swz) {
    long long *dc;
    cudaMalloc(&dc, 8);
    const int reps = 4096;
    probe_tf32<<<1, 128>>>(reps, swz, dc);
    cudaError_t e = cudaDeviceSynchronize();
    long long cyc = 0;
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    printf("tf32 K=8 N=64 %s: %.1f cycles per MMA %s\n", swz ? "SW32" : "no-swizzle", (double)cyc / reps, cudaGetErrorString(e));
}

template <int N>
void run_acc(int nacc) {
    __half *dA, *dB;
    float *dD;
    long long *dc;
    cudaMalloc(&dA, 128 * 16 * 2);
    cudaMalloc(&dB, N * 16 * 2);
    cudaMalloc(&dD, 128 * N * 4);
    cudaMalloc(&dc, 8);
    cudaMemset(dA, 0, 128 * 16 * 2);
    cudaMemset(dB, 0, N * 16 * 2);
    const int reps = 2048;
    long long cyc = 0;
    probe<N><<<1, 128>>>(dA, dB, dD, 0, reps, dc, nacc);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    printf("N=%d ss, %d independent accumulators: %.1f cycles per MMA %s\n", N, nacc, (double)cyc / reps, cudaGetErrorString(e));
}

int main() {
    int f = run<64>() + run<128>();
    run_tf32(0);
    run_tf32(1);
    run_sw<64>(1);
    run_sw<64>(2);
    run_sw<128>(1);
    run_sw<128>(2);
    run_sw<256>(1);
    run_sw<64>(4);
    return f;
}
