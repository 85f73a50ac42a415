// Hardware probe (not product code): tcgen05.mma kind::i8, M=128 N=16 K=64
// (two K=32 instructions) from K-major SWIZZLE_NONE operands
// offset(r,k) = (r/8)*512 + (k/16)*128 + (r%8)*16 + k%16  (LBO=128, SBO=512),
// for all four signedness combinations; int32 accumulate, compared with a
// host GEMM. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o i8_probe i8_probe.cu
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

__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, int as, int bs) {
    return (2u << 4) | ((uint32_t)as << 7) | ((uint32_t)bs << 10) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}

__global__ void probe(const int8_t *A, const int8_t *B, int *D, int as, int bs) {
    __shared__ __align__(1024) unsigned char sa[128 * 64];
    __shared__ __align__(1024) unsigned char sb[16 * 64];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) unsigned long long bar;
    const int tid = threadIdx.x;
    for (int i = tid; i < 128 * 64; i += blockDim.x) {
        const int r = i / 64, k = i % 64;
        sa[(r / 8) * 512 + (k / 16) * 128 + (r % 8) * 16 + k % 16] = (unsigned char)A[i];
    }
    for (int i = tid; i < 16 * 64; i += blockDim.x) {
        const int r = i / 64, k = i % 64;
        sb[(r / 8) * 512 + (k / 16) * 128 + (r % 8) * 16 + k % 16] = (unsigned char)B[i];
    }
    if (tid < 32) wptc::tmem_alloc(wptc::smem_u32(&tslot), 32);
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
        const uint32_t id = idesc_i8(128, 16, as, bs);
        for (int kh = 0; kh < 2; ++kh) {
            const uint64_t da = desc_none(wptc::smem_u32(sa) + 256u * kh, 128, 512);
            const uint64_t db = desc_none(wptc::smem_u32(sb) + 256u * kh, 128, 512);
            mma_i8(tmem, da, db, id, kh);
        }
        wptc::mma_commit(wptc::smem_u32(&bar));
    }
    wptc::mbar_wait(wptc::smem_u32(&bar), 0);
    wptc::fence_after_sync();
    // warp w reads lanes 32w..32w+31
    const int w = tid >> 5, lane = tid & 31;
    float v[8], u[8];
    wptc::tmem_ld8(tmem + ((uint32_t)(32 * w) << 16), v);
    wptc::tmem_ld8(tmem + ((uint32_t)(32 * w) << 16) + 8u, u);
    wptc::tmem_wait_ld();
    const int row = 32 * w + lane;
    for (int j = 0; j < 8; ++j) {
        D[row * 16 + j] = __float_as_int(v[j]);
        D[row * 16 + 8 + j] = __float_as_int(u[j]);
    }
    wptc::fence_before_sync();
    __syncthreads();
    wptc::fence_after_sync();
    if (tid < 32) wptc::tmem_dealloc(tmem, 32);
}

int main() {
    std::vector<int8_t> A(128 * 64), B(16 * 64);
    srand(1);
    for (auto &a : A) a = (int8_t)(rand() & 255);
    for (auto &b : B) b = (int8_t)(rand() & 255);
    int8_t *dA, *dB;
    int *dD;
    cudaMalloc(&dA, A.size());
    cudaMalloc(&dB, B.size());
    cudaMalloc(&dD, 128 * 16 * 4);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
    int fails = 0;
    for (int as = 0; as < 2; ++as)
        for (int bs = 0; bs < 2; ++bs) {
            cudaMemset(dD, 0, 128 * 16 * 4);
            probe<<<1, 128>>>(dA, dB, dD, as, bs);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<int> D(128 * 16);
            cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
            int bad = 0;
            for (int r = 0; r < 128; ++r)
                for (int n = 0; n < 16; ++n) {
                    long long ref = 0;
                    for (int k = 0; k < 64; ++k) {
                        const int a = as ? (int)A[r * 64 + k] : (int)(uint8_t)A[r * 64 + k];
                        const int b = bs ? (int)B[n * 64 + k] : (int)(uint8_t)B[n * 64 + k];
                        ref += (long long)a * b;
                    }
                    if (ref != D[r * 16 + n]) {
                        if (bad < 3) printf("  mismatch r=%d n=%d got %d want %lld\n", r, n, D[r * 16 + n], ref);
                        ++bad;
                    }
                }
            printf("i8 probe a_signed=%d b_signed=%d: %s (%d mismatches) %s\n", as, bs, bad ? "FAIL" : "ok", bad,
                   cudaGetErrorString(e));
            fails += bad != 0;
        }
    return fails;
}
