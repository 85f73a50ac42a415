// Hardware probe (not product code): tcgen05.mma kind::tf32, M=128 N=64 K=8,
// K-major SWIZZLE_NONE operands with 32-byte rows
// offset(r,k) = (r/8)*256 + (k/4)*128 + (r%8)*16 + (k%4)*4  (LBO=128, SBO=256).
// Checks (1) the layout against a host GEMM on tf32-exact values and (2) the
// accuracy of a 3-way split product sum (the chain kernel's state term) that
// cancels against a large accumulator value.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tf32_probe tf32_probe.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
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

__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__host__ __device__ inline int off32(int r, int k) { return (r / 8) * 256 + (k / 4) * 128 + (r % 8) * 16 + (k % 4) * 4; }

// nA splits of A (each [128][8]) times nB splits of B ([64][8]), products (i, j)
// with i + j < 3, accumulated on top of an initial value loaded with a first
// MMA of A0 x B0 where A0 = diag-ish "init" operand.
__global__ void probe(const float *A, const float *B, int npairs, const int *pa, const int *pb, float *D) {
    __shared__ __align__(1024) unsigned char sa[3][4096];
    __shared__ __align__(1024) unsigned char sb[3][2048];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) unsigned long long bar;
    const int tid = threadIdx.x;
    for (int s = 0; s < 3; ++s) {
        for (int i = tid; i < 128 * 8; i += blockDim.x)
            *reinterpret_cast<float *>(&sa[s][off32(i / 8, i % 8)]) = A[s * 1024 + i];
        for (int i = tid; i < 64 * 8; i += blockDim.x)
            *reinterpret_cast<float *>(&sb[s][off32(i / 8, i % 8)]) = B[s * 512 + i];
    }
    if (tid < 32) wptc::tmem_alloc(wptc::smem_u32(&tslot), 64);
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
        for (int j = 0; j < npairs; ++j) {
            const uint64_t da = desc_none(wptc::smem_u32(sa[pa[j]]), 128, 256);
            const uint64_t db = desc_none(wptc::smem_u32(sb[pb[j]]), 128, 256);
            mma_tf32(tmem, da, db, idesc_tf32(128, 64), j > 0);
        }
        wptc::mma_commit(wptc::smem_u32(&bar));
    }
    wptc::mbar_wait(wptc::smem_u32(&bar), 0);
    wptc::fence_after_sync();
    const int w = tid >> 5, lane = tid & 31;
    for (int c = 0; c < 64; c += 8) {
        float v[8];
        wptc::tmem_ld8(tmem + ((uint32_t)(32 * w) << 16) + (uint32_t)c, v);
        wptc::tmem_wait_ld();
        for (int j = 0; j < 8; ++j) D[(32 * w + lane) * 64 + c + j] = v[j];
    }
    wptc::fence_before_sync();
    __syncthreads();
    wptc::fence_after_sync();
    if (tid < 32) wptc::tmem_dealloc(tmem, 64);
}

static float tf32r(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    u = (u + 0x1000u) & 0xFFFFE000u;
    memcpy(&f, &u, 4);
    return f;
}

int main() {
    srand(7);
    auto rnd = [] { return (double)rand() / RAND_MAX * 2.0 - 1.0; };
    float *dA, *dB, *dD;
    int *dpa, *dpb;
    cudaMalloc(&dA, 3 * 1024 * 4);
    cudaMalloc(&dB, 3 * 512 * 4);
    cudaMalloc(&dD, 128 * 64 * 4);
    cudaMalloc(&dpa, 64);
    cudaMalloc(&dpb, 64);
    int fails = 0;
    // (1) layout: one MMA of tf32-exact values vs host
    {
        std::vector<float> A(3 * 1024, 0.f), B(3 * 512, 0.f), D(128 * 64);
        for (int i = 0; i < 1024; ++i) A[i] = tf32r((float)rnd());
        for (int i = 0; i < 512; ++i) B[i] = tf32r((float)rnd());
        int pa[1] = {0}, pb[1] = {0};
        cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dpa, pa, 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dpb, pb, 4, cudaMemcpyHostToDevice);
        probe<<<1, 128>>>(dA, dB, 1, dpa, dpb, dD);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double worst = 0;
        for (int r = 0; r < 128; ++r)
            for (int n = 0; n < 64; ++n) {
                double ref = 0;
                for (int k = 0; k < 8; ++k) ref += (double)A[r * 8 + k] * B[n * 8 + k];
                worst = std::max(worst, std::fabs(ref - D[r * 64 + n]));
            }
        printf("tf32 layout probe: max abs err %.3g (%s) %s\n", worst, worst < 1e-5 ? "ok" : "FAIL", cudaGetErrorString(e));
        fails += worst >= 1e-5;
    }
    // (2) split state term: s (double, large, cancelling) x E, 3-way splits
    {
        std::vector<double> s(128 * 8), E(64 * 8);
        for (auto &v : s) v = rnd() * 3.0e4;
        for (auto &v : E) v = rnd() * 0.7;
        std::vector<float> A(3 * 1024), B(3 * 512), D(128 * 64);
        for (int i = 0; i < 1024; ++i) {
            const float a1 = tf32r((float)s[i]);
            const double r1 = s[i] - a1;
            const float a2 = tf32r((float)r1);
            const float a3 = tf32r((float)(r1 - a2));
            A[i] = a1, A[1024 + i] = a2, A[2048 + i] = a3;
        }
        for (int i = 0; i < 512; ++i) {
            const float b1 = tf32r((float)E[i]);
            const double r1 = E[i] - b1;
            const float b2 = tf32r((float)r1);
            const float b3 = tf32r((float)(r1 - b2));
            B[i] = b1, B[512 + i] = b2, B[1024 + i] = b3;
        }
        int pa[6] = {0, 0, 1, 0, 1, 2}, pb[6] = {0, 1, 0, 2, 1, 0};
        cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dpa, pa, 24, cudaMemcpyHostToDevice);
        cudaMemcpy(dpb, pb, 24, cudaMemcpyHostToDevice);
        probe<<<1, 128>>>(dA, dB, 6, dpa, dpb, dD);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double worst = 0, scale = 0, mag = 0;
        for (int r = 0; r < 128; ++r)
            for (int n = 0; n < 64; ++n) {
                double ref = 0, m = 0;
                for (int k = 0; k < 8; ++k) ref += s[r * 8 + k] * E[n * 8 + k], m += std::fabs(s[r * 8 + k] * E[n * 8 + k]);
                worst = std::max(worst, std::fabs(ref - D[r * 64 + n]));
                scale = std::max(scale, m);
                mag = std::max(mag, std::fabs(ref));
            }
        printf("tf32 3-split state term: max abs err %.3g, max sum|products| %.3g (rel %.3g), max |result| %.3g %s\n", worst,
               scale, worst / scale, mag, cudaGetErrorString(e));
        fails += worst / scale > 1e-6;
    }
    return fails;
}
