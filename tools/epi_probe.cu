// Probe (not product code): the chain kernel's epilogue work per tile in
// isolation - 4 warps (one row each per thread), fp32 double-single state term
// from smem tables, staging, coalesced stores - to measure its intrinsic cost.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o epi_probe epi_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int D = 8;
constexpr int PITCH = 144;

__global__ void __launch_bounds__(128, 1) epi(float *y, int tiles, int mode) {
    __shared__ __align__(16) float Esh[D * 64], Esl[D * 64];
    __shared__ __align__(16) unsigned char stg[4 * 32 * PITCH];
    const int tid = threadIdx.x, lane = tid & 31, wq = tid >> 5;
    for (int i = tid; i < D * 64; i += 128) {
        Esh[i] = 0.001f * i;
        Esl[i] = 1e-9f * i;
    }
    __syncthreads();
    float sh[D], sl[D];
    for (int d = 0; d < D; ++d) {
        sh[d] = 0.1f * (d + lane);
        sl[d] = 1e-8f * d;
    }
    unsigned char *mystg = stg + wq * 32 * PITCH;
    for (int t = 0; t < tiles; ++t) {
        float *yr = y + ((size_t)(blockIdx.x * tiles + t) * 8192);
#pragma unroll 1
        for (int ch = 0; ch < 4; ++ch) {
            const int h = ch >> 1, hh = ch & 1;
            float acc[16], cor[16];
#pragma unroll
            for (int pp = 0; pp < 16; ++pp) {
                acc[pp] = 0.5f * (pp + t + lane);
                cor[pp] = 0.f;
            }
            if (mode & 1) {
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    const float4 *eh = reinterpret_cast<const float4 *>(Esh + d * 64 + 16 * ch);
                    const float4 *el = reinterpret_cast<const float4 *>(Esl + d * 64 + 16 * ch);
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        const float4 h4 = eh[q4], l4 = el[q4];
                        const float hv[4] = {h4.x, h4.y, h4.z, h4.w}, lv4[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            acc[4 * q4 + u] = fmaf(hv[u], sh[d], acc[4 * q4 + u]);
                            cor[4 * q4 + u] = fmaf(lv4[u], sh[d], fmaf(hv[u], sl[d], cor[4 * q4 + u]));
                        }
                    }
                }
            }
            float4 *dst = reinterpret_cast<float4 *>(mystg + lane * PITCH + 64 * hh);
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
                dst[q4] = make_float4(acc[4 * q4] + cor[4 * q4], acc[4 * q4 + 1] + cor[4 * q4 + 1],
                                      acc[4 * q4 + 2] + cor[4 * q4 + 2], acc[4 * q4 + 3] + cor[4 * q4 + 3]);
            if (hh == 1 && (mode & 2)) {
                __syncwarp();
#pragma unroll 1
                for (int r = 0; r < 8; ++r) {
                    const int q = lane + 32 * r;
                    const int rr = q >> 3, c4 = q & 7;
                    const float4 v = *reinterpret_cast<const float4 *>(mystg + rr * PITCH + 16 * c4);
                    const int o = 64 * (32 * wq + rr) + 32 * h + 4 * c4;
                    __stcs(reinterpret_cast<float4 *>(yr + o), v);
                }
                __syncwarp();
            }
        }
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int tiles = 200;
    float *y;
    cudaMalloc(&y, (size_t)sms * tiles * 8192 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 4; ++mode) {
        epi<<<sms, 128>>>(y, 4, mode);
        cudaEventRecord(e0);
        epi<<<sms, 128>>>(y, tiles, mode);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("mode %d (state=%d stores=%d): %.3f us per tile per SM\n", mode, mode & 1, (mode >> 1) & 1,
               ms * 1e3 / tiles);
    }
    return 0;
}
