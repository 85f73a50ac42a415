// Throughput probe (not product code): DFMA / FFMA lanes per clock per SM on
// this part, high ILP, full occupancy.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp_probe fp_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <typename T>
__global__ void fma_loop(T *out, int iters, T a, T b) {
    T r[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = T(threadIdx.x + i);
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] = fma(r[i], a, b);
    }
    T s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += r[i];
    if (s == T(-1.2345)) out[0] = s;
}

template <typename T>
void run(const char *name, int threads, int blocks_per_sm) {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    T *out;
    cudaMalloc(&out, sizeof(T));
    const int iters = 4096;
    fma_loop<T><<<sms * blocks_per_sm, threads>>>(out, 16, T(0.999), T(0.001));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    fma_loop<T><<<sms * blocks_per_sm, threads>>>(out, iters, T(0.999), T(0.001));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fmas = (double)sms * blocks_per_sm * threads * iters * 8;
    const double per_s = fmas / (ms * 1e-3);
    printf("%s threads=%d blocks/SM=%d: %.3f ms, %.2f T fma/s, %.1f fma/clk/SM at %.0f MHz (max clock)\n", name,
           threads, blocks_per_sm, ms, per_s / 1e12, per_s / sms / (clk * 1e3), clk / 1e3);
    cudaFree(out);
}

int main() {
    run<double>("DFMA", 256, 4);
    run<double>("DFMA", 128, 1);
    run<double>("DFMA", 32, 4);
    run<float>("FFMA", 256, 4);
    run<float>("FFMA", 32, 4);
    return 0;
}
