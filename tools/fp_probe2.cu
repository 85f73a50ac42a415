// Throughput probe (not product code): F2F f32<->f64 conversion, I2F.F64,
// uniform-address LDS.128, per SM per clock. Build:
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp_probe2 fp_probe2.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void cvt_loop(float *out, int iters) {
    float f[8];
    for (int i = 0; i < 8; ++i) f[i] = threadIdx.x * 0.001f + i;
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            double d = (double)f[i];
            d = d * 1.0000001;
            f[i] = (float)d;
        }
    }
    float s = 0;
    for (int i = 0; i < 8; ++i) s += f[i];
    if (s == -1.f) out[0] = s;
}

__global__ void i2f_loop(double *out, int iters) {
    int v[8];
    double acc[8];
    for (int i = 0; i < 8; ++i) { v[i] = threadIdx.x + i; acc[i] = 0; }
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int i = 0; i < 8; ++i) { acc[i] = acc[i] * 256.0 + (double)v[i]; v[i] += 3; }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == -1.0) out[0] = s;
}

__global__ void lds_loop(double *out, int iters) {
    __shared__ double tab[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) tab[i] = i * 0.5;
    __syncthreads();
    double acc[16];
    for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x;
    for (int k = 0; k < iters; ++k) {
        const double *e = tab + (k & 31) * 32;
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fma(e[i], 1.0000001, acc[i]);
    }
    double s = 0;
    for (int i = 0; i < 16; ++i) s += acc[i];
    if (s == -1.0) out[0] = s;
}

template <typename K, typename T>
void run(const char *name, K kern, int threads, int per_iter_ops) {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    T *out;
    cudaMalloc(&out, sizeof(T));
    kern<<<sms, threads>>>(out, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    cudaEventRecord(e0);
    kern<<<sms, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)sms * threads * iters * per_iter_ops;
    printf("%s threads/SM=%d: %.1f ops/clk/SM (%.3f ms)\n", name, threads, ops / (ms * 1e-3) / sms / (clk * 1e3), ms);
    cudaFree(out);
}

int main() {
    run<decltype(&cvt_loop), float>("F2F f32->f64->f32 pairs", cvt_loop, 128, 8);
    run<decltype(&cvt_loop), float>("F2F f32->f64->f32 pairs", cvt_loop, 512, 8);
    run<decltype(&i2f_loop), double>("I2F.F64 + DFMA", i2f_loop, 128, 8);
    run<decltype(&lds_loop), double>("LDS uniform + DFMA (per DFMA)", lds_loop, 128, 16);
    run<decltype(&lds_loop), double>("LDS uniform + DFMA (per DFMA)", lds_loop, 512, 16);
    return 0;
}
