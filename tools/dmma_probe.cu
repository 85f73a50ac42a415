// Hardware probe (not product code): fp64 throughput of mma.sync m8n8k4 f64
// (DMMA) vs DFMA on this part, 148 x 8 warps of independent work.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o dmma_probe dmma_probe.cu
#include <cstdio>

__global__ void dmma_kernel(double *out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.5, c[8][2];
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_kernel(double *out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.5, c[16];
    for (int i = 0; i < 16; ++i) c[i] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) c[i] = fma(a, b, c[i]);
    }
    double s = 0;
    for (int i = 0; i < 16; ++i) s += c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    double *d;
    cudaMalloc(&d, 148 * 256 * 8 * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int rep = 0; rep < 2; ++rep) {
        float ms = 0;
        cudaEventRecord(e0);
        dmma_kernel<<<148 * 2, 256>>>(d, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        // per warp per iter: 8 MMAs x 8x8x4 = 2048 FMA
        const double fma_dmma = 148.0 * 2 * 8 * (double)iters * 8 * 256;
        printf("DMMA m8n8k4: %.2f ms, %.1f TFMA/s (%.1f TFLOP/s)  %s\n", ms, fma_dmma / ms / 1e9, 2 * fma_dmma / ms / 1e9,
               cudaGetErrorString(cudaGetLastError()));
        cudaEventRecord(e0);
        dfma_kernel<<<148 * 2, 256>>>(d, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double fma_dfma = 148.0 * 2 * 256 * (double)iters * 16;
        printf("DFMA:        %.2f ms, %.1f TFMA/s (%.1f TFLOP/s)\n", ms, fma_dfma / ms / 1e9, 2 * fma_dfma / ms / 1e9);
    }
    return 0;
}
