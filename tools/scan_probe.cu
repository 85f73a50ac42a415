// Probe (not product code): the chain kernel's row scan per tile in isolation
// - 4 warps, one row per thread, fp64 D=8: e combine, Kogge-Stone over rows,
// CTA prefix, row prefix via M^lane - to measure its intrinsic cost.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scan_probe scan_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2504_08624_b200/csrc/wp_common.cuh"  // (round-1 probe: built against wp_chain_tc.cuh, since removed)

using namespace wpk;
constexpr int D = 8;

__global__ void __launch_bounds__(128, 1) scanp(double *out, int tiles, int mode) {
    __shared__ double Ps[5 * D * D], Ws[4 * D * D], gsm[lt_size(D) * 32], wi[4 * D], sbuf[128 * D];
    const int tid = threadIdx.x, lane = tid & 31, wq = tid >> 5;
    for (int i = tid; i < 5 * D * D; i += 128) Ps[i] = 0.01 * (i % 7) * ((i % D) <= (i / D) % D ? 1 : 0);
    for (int i = tid; i < 4 * D * D; i += 128) Ws[i] = 0.02 * (i % 5);
    for (int i = tid; i < lt_size(D) * 32; i += 128) gsm[i] = 0.03 * (i % 11);
    __syncthreads();
    double acc_out = 0;
    for (int t = 0; t < tiles; ++t) {
        double e[D];
        for (int d = 0; d < D; ++d) e[d] = 1.0 + 0.001 * (d + lane + t);
        double incl[D];
#pragma unroll
        for (int d = 0; d < D; ++d) incl[d] = e[d];
        if (mode & 1) {
#pragma unroll 1
            for (int stp = 0; stp < 5; ++stp) {
                const int off = 1 << stp;
                double prev[D];
#pragma unroll
                for (int d = 0; d < D; ++d) prev[d] = __shfl_up_sync(0xffffffffu, incl[d], off);
                if (lane >= off) ctd::matvec_tree<D, double>(incl, prev, [&](int r, int q) { return Ps[(stp * D + r) * D + q]; });
            }
        }
        double Lm[D];
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const double v = __shfl_up_sync(0xffffffffu, incl[d], 1);
            Lm[d] = lane == 0 ? 0.0 : v;
        }
        if (lane == 31)
            for (int d = 0; d < D; ++d) wi[wq * D + d] = incl[d];
        __syncthreads();
        if (mode & 2) {
            double wc[D];
#pragma unroll
            for (int d = 0; d < D; ++d) wc[d] = 0.0;
#pragma unroll
            for (int u = 0; u < 3; ++u) {
                if (u < wq) {
                    double iu[D];
#pragma unroll
                    for (int d = 0; d < D; ++d) iu[d] = wi[u * D + d];
                    const int pw = wq - 1 - u;
                    ctd::matvec_tree<D, double>(wc, iu, [&](int r, int q) { return Ws[(pw * D + r) * D + q]; });
                }
            }
            ctd::matvec_tree<D, double>(Lm, wc, [&](int r, int q) { return gsm[(lt_off(r) + q) * 32 + lane]; });
        }
        for (int d = 0; d < D; ++d) sbuf[tid * D + d] = Lm[d];
        __syncthreads();
        acc_out += sbuf[((tid + 1) & 127) * D];
    }
    if (acc_out == -1.0) out[0] = acc_out;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *o;
    cudaMalloc(&o, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int tiles = 400;
    for (int mode = 0; mode < 4; ++mode) {
        scanp<<<sms, 128>>>(o, 4, mode);
        cudaEventRecord(e0);
        scanp<<<sms, 128>>>(o, tiles, mode);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("mode %d (kogge=%d cta=%d): %.3f us per tile\n", mode, mode & 1, (mode >> 1) & 1, ms * 1e3 / tiles);
    }
    return 0;
}
