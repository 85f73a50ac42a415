// Signal source and reduction kernels:
//  * white_noise: counter-based splitmix64 + Box-Muller in float64, the
//    generator of wave.py:103-168 (pair j draws counters 2j, 2j+1; values depend
//    only on (seed, flat channel-major position)), rounded to float32.
//  * peak_abs / scale_by_peak: the Normalize stage (device-side max, no host
//    round trip).
#include <math.h>

#include "wp_internal.h"

namespace wpk {

__device__ __forceinline__ unsigned long long splitmix(unsigned long long seed, unsigned long long ctr) {
    unsigned long long z = seed + ctr * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void white_noise_kernel(float *y, long long C, long long N, long long ld, unsigned long long seed) {
    const long long total = C * N;
    const long long pairs = (total + 1) / 2;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < pairs; j += stride) {
        const unsigned long long b0 = splitmix(seed, (unsigned long long)(2 * j + 1));
        const unsigned long long b1 = splitmix(seed, (unsigned long long)(2 * j + 2));
        const double u1 = ((double)(b0 >> 11) + 1.0) * 0x1.0p-53;
        const double u2 = (double)(b1 >> 11) * 0x1.0p-53;
        const double radius = sqrt(-2.0 * log(u1));
        const double angle = (2.0 * 3.141592653589793) * u2;
        double s, c;
        sincos(angle, &s, &c);
        const long long f0 = 2 * j;
        const long long c0 = f0 / N, n0 = f0 - c0 * N;
        y[c0 * ld + n0] = (float)(radius * c);
        const long long f1 = f0 + 1;
        if (f1 < total) {
            const long long c1 = f1 / N, n1 = f1 - c1 * N;
            y[c1 * ld + n1] = (float)(radius * s);
        }
    }
}

__global__ void peak_abs_kernel(const float *x, long long C, long long N, long long ld, unsigned int *out_bits) {
    float m = 0.f;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long c = 0; c < C; ++c) {
        const float *row = x + c * ld;
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride)
            m = fmaxf(m, fabsf(__ldcs(row + i)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    // non-negative floats order like their bit patterns
    if ((threadIdx.x & 31) == 0) atomicMax(out_bits, __float_as_uint(m));
}

__global__ void scale_by_peak_kernel(const float *x, float *y, long long C, long long N, long long ldx, long long ldy,
                                     const unsigned int *peak_bits, float target) {
    const float peak = __uint_as_float(*peak_bits);
    const float s = peak > 0.f ? target / peak : 1.f;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long c = 0; c < C; ++c) {
        const float *xr = x + c * ldx;
        float *yr = y + c * ldy;
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride)
            yr[i] = peak > 0.f ? xr[i] * s : xr[i];
    }
}

}  // namespace wpk

namespace wp {

static int grid_for(long long work, int threads) {
    long long g = (work + threads - 1) / threads;
    const long long cap = (long long)sm_count() * 8;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

cudaError_t launch_white_noise(float *y, long long C, long long N, long long ld, unsigned long long seed,
                               cudaStream_t st) {
    const long long pairs = (C * N + 1) / 2;
    wpk::white_noise_kernel<<<grid_for(pairs, 256), 256, 0, st>>>(y, C, N, ld, seed);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_peak_abs(const float *x, long long C, long long N, long long ld, unsigned int *out_bits,
                            cudaStream_t st) {
    wpk::peak_abs_kernel<<<grid_for(N, 256), 256, 0, st>>>(x, C, N, ld, out_bits);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_scale_by_peak(const float *x, float *y, long long C, long long N, long long ldx, long long ldy,
                                 const unsigned int *peak_bits, float target, cudaStream_t st) {
    wpk::scale_by_peak_kernel<<<grid_for(N, 256), 256, 0, st>>>(x, y, C, N, ldx, ldy, peak_bits, target);
    count_launch();
    return cudaGetLastError();
}

}  // namespace wp
