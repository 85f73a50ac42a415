// WAV payload codec on the device: interleaved
// little-endian RIFF payload <-> planar float32 [C][ld], replacing the
// reference's numpy decode/encode (wavio.py:155-200 _decode, :69-98 save_wav).
//
// Decode: pcm16 -> x / 2^15, pcm24 (sign-extended 3 bytes) -> x / 2^23,
// float32 -> bit copy. Every value is exactly representable in float32, so the
// planar result equals the reference's float64 samples rounded to float32
// bit for bit.
// Encode: float32 -> bit copy; pcm -> clamp to [-1, 1], quantize
// round-half-away-from-zero: copysign(floor(|x| 2^(b-1) + 0.5), x), clipped to
// [-2^(b-1), 2^(b-1) - 1]. For float32 inputs every step is exact in float32
// (power-of-two scaling, +0.5 within the significand), so the bytes equal the
// reference's float64 computation. Samples with |x| > 1 are counted.
//
// Both directions go through a 32 x 32 (frames x channels) shared-memory tile
// so that the interleaved side and the planar side are both accessed in
// contiguous runs.
#include <stdint.h>

#include "wp_internal.h"

namespace wpk {

namespace {

constexpr int TW = 32;

__device__ __forceinline__ float decode_one(const unsigned char *p, long long e, int enc) {
    if (enc == 16) {
        const int16_t v = (int16_t)((uint16_t)p[2 * e] | ((uint16_t)p[2 * e + 1] << 8));
        return (float)v * (1.0f / 32768.0f);
    }
    if (enc == 24) {
        const int32_t v = (int32_t)(((uint32_t)p[3 * e] << 8) | ((uint32_t)p[3 * e + 1] << 16) |
                                    ((uint32_t)p[3 * e + 2] << 24)) >> 8;
        return (float)v * (1.0f / 8388608.0f);
    }
    const uint32_t b = (uint32_t)p[4 * e] | ((uint32_t)p[4 * e + 1] << 8) | ((uint32_t)p[4 * e + 2] << 16) |
                       ((uint32_t)p[4 * e + 3] << 24);
    return __uint_as_float(b);
}

__device__ __forceinline__ int quantize(float x, float full) {
    float c = fminf(fmaxf(x, -1.0f), 1.0f);
    const float q = copysignf(floorf(fabsf(c) * full + 0.5f), c);
    return (int)fminf(fmaxf(q, -full), full - 1.0f);
}

}  // namespace

__global__ void wav_decode_kernel(const unsigned char *payload, int enc, float *y, long long C, long long N,
                                  long long ld) {
    __shared__ float tile[TW][TW + 1];
    const long long n0 = (long long)blockIdx.x * TW, c0 = (long long)blockIdx.y * TW;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    // read: frame n0+r, channels c0+tx (contiguous in the interleaved payload)
    for (int r = ty; r < TW; r += 8) {
        const long long n = n0 + r, c = c0 + tx;
        if (n < N && c < C) tile[r][tx] = decode_one(payload, n * C + c, enc);
    }
    __syncthreads();
    // write: channel c0+r, frames n0+tx (contiguous in the planar output)
    for (int r = ty; r < TW; r += 8) {
        const long long c = c0 + r, n = n0 + tx;
        if (n < N && c < C) y[c * ld + n] = tile[tx][r];
    }
}

__global__ void wav_encode_kernel(const float *x, long long C, long long N, long long ld, int enc,
                                  unsigned char *payload, unsigned long long *clipped) {
    __shared__ float tile[TW][TW + 1];
    const long long n0 = (long long)blockIdx.x * TW, c0 = (long long)blockIdx.y * TW;
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int r = ty; r < TW; r += 8) {
        const long long c = c0 + r, n = n0 + tx;
        if (n < N && c < C) tile[tx][r] = x[c * ld + n];
    }
    __syncthreads();
    unsigned int clip = 0;
    for (int r = ty; r < TW; r += 8) {
        const long long n = n0 + r, c = c0 + tx;
        if (n < N && c < C) {
            const float v = tile[r][tx];
            const long long e = n * C + c;
            if (enc == 32) {
                const uint32_t b = __float_as_uint(v);
                payload[4 * e] = (unsigned char)b;
                payload[4 * e + 1] = (unsigned char)(b >> 8);
                payload[4 * e + 2] = (unsigned char)(b >> 16);
                payload[4 * e + 3] = (unsigned char)(b >> 24);
            } else {
                clip += fabsf(v) > 1.0f;
                const int q = quantize(v, enc == 16 ? 32768.0f : 8388608.0f);
                payload[(enc / 8) * e] = (unsigned char)q;
                payload[(enc / 8) * e + 1] = (unsigned char)(q >> 8);
                if (enc == 24) payload[3 * e + 2] = (unsigned char)(q >> 16);
            }
        }
    }
    if (enc != 32) {
        const unsigned int w = __reduce_add_sync(0xffffffffu, clip);
        if ((threadIdx.x & 31) == 0 && w) atomicAdd(clipped, (unsigned long long)w);
    }
}

}  // namespace wpk

namespace wp {

cudaError_t launch_wav_decode(const void *payload, int enc, float *y, long long C, long long N, long long ld,
                              cudaStream_t st) {
    const dim3 grid((unsigned)((N + 31) / 32), (unsigned)((C + 31) / 32)), block(32, 8);
    wpk::wav_decode_kernel<<<grid, block, 0, st>>>(static_cast<const unsigned char *>(payload), enc, y, C, N, ld);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_wav_encode(const float *x, long long C, long long N, long long ld, int enc, void *payload,
                              unsigned long long *clipped, cudaStream_t st) {
    const dim3 grid((unsigned)((N + 31) / 32), (unsigned)((C + 31) / 32)), block(32, 8);
    wpk::wav_encode_kernel<<<grid, block, 0, st>>>(x, C, N, ld, enc, static_cast<unsigned char *>(payload), clipped);
    count_launch();
    return cudaGetLastError();
}

}  // namespace wp
