// Internal host-side interfaces shared by the C-ABI translation unit and the
// per-dtype kernel translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "wp_fused.cuh"

namespace wpk {
constexpr int TC_M = 128;                     // UMMA M: rows of the Hankel operand
constexpr int TC_N = 64;                      // UMMA N: output phases per row (= row stride)
constexpr int TC_TOUT = TC_M * TC_N;          // outputs per tile (8192)

struct FirTcArgs {
    const float *x;
    float *y;
    long long C, N, ldx, ldy;
    long long total_tiles;
    int Tp, K, W;
    int nin;                    // window/operand slots in the ring (1..4)
    const unsigned char *Bimg;  // [2][K/16][512]
    float out_scale;            // 2^-f of the taps
    float pre_gain;
    int n_post;
    float post[MAXPOST];
    int vec_x, vec_y;
    int tma_y;                  // the y tensor map is valid: full tiles leave through TMA stores
    unsigned long long *trace;  // [tiles][FT_TRACE_EV] stage stamps (-DFT_TRACE builds only)
};

constexpr int FT_TRACE_EV = 16;

constexpr int FFT_M = 16384;      // complex FFT size of the overlap-save path
constexpr int FFT_THREADS = 512;

struct FftArgs {
    const float *x;
    float *y;
    long long C, N, ldx, ldy;
    long long nblk;    // blocks per channel
    long long total;   // work items: channel pairs x blocks
    int Tpad, L;       // halo (multiple of 512, >= taps-1), new outputs per block
    const float2 *H;   // [16][1024] spectrum of the taps, digit-reversed order, x gain / M
    const float2 *tw;  // [256] W_M^n (n < 128), W_M^(128 k) (k < 128)
    long long delay;   // input delay in samples (taps segment j of a long FIR: j x 8192)
    int accumulate;    // add to y instead of storing (segments after the first)
};

}  // namespace wpk

namespace wp {

// float64 scan tables of one fused IIR block (D = 2S), computed on the host.
struct HostTables {
    int S = 0;
    int D = 1;
    std::vector<double> sos;  // [S][5]
    std::vector<double> K;    // [L][D]
    std::vector<double> P;    // [5][D][D]
    std::vector<double> W;    // [NW][D][D]
    std::vector<double> MT;   // [D][D]
    std::vector<double> G;    // [D][D][33]  lane-minor
    std::vector<double> TP;   // [33][D][D]
};

// Launch one fused pass. `grid` = number of persistent CTAs.
cudaError_t launch_fused_f32(int S, bool fir, const wpk::FusedArgs &a, const HostTables &t, int grid,
                             size_t smem, cudaStream_t st);
cudaError_t launch_fused_f64(int S, bool fir, const wpk::FusedArgs &a, const HostTables &t, int grid,
                             size_t smem, cudaStream_t st);
// Max resident CTAs per SM for the instantiation (0 on error).
int fused_occupancy(bool f64, int S, bool fir, size_t smem);
size_t fused_smem_bytes(bool f64, int S, int tpad);

// misc kernels (wp_misc.cu)
cudaError_t launch_white_noise(float *y, long long C, long long N, long long ld, unsigned long long seed,
                               cudaStream_t st);
cudaError_t launch_peak_abs(const float *x, long long C, long long N, long long ld, unsigned int *out_bits,
                            cudaStream_t st);
cudaError_t launch_scale_by_peak(const float *x, float *y, long long C, long long N, long long ldx, long long ldy,
                                 const unsigned int *peak_bits, float target, cudaStream_t st);

// tensor-core FIR (wp_fir_tc.cu)
size_t fir_tc_smem_bytes(int W, int K, int nin);
// TMA view of an output signal y as [C][N / 64][64] floats, 32 x 32 boxes, 128-B swizzle
// (false: no driver entry point, N < 64 or unaligned - the caller keeps its LDS/STG path)
bool encode_ymap(CUtensorMap &m, float *y, long long C, long long N, long long ldy);
cudaError_t fft_ols_prepare();
cudaError_t launch_fir_tc(const wpk::FirTcArgs &a, const CUtensorMap &ymap, int grid, size_t smem, cudaStream_t st);
int fir_tc_occupancy(size_t smem);

// single-pass tensor-core chain with look-back (wp_lb.cu / wp_lb.cuh)
struct LbPlan {
    int D = 0, H = 0, K = 0, W = 0, nop = 2;
    bool tma_stage = false;  // epilogue staging laid out for TMA output stores
    bool dense = false;      // globally balanced (dense) state basis: the block basis is ill-conditioned
    double cond_ratio = 0;   // fp32 roundoff gain of the block basis
    size_t smem = 0;
    unsigned char *d_bimg = nullptr;
    float *d_stabs = nullptr, *d_MTl = nullptr;
    float out_scale = 1.f;
    float escale[16] = {};
    float4 Ep[256] = {};          // E pairs for the kernel's parameter space
    float Mpw[11 * 16 * 16] = {};  // M^(2^b), M^(32 w) for the kernel's parameter space
    std::string desc;
};
// S sections (<= 8) and T taps (T <= 1: no FIR) fit the kernel's shared memory
bool lb_fits(int S, int T);
size_t lb_smem_bytes(int D, int H, int nop, bool tma, bool dense);
bool lb_ill_conditioned(const double *sos, int S);  // block basis fp32 roundoff gain past the dense threshold
int lb_build(LbPlan &p, const std::vector<double> &sos, int S, const std::vector<double> &taps, double gain,
             std::string &err);
void lb_free(LbPlan &p);
size_t lb_workspace_bytes(const LbPlan &p, long long channels, long long tiles);
cudaError_t lb_launch(const LbPlan &p, const float *x, float *y, long long C, long long N, long long ldx, long long ldy,
                      void *ws, unsigned long long *trace, cudaStream_t st);

// WAV payload codec (wp_wav.cu)
cudaError_t launch_wav_decode(const void *payload, int enc, float *y, long long C, long long N, long long ld,
                              cudaStream_t st);
cudaError_t launch_wav_encode(const float *x, long long C, long long N, long long ld, int enc, void *payload,
                              unsigned long long *clipped, cudaStream_t st);

// FFT overlap-save long FIR (wp_fft_ols.cu)
size_t fft_ols_smem_bytes();
cudaError_t launch_fft_ols(const wpk::FftArgs &a, int grid, cudaStream_t st);

void count_launch(int n = 1);
int sm_count();

}  // namespace wp
