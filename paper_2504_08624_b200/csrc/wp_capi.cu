// C ABI of libwpb200.so (declarations in include/wavepipe_b200.h).
//
// A plan turns the reference's stage list (Chain.stages, chain.py:27-41) into
// fused passes (each run of IIR / FIR / gain stages is one LTI pass while it
// fits chain_lb) and precomputes, in long double on the host, every table the
// kernels need. Executing a plan issues one kernel per pass (plus a small
// stream-ordered memset of the look-back records / tile counter), never
// allocates and never synchronizes.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>
#include <complex>
#include <cstdlib>
#include <unistd.h>

#include "../../include/wavepipe_b200.h"
#include "wp_internal.h"
#include "wp_lb.cuh"

namespace wp {
int fused_occupancy_f32(int S, bool fir, size_t smem);
int fused_occupancy_f64(int S, bool fir, size_t smem);
size_t fused_smem_bytes_f32(int S, int tpad);
size_t fused_smem_bytes_f64(int S, int tpad);
}  // namespace wp

namespace {

thread_local std::string g_err;
unsigned long long *g_trace = nullptr;  // diagnostics: per-tile stage timestamps (wp_set_trace)
size_t g_trace_entries = 0;
std::atomic<unsigned long long> g_launches{0};

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char *what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return WP_ECUDA;
}

constexpr double kF64Radius = 0.98;

// ---------------------------------------------------------------- matrices
using Mat = std::vector<double>;  // row-major D x D

Mat identity(int D) {
    Mat m(D * D, 0.0);
    for (int i = 0; i < D; ++i) m[i * D + i] = 1.0;
    return m;
}

Mat matmul(const Mat &a, const Mat &b, int D) {
    Mat c(D * D, 0.0);
    for (int i = 0; i < D; ++i)
        for (int k = 0; k < D; ++k) {
            const long double aik = a[i * D + k];
            if (aik == 0.0L) continue;
            for (int j = 0; j < D; ++j) c[i * D + j] += (double)(aik * (long double)b[k * D + j]);
        }
    return c;
}

Mat matpow(const Mat &m, int e, int D) {
    Mat r = identity(D), base = m;
    while (e > 0) {
        if (e & 1) r = matmul(r, base, D);
        base = matmul(base, base, D);
        e >>= 1;
    }
    return r;
}

// One DF2T cascade step: state (w1_s, w2_s) per section, input u.
void cascade_step(const std::vector<double> &sos, int S, const double *st, double u, double *out) {
    for (int s = 0; s < S; ++s) {
        const double b0 = sos[5 * s], b1 = sos[5 * s + 1], b2 = sos[5 * s + 2];
        const double a1 = sos[5 * s + 3], a2 = sos[5 * s + 4];
        const double w1 = st[2 * s], w2 = st[2 * s + 1];
        const double y = b0 * u + w1;
        out[2 * s] = b1 * u - a1 * y + w2;
        out[2 * s + 1] = b2 * u - a2 * y;
        u = y;
    }
}

// Output of one DF2T cascade step (the last section's y) for state st, input u.
double cascade_out(const std::vector<double> &sos, int S, const double *st, double u) {
    for (int s = 0; s < S; ++s) {
        const double y = sos[5 * s] * u + st[2 * s];
        u = y;
    }
    return u;
}

// State space of the cascade: s' = A s + B u, y = C s + d u (DF2T states).
void cascade_ss(const std::vector<double> &sos, int S, Mat &A, std::vector<double> &B, std::vector<double> &C,
                double &d) {
    const int D = 2 * S;
    A.assign(D * D, 0.0);
    B.assign(D, 0.0);
    C.assign(D, 0.0);
    std::vector<double> e(D), o(D);
    for (int j = 0; j < D; ++j) {
        std::fill(e.begin(), e.end(), 0.0);
        e[j] = 1.0;
        cascade_step(sos, S, e.data(), 0.0, o.data());
        for (int i = 0; i < D; ++i) A[i * D + j] = o[i];
        C[j] = cascade_out(sos, S, e.data(), 0.0);
    }
    std::fill(e.begin(), e.end(), 0.0);
    cascade_step(sos, S, e.data(), 1.0, B.data());
    d = cascade_out(sos, S, e.data(), 1.0);
}

void build_tables(wp::HostTables &t, const std::vector<double> &sos, int S, int H) {
    const int D = 2 * S;
    t.S = S;
    t.D = D;
    t.sos = sos;
    Mat A(D * D);
    std::vector<double> B(D), e(D), o(D);
    for (int j = 0; j < D; ++j) {
        std::fill(e.begin(), e.end(), 0.0);
        e[j] = 1.0;
        cascade_step(sos, S, e.data(), 0.0, o.data());
        for (int i = 0; i < D; ++i) A[i * D + j] = o[i];
    }
    std::fill(e.begin(), e.end(), 0.0);
    cascade_step(sos, S, e.data(), 1.0, B.data());
    const int L = wpk::L;
    // K[n] = A^(L-1-n) B
    t.K.assign(L * D, 0.0);
    std::vector<double> v = B, nv(D);
    for (int n = L - 1; n >= 0; --n) {
        for (int i = 0; i < D; ++i) t.K[n * D + i] = v[i];
        for (int i = 0; i < D; ++i) {
            long double acc = 0;
            for (int j = 0; j < D; ++j) acc += (long double)A[i * D + j] * v[j];
            nv[i] = (double)acc;
        }
        v = nv;
    }
    const Mat M = matpow(A, L, D);
    t.P.assign(5 * D * D, 0.0);
    Mat p = M;
    for (int q = 0; q < 5; ++q) {
        std::copy(p.begin(), p.end(), t.P.begin() + q * D * D);
        p = matmul(p, p, D);
    }
    std::vector<Mat> G(33);
    G[0] = identity(D);
    for (int l = 1; l <= 32; ++l) G[l] = matmul(G[l - 1], M, D);
    t.G.assign(D * D * 33, 0.0);
    for (int l = 0; l <= 32; ++l)
        for (int i = 0; i < D; ++i)
            for (int j = 0; j < D; ++j) t.G[(i * D + j) * 33 + l] = G[l][i * D + j];
    t.W.assign(wpk::NW * D * D, 0.0);
    Mat w = identity(D);
    for (int q = 0; q < wpk::NW; ++q) {
        std::copy(w.begin(), w.end(), t.W.begin() + q * D * D);
        w = matmul(w, G[32], D);
    }
    const int chunks = wpk::NT - H / L;
    const Mat MT = matpow(M, chunks, D);
    t.MT = MT;
    t.TP.assign(33 * D * D, 0.0);
    Mat tp = identity(D);
    for (int j = 0; j <= 32; ++j) {
        std::copy(tp.begin(), tp.end(), t.TP.begin() + j * D * D);
        tp = matmul(tp, MT, D);
    }
}

double section_radius(const double *r) {
    const double a1 = r[3], a2 = r[4];
    const double disc = a1 * a1 - 4.0 * a2;
    if (disc < 0) return std::sqrt(a2);
    const double q = std::sqrt(disc);
    return 0.5 * std::max(std::fabs(-a1 + q), std::fabs(-a1 - q));
}

struct Pass {
    enum Kind { FUSED = 0, NORMALIZE = 1 } kind = FUSED;
    int S = 0;
    std::vector<double> sos;
    int prec_flag = 0;  // OR of stage precision flags
    bool f64 = false;
    int T = 0, Tpad = 0, H = 0, Lout = wpk::REGION;
    std::vector<double> taps;
    float pre = 1.f;
    std::vector<float> post;
    double target = 1.0;
    wp::HostTables tables;
    void *d_G = nullptr, *d_TP = nullptr;
    float *d_taps = nullptr;
    size_t smem = 0;
    int grid_cap = 0;
    int fir_flags = 0;
    // tensor-core FIR (FIR-only passes)
    bool fir_tc = false;
    int tc_Tp = 0, tc_K = 0, tc_W = 0, tc_nin = 2;
    float tc_out_scale = 1.f;
    unsigned char *d_Bimg = nullptr;
    // FFT overlap-save (long FIR-only passes)
    bool fft = false;
    int fft_Tpad = 0;
    int fft_segs = 1;        // > 1: taps split into segments of kFftSegTaps, one launch each (accumulating)
    float2 *d_H = nullptr, *d_tw = nullptr;  // d_H: [segs][M]
    // single-pass tensor-core chain with look-back (wp_lb.cuh): IIR [+ FIR] passes;
    // IIR-only passes of <= 4 sections keep the fused kernel for small calls
    bool lb = false, lb_large = false;
    long long lb_min_tiles = 0;
    double gain = 1.0;  // combined gain of an LTI pass (lti planner)
    wp::LbPlan lbp;
    std::string desc;
    bool empty() const { return kind == FUSED && S == 0 && T == 0 && pre == 1.f && post.empty(); }
};

}  // namespace

struct wp_plan {
    std::vector<Pass> passes;
    int device = 0;
};

namespace wp {

void count_launch(int n) { g_launches.fetch_add((unsigned long long)n); }

int sm_count() {
    static std::atomic<int> cached[64];  // per device; benign races write the same value
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    int v = cached[dev].load(std::memory_order_relaxed);
    if (!v) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        v = n > 0 ? n : 1;
        cached[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

}  // namespace wp

namespace {

bool fir_tc_enabled() {
    const char *v = std::getenv("WP_FIR_IMPL");
    return !(v && std::string(v) == "cuda");
}

// WP_CHAIN_IMPL=cuda: IIR passes on the CUDA-core chunked scan only; =lb: chain_lb
// for every IIR-only call, however small (A/B diagnostics and tests)
bool lb_enabled() {
    const char *v = std::getenv("WP_CHAIN_IMPL");
    return !(v && std::string(v) == "cuda");
}
// sections per chain_lb pass for a run of `total` IIR sections. One pass costs
// more than linearly in the state size past 4 sections (D = 16: the D^2 scan and
// look-back work and 2 x the E s FMAs), so measured on the reference's 8-SOS
// bench chain (32 x 5.29 M): one 8-section pass 1.71 ms, 4 + 4 0.92 ms, 5 + 3
// 1.05, 6 + 2 1.25, 3 + 3 + 2 1.18; five sections: one pass 0.65 vs 3 + 2 0.76.
// Hence: up to 5 sections in one pass, more split into balanced passes of <= 4.
// WP_LB_MAXS=n forces at most n per pass (A/B).
int lb_max_sections(int total) {
    const char *v = std::getenv("WP_LB_MAXS");
    if (v) {
        const int n = std::atoi(v);
        if (n >= 1 && n <= 8) return n;
    }
    if (total <= 5) return 8;
    const int passes = (total + 3) / 4;
    return (total + passes - 1) / passes;
}
int env_int(const char *name, int dflt) {
    const char *v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
}
bool lb_forced() {
    const char *v = std::getenv("WP_CHAIN_IMPL");
    return v && std::string(v) == "lb";
}

void host_fft(std::vector<std::complex<double>> &a) {
    const size_t n = a.size();
    for (size_t i = 1, j = 0; i < n; ++i) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(a[i], a[j]);
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        const double ang = -2.0 * M_PI / (double)len;
        for (size_t i = 0; i < n; i += len)
            for (size_t k = 0; k < len / 2; ++k) {
                const std::complex<double> w(std::cos(ang * (double)k), std::sin(ang * (double)k));
                const std::complex<double> u = a[i + k], v = a[i + k + len / 2] * w;
                a[i + k] = u + v;
                a[i + k + len / 2] = u - v;
            }
    }
}

// taps per segment when a FIR is longer than one 16 K-point overlap-save block
// can hold (> 15361 taps): 8192 minimises the transform work per tap
// (segments x M / (M - 8192)), one accumulating launch per segment
constexpr int kFftSegTaps = 8192;

// FFT overlap-save tables of pass p: spectrum of the (gain-scaled) taps in the
// kernel's digit-reversed order k = k1 + 32 k2 + 1024 k3 -> [k3][k1*32 + k2],
// pre-divided by M, and the two-level twiddle table. Taps beyond one block's
// reach are split into segments, segment j convolving x delayed by j * kFftSegTaps.
int build_fft(Pass &p) {
    const int M = wpk::FFT_M;
    int Tpad = (p.T - 1 + 511) / 512 * 512;
    int segs = 1, seg_taps = p.T;
    if (Tpad >= M - 512) {
        seg_taps = kFftSegTaps;
        segs = (p.T + seg_taps - 1) / seg_taps;
        Tpad = (seg_taps - 1 + 511) / 512 * 512;
    }
    double gain = (double)p.pre;
    for (float g : p.post) gain *= (double)g;
    std::vector<float2> Hp((size_t)segs * M), tw(256 + 512 + 2048);
    for (int j = 0; j < segs; ++j) {
        std::vector<std::complex<double>> h(M, 0.0);
        for (int i = 0; i < seg_taps && j * seg_taps + i < p.T; ++i)
            h[i] = p.taps[(size_t)j * seg_taps + i] * gain / (double)M;
        host_fft(h);
        for (int k3 = 0; k3 < 16; ++k3)
            for (int k1 = 0; k1 < 32; ++k1)
                for (int k2 = 0; k2 < 32; ++k2) {
                    const std::complex<double> v = h[k1 + 32 * k2 + 1024 * k3];
                    Hp[(size_t)j * M + k3 * 1024 + k1 * 32 + k2] = make_float2((float)v.real(), (float)v.imag());
                }
    }
    for (int i = 0; i < 128; ++i) {
        const double a1 = -2.0 * M_PI * i / M, a2 = -2.0 * M_PI * 128.0 * i / M;
        tw[i] = make_float2((float)std::cos(a1), (float)std::sin(a1));
        tw[128 + i] = make_float2((float)std::cos(a2), (float)std::sin(a2));
    }
    for (int k = 0; k < 32; ++k)  // pass-2 twiddles W_M^(32 bp k), [k][bp]
        for (int bp = 0; bp < 16; ++bp) {
            const double an = -2.0 * M_PI * (double)(((long long)32 * bp * k) % M) / M;
            tw[256 + 16 * k + bp] = make_float2((float)std::cos(an), (float)std::sin(an));
        }
    for (int m = 0; m < 2048; ++m) {  // pass-1 anchors W_M^(8 m)
        const double an = -2.0 * M_PI * 8.0 * m / M;
        tw[768 + m] = make_float2((float)std::cos(an), (float)std::sin(an));
    }
    cudaError_t e = cudaMalloc(&p.d_H, sizeof(float2) * Hp.size());
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(H)");
    e = cudaMemcpy(p.d_H, Hp.data(), sizeof(float2) * Hp.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(H)");
    e = cudaMalloc(&p.d_tw, sizeof(float2) * tw.size());
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(tw)");
    e = cudaMemcpy(p.d_tw, tw.data(), sizeof(float2) * tw.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(tw)");
    e = wp::fft_ols_prepare();  // kernel attribute, once per plan (not per execute)
    if (e != cudaSuccess) return cuda_fail(e, "fft_ols attribute");
    p.fft = true;
    p.fft_Tpad = Tpad;
    p.fft_segs = segs;
    p.Lout = M - Tpad;
    p.grid_cap = wp::sm_count();
    char buf[256];
    snprintf(buf, sizeof buf, "fft_ols[pre=%g taps=%d post=%zu] M=%d halo=%d block=%d 2 ch/CTA smem=%zu segments=%d",
             (double)p.pre, p.T, p.post.size(), M, Tpad, M - Tpad, wp::fft_ols_smem_bytes(), segs);
    p.desc = buf;
    return WP_OK;
}

int finalize_pass(Pass &p) {
    if (p.kind != Pass::FUSED) {
        char buf[128];
        snprintf(buf, sizeof buf, "normalize(peak=%g): peak_abs + scale", p.target);
        p.desc = buf;
        return WP_OK;
    }
    if (p.S > 0 && lb_enabled() && wp::lb_fits(p.S, p.T)) {
        double gain = (double)p.pre;
        for (float g : p.post) gain *= (double)g;
        if (p.gain != 1.0) gain = p.gain;
        std::string err;
        const int rc = wp::lb_build(p.lbp, p.sos, p.S, p.T > 0 ? p.taps : std::vector<double>{}, gain, err);
        if (rc != WP_OK) return fail(rc, err);
        if (p.T > 1 || p.S > wpk::MAXS) {
            p.lb = true;
            p.desc = p.lbp.desc;
            return WP_OK;
        }
        // IIR-only: small calls keep the fused chunked scan (one launch, exact
        // per-chunk recurrence for the known-answer cases)
        p.lb_large = true;
        // measured crossover (tools/iir_small_probe.py): chain_lb is faster from ~16 tiles
        // for >= 3 sections and from ~64 tiles for 1-2 sections; below that the single
        // fused launch wins and keeps its exact per-chunk recurrence for the KAT cases
        p.lb_min_tiles = lb_forced() ? 0 : (p.S >= 3 ? 16 : 64);
        if (p.T == 1) {
            // a 1-tap FIR is a gain: the fused kernel takes it as a post gain
            p.post.push_back((float)p.taps[0]);
            p.T = 0;
            p.taps.clear();
        }
    }
    if (p.S == 0 && p.T >= 8 && fir_tc_enabled()) {
        // tensor-core direct FIR: rows of 64 samples, K covers taps + 63 phases
        p.tc_Tp = (p.T - 1 + 7) / 8 * 8;
        p.tc_K = (p.tc_Tp + wpk::TC_N + 15) / 16 * 16;
        p.tc_W = wpk::TC_N * (wpk::TC_M - 1) + p.tc_K;
        // double-buffered fp32 windows up to 129 taps, one window buffer up to 257 taps (the
        // B image grows with the taps); beyond that FFT overlap-save is the faster path anyway
        // (profiles/r2_fir_crossover.md: fir_tc 0.19-0.21 ms vs fft_ols 0.31 ms per pass)
        // window/operand slots in the ring: as many as shared memory holds (<= 4); WP_FIR_NIN caps it (A/B)
        const int nin_cap = env_int("WP_FIR_NIN", 4);
        p.tc_nin = 1;
        for (int n = std::min(4, std::max(1, nin_cap)); n > 1; --n)
            if (wp::fir_tc_smem_bytes(p.tc_W, p.tc_K, n) <= 227 * 1024) {
                p.tc_nin = n;
                break;
            }
        p.fir_tc = wp::fir_tc_smem_bytes(p.tc_W, p.tc_K, p.tc_nin) <= 227 * 1024 && p.tc_W <= 10 * 4 * 256;
    }
    // FIR-only: FFT overlap-save unless forced direct; a forced-direct FIR beyond the
    // fused direct kernel's halo (> ~7680 taps) also takes the FFT path
    const bool direct_fits = (p.T + 7) / 8 * 8 <= wpk::REGION - 9 * wpk::L;
    if (p.S == 0 && p.T > 1 && (!(p.fir_flags & WP_FIR_DIRECT) || (!p.fir_tc && !direct_fits)) &&
        ((p.fir_flags & WP_FIR_FFT) || !p.fir_tc)) {
        p.fir_tc = false;
        return build_fft(p);
    }
    if (p.fir_tc) {
        double hmax = 0;
        for (double v : p.taps) hmax = std::max(hmax, std::fabs(v));
        int ex = 0;
        if (hmax > 0) std::frexp(hmax, &ex);
        const int f = hmax > 0 ? 14 - ex : 0;
        p.tc_out_scale = (float)std::ldexp(1.0, -f);
        // B image, K-major SWIZZLE_128B: [split][K atom of 64][row p][128 B],
        // 16-byte chunks XOR-swizzled by (row & 7)
        const int atoms = (p.tc_K + 63) / 64;
        const size_t split = (size_t)atoms * 8192 / sizeof(__half);
        std::vector<__half> img(2 * split, __float2half_rn(0.f));
        for (int pcol = 0; pcol < wpk::TC_N; ++pcol)
            for (int k = 0; k < p.tc_K; ++k) {
                const int t = pcol + p.tc_Tp - k;
                const float val = (t >= 0 && t < p.T) ? (float)std::ldexp(p.taps[t], f) : 0.f;
                const __half hi = __float2half_rn(val);
                const __half lo = __float2half_rn((val - __half2float(hi)) * 2048.f);
                // [atom][hi rows 0..63 | lo rows 64..127][128 B]: one N = 128 operand per K atom
                const uint32_t logical = (uint32_t)(k / 64) * 16384u + (uint32_t)pcol * 128u + (uint32_t)(k % 64) * 2u;
                const uint32_t phys = logical ^ (((logical >> 7) & 7u) << 4);
                img[phys / 2] = hi;
                img[(phys + 8192u) / 2] = lo;
            }
        cudaError_t e = cudaMalloc(&p.d_Bimg, img.size() * sizeof(__half));
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(Bimg)");
        e = cudaMemcpy(p.d_Bimg, img.data(), img.size() * sizeof(__half), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(Bimg)");
        p.smem = wp::fir_tc_smem_bytes(p.tc_W, p.tc_K, p.tc_nin);
        const int occ = wp::fir_tc_occupancy(p.smem);
        if (occ <= 0) return fail(WP_ECUDA, "tensor-core FIR kernel cannot be resident");
        p.grid_cap = occ * wp::sm_count();
        p.Lout = wpk::TC_TOUT;
        char buf[256];
        snprintf(buf, sizeof buf,
                 "fir_tc[pre=%g taps=%d K=%d post=%zu] tcgen05 f16x3 M128xN64 SW128 tile=%d smem=%zu occ=%d slots=%d",
                 (double)p.pre, p.T, p.tc_K, p.post.size(), wpk::TC_TOUT, p.smem, occ, p.tc_nin);
        p.desc = buf;
        return WP_OK;
    }
    if (p.T > 0) {
        p.Tpad = (p.T + 7) / 8 * 8;
        p.H = (p.Tpad + wpk::L - 1) / wpk::L * wpk::L;
        if (p.H > wpk::REGION - 8 * wpk::L) return fail(WP_EUNSUP, "FIR too long for the direct fused kernel");
        p.Lout = wpk::REGION - p.H;
    }
    if (p.S > 0) {
        double rmax = 0;
        for (int s = 0; s < p.S; ++s) rmax = std::max(rmax, section_radius(&p.sos[5 * s]));
        if (p.prec_flag & WP_IIR_PREC_F64)
            p.f64 = true;
        else if (p.prec_flag & WP_IIR_PREC_F32)
            p.f64 = false;
        else
            p.f64 = rmax > kF64Radius;
        build_tables(p.tables, p.sos, p.S, p.H);
        const size_t es = p.f64 ? sizeof(double) : sizeof(float);
        const int D = 2 * p.S;
        std::vector<unsigned char> gbuf(es * D * D * 33), tbuf(es * 33 * D * D);
        for (size_t i = 0; i < p.tables.G.size(); ++i) {
            if (p.f64)
                reinterpret_cast<double *>(gbuf.data())[i] = p.tables.G[i];
            else
                reinterpret_cast<float *>(gbuf.data())[i] = (float)p.tables.G[i];
        }
        for (size_t i = 0; i < p.tables.TP.size(); ++i) {
            if (p.f64)
                reinterpret_cast<double *>(tbuf.data())[i] = p.tables.TP[i];
            else
                reinterpret_cast<float *>(tbuf.data())[i] = (float)p.tables.TP[i];
        }
        cudaError_t e = cudaMalloc(&p.d_G, gbuf.size());
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(G)");
        e = cudaMalloc(&p.d_TP, tbuf.size());
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(TP)");
        e = cudaMemcpy(p.d_G, gbuf.data(), gbuf.size(), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(G)");
        e = cudaMemcpy(p.d_TP, tbuf.data(), tbuf.size(), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(TP)");
    }
    if (p.T > 0) {
        std::vector<float> tp(p.Tpad, 0.f);
        for (int i = 0; i < p.T; ++i) tp[i] = (float)p.taps[i];
        cudaError_t e = cudaMalloc(&p.d_taps, sizeof(float) * p.Tpad);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(taps)");
        e = cudaMemcpy(p.d_taps, tp.data(), sizeof(float) * p.Tpad, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(taps)");
    }
    p.smem = p.f64 ? wp::fused_smem_bytes_f64(p.S, p.Tpad) : wp::fused_smem_bytes_f32(p.S, p.Tpad);
    const int occ = p.f64 ? wp::fused_occupancy_f64(p.S, p.T > 0, p.smem) : wp::fused_occupancy_f32(p.S, p.T > 0, p.smem);
    if (occ <= 0) return fail(WP_ECUDA, "fused kernel cannot be resident (occupancy 0): " + std::string(cudaGetErrorString(cudaGetLastError())));
    p.grid_cap = occ * wp::sm_count();
    char buf[256];
    snprintf(buf, sizeof buf, "fused[pre=%g iir=%d%s fir=%d post=%zu] tile=%d halo=%d smem=%zu occ=%d", (double)p.pre, p.S,
             p.S ? (p.f64 ? "(f64)" : "(f32)") : "", p.T, p.post.size(), p.Lout, p.H, p.smem, occ);
    p.desc = buf;
    if (p.lb_large) p.desc += " ; from " + std::to_string(p.lb_min_tiles) + " tiles: " + p.lbp.desc;
    return WP_OK;
}

void free_pass(Pass &p) {
    wp::lb_free(p.lbp);
    if (p.d_Bimg) cudaFree(p.d_Bimg);
    p.d_Bimg = nullptr;
    if (p.d_H) cudaFree(p.d_H);
    if (p.d_tw) cudaFree(p.d_tw);
    p.d_H = p.d_tw = nullptr;
    if (p.d_G) cudaFree(p.d_G);
    if (p.d_TP) cudaFree(p.d_TP);
    if (p.d_taps) cudaFree(p.d_taps);
    p.d_G = p.d_TP = nullptr;
    p.d_taps = nullptr;
}

size_t rec_bytes(const Pass &p) {
    if (p.kind != Pass::FUSED || p.S == 0) return 0;
    const size_t es = p.f64 ? 8 : 4;
    return (16 + 2 * (size_t)(2 * p.S) * es + 15) / 16 * 16;  // fused kernel's look-back record per tile
}

long long tiles_per_channel(const Pass &p, long long N) { return (N + p.Lout - 1) / p.Lout; }

// wp_plan_execute_host runs channel blocks of one call: while it does, every
// block takes the kernel route of the WHOLE call (t_route_C = its channels),
// so the result is bit-identical to one wp_plan_execute over all channels
static thread_local long long t_route_C = 0;
bool uses_lb(const Pass &p, long long C, long long N) {
    const long long Cr = std::max(C, t_route_C);
    return p.lb || (p.lb_large && ((N + wpk::CT_TOUT - 1) / wpk::CT_TOUT) * Cr >= p.lb_min_tiles);
}

// look-back records / scan buffers of one pass for a [C x N] call
size_t pass_rec_bytes(const Pass &p, long long C, long long N) {
    size_t b = rec_bytes(p) * (size_t)(tiles_per_channel(p, N) * C);
    if (p.lb || p.lb_large) b = std::max(b, wp::lb_workspace_bytes(p.lbp, C, ((N + wpk::CT_TOUT - 1) / wpk::CT_TOUT) * C));
    return b;
}

int arch_ok() {
    static int cached = -99;
    if (cached == -99) {
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
        cudaDeviceProp prop;
        e = cudaGetDeviceProperties(&prop, dev);
        if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
        if (prop.major != 10 || prop.minor != 0) {
            char buf[128];
            snprintf(buf, sizeof buf, "device %s is sm_%d%d; this build carries sm_100a code only", prop.name,
                     prop.major, prop.minor);
            g_err = buf;
            cached = WP_EARCH;
        } else {
            cached = WP_OK;
        }
    }
    return cached;
}

}  // namespace

extern "C" {

const char *wp_last_error(void) { return g_err.c_str(); }
int wp_abi_version(void) { return 1; }
uint64_t wp_launch_count(void) { return (uint64_t)g_launches.load(); }
int wp_check_device(void) { return arch_ok(); }
int wp_set_trace(uint64_t *device_buffer, size_t entries) {
    g_trace = reinterpret_cast<unsigned long long *>(device_buffer);
    g_trace_entries = device_buffer ? entries : 0;
    return WP_OK;
}

int wp_plan_create(const wp_stage *stages, int32_t n_stages, wp_plan **out_plan) {
    if (!out_plan) return fail(WP_EINVAL, "out_plan is NULL");
    *out_plan = nullptr;
    if (n_stages < 0 || (n_stages > 0 && !stages)) return fail(WP_EINVAL, "bad stage array");
    int rc = arch_ok();
    if (rc != WP_OK) return rc;
    wp_plan *plan = new wp_plan();
    cudaGetDevice(&plan->device);
    std::vector<Pass> &passes = plan->passes;
    Pass cur;
    auto close = [&]() {
        if (!cur.empty()) passes.push_back(cur);
        cur = Pass();
    };
    const bool lti = lb_enabled();
    // IIR sections (non-identity) in the LTI run (stages up to the next Normalize) of each stage
    std::vector<int> run_sections(n_stages > 0 ? n_stages : 1, 0);
    std::vector<char> run_one_pass(n_stages > 0 ? n_stages : 1, 0);
    for (int a = 0; a < n_stages;) {
        int b = a, tot = 0;
        std::vector<double> run_sos;
        while (b < n_stages && stages[b].kind != WP_STAGE_NORMALIZE) {
            if (stages[b].kind == WP_STAGE_IIR && stages[b].coef)
                for (int k = 0; k < stages[b].n; ++k) {
                    const double *r = stages[b].coef + 5 * k;
                    if (!(r[0] == 1.0 && r[1] == 0.0 && r[2] == 0.0 && r[3] == 0.0 && r[4] == 0.0)) {
                        ++tot;
                        run_sos.insert(run_sos.end(), r, r + 5);
                    }
                }
            ++b;
        }
        // a run of 6-8 sections whose block basis is ill-conditioned in fp32 stays ONE
        // pass (then in the globally balanced basis): splitting it would pass an fp32
        // intermediate whose error later sections can amplify past the bar
        const bool one = lti && tot > 5 && tot <= 8 && !std::getenv("WP_LB_MAXS") &&
                         wp::lb_ill_conditioned(run_sos.data(), tot);
        for (int q = a; q < b; ++q) {
            run_sections[q] = tot;
            run_one_pass[q] = one;
        }
        a = b + 1;
    }
    for (int si = 0; si < n_stages; ++si) {
        const wp_stage &st = stages[si];
        if (lti) {
            // LTI planner: every run of IIR / FIR / gain stages between
            // Normalize stages is ONE linear time-invariant system, so its
            // order does not matter (FIR -> IIR fuses like IIR -> FIR) and it
            // runs as one pass while it fits the single-pass kernel (<= 8
            // sections, FIR halo <= LB_MAX_H); a longer FIR gets its own pass.
            const int lbh = wpk::LB_MAX_H;
            if (st.kind == WP_STAGE_GAIN) {
                if (!std::isfinite(st.value)) {
                    delete plan;
                    return fail(WP_EINVAL, "gain must be finite");
                }
                cur.gain *= st.value;
                cur.pre = (float)cur.gain;
                continue;
            }
            if (st.kind == WP_STAGE_IIR) {
                if (st.n < 1 || !st.coef) {
                    delete plan;
                    return fail(WP_EINVAL, "IIR stage needs >= 1 section");
                }
                std::vector<int> keep;
                for (int k = 0; k < st.n; ++k) {
                    const double *r = st.coef + 5 * k;
                    if (!(r[0] == 1.0 && r[1] == 0.0 && r[2] == 0.0 && r[3] == 0.0 && r[4] == 0.0)) keep.push_back(k);
                }
                if (keep.empty()) continue;
                for (size_t idx = 0; idx < keep.size(); ++idx) {
                    // ... and while the IIR + FIR pass fits the single-pass kernel's shared memory
                    if (cur.S == (run_one_pass[si] ? 8 : lb_max_sections(run_sections[si])) ||
                        (cur.T > 0 && cur.T - 1 > lbh) ||
                        (cur.T > 1 && !wp::lb_fits(cur.S + 1, cur.T)))
                        close();
                    for (int j = 0; j < 5; ++j) cur.sos.push_back(st.coef[5 * keep[idx] + j]);
                    cur.S += 1;
                    cur.prec_flag |= st.flags & (WP_IIR_PREC_F32 | WP_IIR_PREC_F64);
                }
                continue;
            }
            if (st.kind == WP_STAGE_FIR) {
                if (st.n < 1 || !st.coef) {
                    delete plan;
                    return fail(WP_EINVAL, "FIR stage needs >= 1 tap");
                }
                const bool long_fir = st.n - 1 > lbh;
                if (cur.T > 0) {
                    const int comb = cur.T + st.n - 1;
                    if (comb - 1 > lbh || long_fir) close();
                } else if (long_fir && cur.S > 0) {
                    close();
                }
                if (cur.S > 0 && !wp::lb_fits(cur.S, cur.T > 0 ? cur.T + st.n - 1 : st.n))
                    close();  // the merged pass would not fit the single-pass kernel: the FIR starts a new one
                if (cur.T > 0) {
                    // convolve with the pass's FIR (both causal, same-length truncation later)
                    std::vector<long double> t((size_t)cur.T + st.n - 1, 0.0L);
                    for (int a = 0; a < cur.T; ++a)
                        for (int b = 0; b < st.n; ++b) t[a + b] += (long double)cur.taps[a] * (long double)st.coef[b];
                    cur.taps.assign(t.size(), 0.0);
                    for (size_t i = 0; i < t.size(); ++i) cur.taps[i] = (double)t[i];
                    cur.T = (int)t.size();
                    cur.fir_flags = 0;
                } else {
                    cur.T = st.n;
                    cur.taps.assign(st.coef, st.coef + st.n);
                    cur.fir_flags = st.flags & (WP_FIR_DIRECT | WP_FIR_FFT);
                }
                if (long_fir) close();  // a long FIR stays a FIR-only pass
                continue;
            }
        }
        switch (st.kind) {
            case WP_STAGE_GAIN: {
                if (!std::isfinite(st.value)) {
                    delete plan;
                    return fail(WP_EINVAL, "gain must be finite");
                }
                if (cur.S == 0 && cur.T == 0 && cur.post.empty()) {
                    cur.pre = cur.pre * (float)st.value;
                } else {
                    if ((int)cur.post.size() == wpk::MAXPOST) {
                        close();
                        cur.pre = (float)st.value;
                    } else {
                        cur.post.push_back((float)st.value);
                    }
                }
                break;
            }
            case WP_STAGE_IIR: {
                if (st.n < 1 || !st.coef) {
                    delete plan;
                    return fail(WP_EINVAL, "IIR stage needs >= 1 section");
                }
                // Exact no-op sections (b = (1,0,0), a = (0,0); e.g. design_peaking
                // at 0 dB, design.py:437-438) are dropped: the reference's DF2T
                // passes samples through them bit for bit (y = 1*x + 0).
                std::vector<int> keep;
                for (int k = 0; k < st.n; ++k) {
                    const double *r = st.coef + 5 * k;
                    if (!(r[0] == 1.0 && r[1] == 0.0 && r[2] == 0.0 && r[3] == 0.0 && r[4] == 0.0)) keep.push_back(k);
                }
                if (keep.empty()) break;
                if (cur.T > 0 || !cur.post.empty()) close();
                size_t idx = 0;
                while (idx < keep.size()) {
                    int room = wpk::MAXS - cur.S;
                    if (room == 0) {
                        close();
                        room = wpk::MAXS;
                    }
                    const int take = std::min<int>(room, (int)(keep.size() - idx));
                    for (int s = 0; s < take; ++s)
                        for (int j = 0; j < 5; ++j) cur.sos.push_back(st.coef[5 * keep[idx + s] + j]);
                    cur.S += take;
                    cur.prec_flag |= st.flags & (WP_IIR_PREC_F32 | WP_IIR_PREC_F64);
                    idx += take;
                }
                break;
            }
            case WP_STAGE_FIR: {
                if (st.n < 1 || !st.coef) {
                    delete plan;
                    return fail(WP_EINVAL, "FIR stage needs >= 1 tap");
                }
                if (cur.T > 0 || !cur.post.empty()) close();
                cur.T = st.n;
                cur.taps.assign(st.coef, st.coef + st.n);
                cur.fir_flags = st.flags & (WP_FIR_DIRECT | WP_FIR_FFT);
                break;
            }
            case WP_STAGE_NORMALIZE: {
                if (!(st.value > 0) || !std::isfinite(st.value)) {
                    delete plan;
                    return fail(WP_EINVAL, "normalize target must be finite and > 0");
                }
                close();
                Pass n;
                n.kind = Pass::NORMALIZE;
                n.target = st.value;
                passes.push_back(n);
                break;
            }
            default:
                delete plan;
                return fail(WP_EINVAL, "unknown stage kind " + std::to_string(st.kind));
        }
    }
    close();
    if (passes.empty()) passes.push_back(Pass());  // identity copy
    for (Pass &p : passes) {
        rc = finalize_pass(p);
        if (rc != WP_OK) {
            for (Pass &q : passes) free_pass(q);
            delete plan;
            return rc;
        }
    }
    *out_plan = plan;
    return WP_OK;
}

int wp_plan_destroy(wp_plan *plan) {
    if (!plan) return WP_OK;
    for (Pass &p : plan->passes) free_pass(p);
    delete plan;
    return WP_OK;
}

int wp_plan_num_passes(const wp_plan *plan) { return plan ? (int)plan->passes.size() : 0; }

int wp_plan_launches(const wp_plan *plan) {
    if (!plan) return 0;
    int n = 0;
    for (const Pass &p : plan->passes) n += p.kind != Pass::FUSED ? 2 : p.fft ? p.fft_segs : 1;
    return n;
}


int wp_plan_launches_for(const wp_plan *plan, int64_t channels, int64_t frames) {
    if (!plan) return 0;
    int n = 0;
    for (const Pass &p : plan->passes)
        n += p.kind != Pass::FUSED ? 2 : p.fft ? p.fft_segs : 1;
    return n;
}

const char *wp_plan_describe_for(const wp_plan *plan, int32_t pass, int64_t channels, int64_t frames) {
    if (!plan || pass < 0 || pass >= (int)plan->passes.size()) return "";
    const Pass &p = plan->passes[pass];
    if (p.lb) return p.desc.c_str();
    if (p.lb_large) return uses_lb(p, channels, frames) ? p.lbp.desc.c_str() : p.desc.c_str();
    return p.desc.c_str();
}

const char *wp_plan_describe(const wp_plan *plan, int32_t pass) {
    if (!plan || pass < 0 || pass >= (int)plan->passes.size()) return "";
    return plan->passes[pass].desc.c_str();
}

static size_t ws_layout(const wp_plan *plan, int64_t C, int64_t N, size_t *rec_off, size_t *tmp_off, int64_t *ld_tmp) {
    size_t recb = 0;
    for (const Pass &p : plan->passes) recb = std::max(recb, pass_rec_bytes(p, C, N));
    *rec_off = 256;
    *tmp_off = (256 + recb + 255) / 256 * 256;
    *ld_tmp = (N + 63) / 64 * 64;
    const size_t tmpb = plan->passes.size() >= 2 ? sizeof(float) * (size_t)C * (size_t)(*ld_tmp) : 0;
    return *tmp_off + tmpb;
}

int wp_plan_workspace_bytes(const wp_plan *plan, int64_t channels, int64_t frames, size_t *bytes) {
    if (!plan || !bytes) return fail(WP_EINVAL, "null argument");
    if (channels < 1 || frames < 1) return fail(WP_EINVAL, "need channels >= 1 and frames >= 1");
    size_t a, b;
    int64_t ld;
    *bytes = ws_layout(plan, channels, frames, &a, &b, &ld);
    return WP_OK;
}

int wp_plan_execute(const wp_plan *plan, const float *x, float *y, int64_t C, int64_t N, int64_t ldx, int64_t ldy,
                    void *workspace, size_t workspace_bytes, wp_stream_t stream_) {
    cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
    if (!plan) return fail(WP_EINVAL, "plan is NULL");
    if (!x || !y) return fail(WP_EINVAL, "x and y must be device pointers");
    if (C < 1 || N < 1) return fail(WP_EINVAL, "need channels >= 1 and frames >= 1");
    if (ldx < N || ldy < N) return fail(WP_EINVAL, "row stride smaller than frames");
    {
        const char *xb = reinterpret_cast<const char *>(x), *xe = xb + sizeof(float) * ((C - 1) * ldx + N);
        const char *yb = reinterpret_cast<const char *>(y), *ye = yb + sizeof(float) * ((C - 1) * ldy + N);
        if (xb < ye && yb < xe) return fail(WP_EINVAL, "x and y overlap");
    }
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != plan->device) return fail(WP_EINVAL, "plan was created on another device");
    size_t rec_off, tmp_off;
    int64_t ld_tmp;
    const size_t need = ws_layout(plan, C, N, &rec_off, &tmp_off, &ld_tmp);
    if (!workspace || workspace_bytes < need)
        return fail(WP_ENOMEM, "workspace too small: need " + std::to_string(need) + " bytes");
    unsigned char *ws = reinterpret_cast<unsigned char *>(workspace);
    unsigned int *counter = reinterpret_cast<unsigned int *>(ws);
    unsigned int *peak = reinterpret_cast<unsigned int *>(ws + 64);
    float *tmp = reinterpret_cast<float *>(ws + tmp_off);
    const int P = (int)plan->passes.size();
    const float *in = x;
    int64_t ld_in = ldx;
    for (int i = 0; i < P; ++i) {
        const Pass &p = plan->passes[i];
        const bool to_y = ((P - 1 - i) % 2) == 0;
        float *out = to_y ? y : tmp;
        const int64_t ld_out = to_y ? ldy : ld_tmp;
        cudaError_t e;
        if (p.kind == Pass::NORMALIZE) {
            e = cudaMemsetAsync(peak, 0, sizeof(unsigned int), stream);
            if (e != cudaSuccess) return cuda_fail(e, "memset(peak)");
            e = wp::launch_peak_abs(in, C, N, ld_in, peak, stream);
            if (e != cudaSuccess) return cuda_fail(e, "peak_abs launch");
            e = wp::launch_scale_by_peak(in, out, C, N, ld_in, ld_out, peak, (float)p.target, stream);
            if (e != cudaSuccess) return cuda_fail(e, "scale launch");
        } else if (uses_lb(p, C, N)) {
            const long long tiles = ((N + wpk::CT_TOUT - 1) / wpk::CT_TOUT) * C;
            if (tiles >= (1LL << 31)) return fail(WP_EUNSUP, "more than 2^31 tiles in one call");
            unsigned long long *tr = (g_trace && g_trace_entries >= (size_t)tiles * wpk::LB_TRACE_EV) ? g_trace : nullptr;
            e = wp::lb_launch(p.lbp, in, out, C, N, ld_in, ld_out, ws + rec_off, tr, stream);
            if (e != cudaSuccess) return cuda_fail(e, "chain_lb launch");
        } else if (p.fft) {
            wpk::FftArgs a{};
            a.x = in;
            a.y = out;
            a.C = C;
            a.N = N;
            a.ldx = ld_in;
            a.ldy = ld_out;
            a.Tpad = p.fft_Tpad;
            a.L = p.Lout;
            a.nblk = (N + a.L - 1) / a.L;
            a.total = a.nblk * ((C + 1) / 2);
            a.tw = p.d_tw;
            const int grid = (int)std::min<long long>(a.total, p.grid_cap);
            for (int j = 0; j < p.fft_segs; ++j) {
                // segment j: taps [j K, (j + 1) K) convolve x delayed by j K, added to the first
                a.H = p.d_H + (size_t)j * wpk::FFT_M;
                a.delay = (long long)j * kFftSegTaps;
                a.accumulate = j > 0;
                e = wp::launch_fft_ols(a, grid, stream);
                if (e != cudaSuccess) return cuda_fail(e, "fft_ols launch");
            }
        } else if (p.fir_tc) {
            wpk::FirTcArgs a{};
            a.x = in;
            a.y = out;
            a.C = C;
            a.N = N;
            a.ldx = ld_in;
            a.ldy = ld_out;
            a.total_tiles = ((N + wpk::TC_TOUT - 1) / wpk::TC_TOUT) * C;
            a.Tp = p.tc_Tp;
            a.K = p.tc_K;
            a.W = p.tc_W;
            a.nin = p.tc_nin;
            a.Bimg = p.d_Bimg;
            a.out_scale = p.tc_out_scale;
            a.pre_gain = p.pre;
            a.n_post = (int)p.post.size();
            for (int j = 0; j < a.n_post; ++j) a.post[j] = p.post[j];
            a.vec_x = (ld_in % 4 == 0) && (reinterpret_cast<uintptr_t>(in) % 16 == 0);
            a.vec_y = (ld_out % 4 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
            a.trace = (g_trace && g_trace_entries >= (size_t)a.total_tiles * wpk::FT_TRACE_EV) ? g_trace : nullptr;
            if (a.total_tiles >= (1LL << 31)) return fail(WP_EUNSUP, "more than 2^31 tiles in one call");
            CUtensorMap ymap;
            std::memset(&ymap, 0, sizeof ymap);
            a.tma_y = a.vec_y && wp::encode_ymap(ymap, out, C, N, ld_out) ? 1 : 0;
            const int grid = (int)std::min<long long>(a.total_tiles, p.grid_cap);
            e = wp::launch_fir_tc(a, ymap, grid, p.smem, stream);
            if (e != cudaSuccess) return cuda_fail(e, "fir_tc launch");
        } else {
            wpk::FusedArgs a{};
            a.x = in;
            a.y = out;
            a.C = C;
            a.N = N;
            a.ldx = ld_in;
            a.ldy = ld_out;
            a.Lout = p.Lout;
            a.H = p.H;
            a.Tpad = p.Tpad;
            a.vec_x = (ld_in % 4 == 0) && (reinterpret_cast<uintptr_t>(in) % 16 == 0);
            a.vec_y = (ld_out % 4 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
            a.taps = p.d_taps;
            a.pre_gain = p.pre;
            a.n_post = (int)p.post.size();
            for (int j = 0; j < a.n_post; ++j) a.post[j] = p.post[j];
            a.G = p.d_G;
            a.TP = p.d_TP;
            a.counter = counter;
            a.recs = ws + rec_off;
            const long long tpc = tiles_per_channel(p, N);
            a.total_tiles = tpc * C;
            // look-back records are zeroed by every launch (stream-ordered, so a
            // captured CUDA graph replays correctly); flags then carry epoch 1
            a.epoch = 1;
            e = cudaMemsetAsync(a.recs, 0, rec_bytes(p) * (size_t)a.total_tiles, stream);
            if (e != cudaSuccess) return cuda_fail(e, "memset(records)");
            const int grid = (int)std::min<long long>(a.total_tiles, p.grid_cap);
            e = cudaMemsetAsync(counter, 0, sizeof(unsigned int), stream);
            if (e != cudaSuccess) return cuda_fail(e, "memset(counter)");
            e = p.f64 ? wp::launch_fused_f64(p.S, p.T > 0, a, p.tables, grid, p.smem, stream)
                      : wp::launch_fused_f32(p.S, p.T > 0, a, p.tables, grid, p.smem, stream);
            if (e != cudaSuccess) return cuda_fail(e, "fused kernel launch");
        }
        in = out;
        ld_in = ld_out;
    }
    return WP_OK;
}

// ---- host -> device -> host streaming (the e2e path of Wave.numpy32) ----
// Per device: an upload, a run and a download stream plus an event ring. One
// mutex per process serialises the ENQUEUE of concurrent calls (the work
// itself runs asynchronously), so an event is never re-recorded between a
// call's record and the wait that consumes it.
namespace {
constexpr int kHostMaxBlocks = 32;
struct HostStreams {
    cudaStream_t in = nullptr, run = nullptr, out = nullptr;
    cudaEvent_t start = nullptr, ev_in[kHostMaxBlocks] = {}, ev_run[kHostMaxBlocks] = {}, done = nullptr;
};
std::mutex g_host_mu;
std::map<int, HostStreams> g_host;

int host_streams(int dev, HostStreams **out) {
    auto it = g_host.find(dev);
    if (it != g_host.end()) {
        *out = &it->second;
        return WP_OK;
    }
    HostStreams h;
    cudaError_t e = cudaStreamCreateWithFlags(&h.in, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h.run, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h.out, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h.start, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h.done, cudaEventDisableTiming);
    for (int i = 0; i < kHostMaxBlocks && e == cudaSuccess; ++i) {
        e = cudaEventCreateWithFlags(&h.ev_in[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h.ev_run[i], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) return cuda_fail(e, "stream/event creation");
    *out = &(g_host[dev] = h);
    return WP_OK;
}
}  // namespace

int wp_plan_execute_host(const wp_plan *plan, const float *hx, float *hy, int64_t C, int64_t N, int64_t ld_hx,
                         int64_t ld_hy, float *dx, float *dy, void *workspace, size_t workspace_bytes,
                         int32_t blocks, wp_stream_t stream_) {
    cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
    if (!plan) return fail(WP_EINVAL, "plan is NULL");
    if (!hx || !hy || !dx || !dy) return fail(WP_EINVAL, "host and device buffers must be non-NULL");
    if (C < 1 || N < 1) return fail(WP_EINVAL, "need channels >= 1 and frames >= 1");
    if (ld_hx < N || ld_hy < N) return fail(WP_EINVAL, "row stride smaller than frames");
    if (dx == dy) return fail(WP_EINVAL, "dx and dy must be distinct [C x N] device buffers");
    bool pairs = false;  // the FFT path filters channel pairs together: pair-aligned blocks
    for (const Pass &p : plan->passes) pairs = pairs || (p.kind != Pass::NORMALIZE && p.fft);
    for (const Pass &p : plan->passes)
        if (p.kind == Pass::NORMALIZE)
            return fail(WP_EUNSUP, "a chain with Normalize needs the whole signal's peak: run wp_plan_execute");
    struct RouteGuard {
        explicit RouteGuard(long long c) { t_route_C = c; }
        ~RouteGuard() { t_route_C = 0; }
    } route(C);
    const int64_t units = pairs ? (C + 1) / 2 : C;
    // default: 16 blocks (same-box probes: cfg3's 737 MB 2-3 % faster than 32:
    // per-block copy/launch overhead), 32 from 4 GiB on (shorter ramp)
    const int64_t dflt = (int64_t)sizeof(float) * C * N >= (4LL << 30) ? kHostMaxBlocks : 16;
    int64_t nb = blocks > 0 ? blocks : dflt;
    nb = std::max<int64_t>(1, std::min<int64_t>({nb, units, (int64_t)kHostMaxBlocks}));
    // contiguous blocks of units (as sharding.partition: the first r blocks one unit larger)
    int64_t bounds[kHostMaxBlocks + 1];
    size_t need = 0;
    for (int64_t b = 0, a = 0; b <= nb; ++b) {
        const int64_t u = b * (units / nb) + std::min<int64_t>(b, units % nb);
        bounds[b] = std::min<int64_t>(C, pairs ? 2 * u : u);
        if (b > 0) {
            size_t r_off, t_off, w;
            int64_t ld;
            w = ws_layout(plan, bounds[b] - a, N, &r_off, &t_off, &ld);
            need = std::max(need, w);
        }
        a = bounds[b];
    }
    if (!workspace || workspace_bytes < need)
        return fail(WP_ENOMEM, "workspace too small: need " + std::to_string(need) + " bytes");
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != plan->device) return fail(WP_EINVAL, "plan was created on another device");
    std::lock_guard<std::mutex> lk(g_host_mu);
    HostStreams *h = nullptr;
    if (int rc = host_streams(dev, &h)) return rc;
    cudaError_t e = cudaEventRecord(h->start, stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->in, h->start, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->run, h->start, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->out, h->start, 0);
    if (e != cudaSuccess) return cuda_fail(e, "stream ordering");
    const size_t row = sizeof(float) * (size_t)N;
    int rc = WP_OK;
    for (int64_t b = 0; b < nb && rc == WP_OK; ++b) {
        const int64_t a = bounds[b], c = bounds[b + 1] - bounds[b];
        if (c <= 0) continue;
        e = cudaMemcpy2DAsync(dx + a * N, row, hx + a * ld_hx, sizeof(float) * ld_hx, row, c,
                              cudaMemcpyHostToDevice, h->in);
        if (e == cudaSuccess) e = cudaEventRecord(h->ev_in[b], h->in);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(h->run, h->ev_in[b], 0);
        if (e != cudaSuccess) {
            rc = cuda_fail(e, "upload");
            break;
        }
        rc = wp_plan_execute(plan, dx + a * N, dy + a * N, c, N, N, N, workspace, workspace_bytes,
                             reinterpret_cast<wp_stream_t>(h->run));
        if (rc != WP_OK) break;
        e = cudaEventRecord(h->ev_run[b], h->run);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(h->out, h->ev_run[b], 0);
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(hy + a * ld_hy, sizeof(float) * ld_hy, dy + a * N, row, row, c,
                                  cudaMemcpyDeviceToHost, h->out);
        if (e != cudaSuccess) rc = cuda_fail(e, "download");
    }
    // even after an error, the caller's stream waits for everything already
    // enqueued on the three streams (its buffers must outlive that work)
    e = cudaEventRecord(h->ev_in[0], h->in);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->out, h->ev_in[0], 0);
    if (e == cudaSuccess) e = cudaEventRecord(h->ev_run[0], h->run);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->out, h->ev_run[0], 0);
    if (e == cudaSuccess) e = cudaEventRecord(h->done, h->out);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, h->done, 0);
    if (e != cudaSuccess && rc == WP_OK) rc = cuda_fail(e, "stream ordering");
    return rc;
}

// ---- seam-level one-shot entry points with a small plan cache ----
// Plans are shared (std::shared_ptr): a caller holds its reference for the
// duration of the execute call, so evicting an entry never frees a plan that
// another thread is still using (the last holder destroys it; cudaFree
// synchronizes the device, so in-flight launches complete first).
static std::mutex g_cache_mu;
static std::map<std::string, std::pair<std::shared_ptr<wp_plan>, unsigned long long>> g_cache;
static unsigned long long g_cache_clock = 0;

static int cached_plan(const wp_stage &st, std::shared_ptr<wp_plan> *out) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::string key((const char *)&st.kind, sizeof st.kind);
    key.append((const char *)&st.flags, sizeof st.flags);
    key.append((const char *)&dev, sizeof dev);
    key.append((const char *)st.coef, sizeof(double) * (size_t)st.n * (st.kind == WP_STAGE_IIR ? 5 : 1));
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        auto it = g_cache.find(key);
        if (it != g_cache.end()) {
            it->second.second = ++g_cache_clock;
            *out = it->second.first;
            return WP_OK;
        }
    }
    wp_plan *raw = nullptr;
    const int rc = wp_plan_create(&st, 1, &raw);
    if (rc != WP_OK) return rc;
    std::shared_ptr<wp_plan> sp(raw, [](wp_plan *p) { wp_plan_destroy(p); });
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cache.find(key);
    if (it != g_cache.end()) {  // another thread built the same plan meanwhile
        *out = it->second.first;
        return WP_OK;
    }
    if (g_cache.size() >= 64) {
        // evict the least recently used entry (holders keep it alive)
        auto lru = g_cache.begin();
        for (auto jt = g_cache.begin(); jt != g_cache.end(); ++jt)
            if (jt->second.second < lru->second.second) lru = jt;
        g_cache.erase(lru);
    }
    g_cache[key] = {sp, ++g_cache_clock};
    *out = sp;
    return WP_OK;
}

static int seam_workspace(const wp_stage &st, int64_t channels, int64_t frames, size_t *bytes) {
    if (!bytes) return fail(WP_EINVAL, "bytes is NULL");
    std::shared_ptr<wp_plan> plan;
    const int rc = cached_plan(st, &plan);
    if (rc != WP_OK) return rc;
    return wp_plan_workspace_bytes(plan.get(), channels, frames, bytes);
}

int wp_iir_cascade(const double *sos, int32_t n_sections, const float *x, float *y, int64_t channels, int64_t frames,
                   int64_t ld_x, int64_t ld_y, int32_t flags, void *workspace, size_t workspace_bytes,
                   wp_stream_t stream) {
    wp_stage st{WP_STAGE_IIR, n_sections, sos, 0.0, flags, 0};
    if (n_sections < 1 || !sos) return fail(WP_EINVAL, "need >= 1 section");
    std::shared_ptr<wp_plan> plan;
    int rc = cached_plan(st, &plan);
    if (rc != WP_OK) return rc;
    return wp_plan_execute(plan.get(), x, y, channels, frames, ld_x, ld_y, workspace, workspace_bytes, stream);
}

int wp_iir_cascade_workspace(const double *sos, int32_t n_sections, int64_t channels, int64_t frames, int32_t flags,
                             size_t *bytes) {
    if (n_sections < 1 || !sos) return fail(WP_EINVAL, "need >= 1 section");
    return seam_workspace(wp_stage{WP_STAGE_IIR, n_sections, sos, 0.0, flags, 0}, channels, frames, bytes);
}

int wp_fir(const double *taps, int32_t n_taps, const float *x, float *y, int64_t channels, int64_t frames, int64_t ld_x,
           int64_t ld_y, int32_t flags, void *workspace, size_t workspace_bytes, wp_stream_t stream) {
    wp_stage st{WP_STAGE_FIR, n_taps, taps, 0.0, flags, 0};
    if (n_taps < 1 || !taps) return fail(WP_EINVAL, "need >= 1 tap");
    std::shared_ptr<wp_plan> plan;
    int rc = cached_plan(st, &plan);
    if (rc != WP_OK) return rc;
    return wp_plan_execute(plan.get(), x, y, channels, frames, ld_x, ld_y, workspace, workspace_bytes, stream);
}

int wp_fir_workspace(const double *taps, int32_t n_taps, int64_t channels, int64_t frames, int32_t flags,
                     size_t *bytes) {
    if (n_taps < 1 || !taps) return fail(WP_EINVAL, "need >= 1 tap");
    return seam_workspace(wp_stage{WP_STAGE_FIR, n_taps, taps, 0.0, flags, 0}, channels, frames, bytes);
}

int wp_white_noise(float *y, int64_t channels, int64_t frames, int64_t ld_y, uint64_t seed, wp_stream_t stream) {
    if (!y || channels < 1 || frames < 1 || ld_y < frames) return fail(WP_EINVAL, "bad noise arguments");
    int rc = arch_ok();
    if (rc != WP_OK) return rc;
    cudaError_t e = wp::launch_white_noise(y, channels, frames, ld_y, seed, reinterpret_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? WP_OK : cuda_fail(e, "white_noise launch");
}

int wp_wav_decode(const void *payload, int32_t encoding, float *y, int64_t channels, int64_t frames, int64_t ld_y,
                  wp_stream_t stream) {
    if (!payload || !y || channels < 1 || frames < 1 || ld_y < frames) return fail(WP_EINVAL, "bad wav decode arguments");
    if (encoding != WP_ENC_PCM16 && encoding != WP_ENC_PCM24 && encoding != WP_ENC_F32)
        return fail(WP_EINVAL, "encoding must be 16 (pcm16), 24 (pcm24) or 32 (float32)");
    int rc = arch_ok();
    if (rc != WP_OK) return rc;
    cudaError_t e = wp::launch_wav_decode(payload, encoding, y, channels, frames, ld_y, reinterpret_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? WP_OK : cuda_fail(e, "wav decode launch");
}

int wp_wav_encode(const float *x, int64_t channels, int64_t frames, int64_t ld_x, int32_t encoding, void *payload,
                  uint64_t *clipped_device, wp_stream_t stream) {
    if (!x || !payload || channels < 1 || frames < 1 || ld_x < frames) return fail(WP_EINVAL, "bad wav encode arguments");
    if (encoding != WP_ENC_PCM16 && encoding != WP_ENC_PCM24 && encoding != WP_ENC_F32)
        return fail(WP_EINVAL, "encoding must be 16 (pcm16), 24 (pcm24) or 32 (float32)");
    if (encoding != WP_ENC_F32 && !clipped_device) return fail(WP_EINVAL, "pcm encodings need a clipped-count buffer");
    int rc = arch_ok();
    if (rc != WP_OK) return rc;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (clipped_device) {
        cudaError_t e0 = cudaMemsetAsync(clipped_device, 0, sizeof(uint64_t), s);
        if (e0 != cudaSuccess) return cuda_fail(e0, "memset(clipped)");
    }
    cudaError_t e = wp::launch_wav_encode(x, channels, frames, ld_x, encoding, payload,
                                          reinterpret_cast<unsigned long long *>(clipped_device), s);
    return e == cudaSuccess ? WP_OK : cuda_fail(e, "wav encode launch");
}

int wp_peak_abs(const float *x, int64_t channels, int64_t frames, int64_t ld_x, float *out_device, wp_stream_t stream) {
    if (!x || !out_device || channels < 1 || frames < 1 || ld_x < frames) return fail(WP_EINVAL, "bad peak arguments");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemsetAsync(out_device, 0, sizeof(float), s);
    if (e != cudaSuccess) return cuda_fail(e, "memset(peak)");
    e = wp::launch_peak_abs(x, channels, frames, ld_x, reinterpret_cast<unsigned int *>(out_device), s);
    return e == cudaSuccess ? WP_OK : cuda_fail(e, "peak launch");
}

}  // extern "C"
