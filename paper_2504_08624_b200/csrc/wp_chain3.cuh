// Decoupled tensor-core chain for sm_100a: pre-gain -> IIR SOS cascade -> FIR
// -> post-gains as three kernels with NO serial dependency between tiles
// inside any of them.
//
// Replaces the reference's per-stage passes (_iir_channel, _kernels_jit.py:
// 14-32; _fir_channel, :51-62; Chain.apply's stage loop, chain.py:66-71).
//
// Same LTI formulation as wp_chain_tc.cuh: for tile rows
// m = 0..127 of 64 outputs (n = n0 + 64 m + p), window start w_m = n0 - H + 64 m,
//
//   y[n] = sum_{k < H+64} g[p + H - k] x[w_m + k]  +  sum_i E[p][i] s_{w_m}[i]
//   s_{w_{m+1}} = M s_{w_m} + e_m,   e_m = sum_j A^(63-j) B x[w_m + j],  M = A^64
//
// The single-kernel version chains tiles through a decoupled look-back, so a
// tile's output waits on the aggregates of tiles other SMs are processing at
// the same moment; the whole pipeline then runs at the latency of that chain.
// Here the recurrence is split along its data dependencies:
//
//   chain_rows   (CUDA cores, every tile independent)  e_m in TS from the fp32
//                samples, Kogge-Stone row scan, zero-carry row prefixes L_m
//                -> HBM (D TS per row), tile aggregate -> HBM
//   chain_carry  (one CTA per channel, tiny)  carry_k = state entering tile k:
//                blocked scan over the channel's tile aggregates
//   chain_gemm   (tensor cores, every tile independent)  main GEMM fp16 x3 into
//                TMEM, then the state term as a tf32 GEMM into the SAME
//                accumulator: s_m = L_m + M^m carry_k split into three tf32
//                parts x E split into three tf32 parts (6 MMAs, K = 8), so the
//                epilogue is TMEM -> scale -> store.
//
// Extra HBM traffic: the samples are read twice and the row prefixes
// (D * sizeof(TS) / 64 bytes per sample) are written once and read once.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "wp_chain_tc.cuh"

namespace wpk {

constexpr int C3_THREADS = 512;
constexpr int C3_NA = 4;          // TMEM accumulator stages (128 columns each)
constexpr int C3_CONV = 192;      // converter threads (warps 2..7)
constexpr int C3_QMAX = 11;       // float4 of the window per converter thread (W <= 8448)
constexpr int C3_ROWS_THREADS = 128;
constexpr int C3_CARRY_THREADS = 256;

struct C3RowsArgs {
    const float *x;
    long long C, N, ldx;
    long long total_tiles;
    int H;
    int vec_x;
    const void *G;  // [D][D][33] TS, M^l lane-minor
    void *rows;     // [tiles][128][D] TS: zero-carry row prefixes within the tile
    void *aggs;     // [tiles][D] TS: tile aggregates
};

template <typename TS, int D>
struct C3RowsTables {
    TS K[64][D];     // A^(63-j) B
    TS P[7][D][D];   // M^(2^i)
    TS W[4][D][D];   // M^(32 w)
};

struct C3CarryArgs {
    long long C, T;  // channels, tiles per channel
    int B;           // tiles per thread
    unsigned long long *trace;  // optional: [C][8] globaltimer stamps of thread 255
    const void *aggs;
    void *carry;     // [tiles][4][D] TS: state entering rows 0, 32, 64, 96 of each tile
};

template <typename TS, int D>
struct C3CarryTables {
    TS MT[D][D];     // M^128: one tile
    TS Q[5][D][D];   // MT^(B 2^i)
    TS R[D][D];      // MT^(32 B): one warp of threads
    TS W[3][D][D];   // M^(32 w), w = 1..3: carries of a tile's row quarters
};

struct C3GemmArgs {
    const float *x;
    float *y;
    long long C, N, ldx, ldy;
    long long total_tiles;
    int H, K, W;
    const unsigned char *Bimg;  // [2][atoms][64 rows][128 B] SW128 K-major fp16 hi / lo of g
    const unsigned char *Eimg;  // [3][64 rows][8] tf32 parts of E, no-swizzle K-major, 32-B rows
    float out_scale;            // 2^-fB of the g image
    double st_scale;            // 2^fB: state operand s' = s * sc * st_scale
    const void *G;              // [D][D][33] TS
    const void *rows;           // [tiles][128][D] TS
    const void *carry;          // [tiles][4][D] TS
    int vec_x, vec_y;
    int dbg;                    // diagnostics: 4 = no state term
    unsigned long long *trace;  // optional: [tiles][C3_TRACE_EV] globaltimer stamps
};
constexpr int C3_TRACE_EV = 10;

namespace c3d {

// no-swizzle K-major, 32-byte rows: core matrices of 8 rows x 16 B, LBO = 128 B
// (next core matrix along K), SBO = 256 B (next 8-row group) (tools/tf32_probe.cu)
__host__ __device__ __forceinline__ uint32_t off32(int r, int k) {
    return (uint32_t)((r >> 3) * 256 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
}

__device__ __forceinline__ uint64_t desc32(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)(128u >> 4) << 16;
    d |= (uint64_t)(256u >> 4) << 32;
    d |= (uint64_t)1u << 46;
    return d;
}

// no-swizzle K-major: LBO = 128 B (next core matrix along K), SBO = sbo (next 8-row group)
__device__ __forceinline__ uint64_t desc_sbo(uint32_t saddr, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)(128u >> 4) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1u << 46;
    return d;
}

__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(a), "l"(b), "r"(idesc)
                 : "memory");
}

__device__ __forceinline__ float tf32_rna(float f) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(f));
    return __uint_as_float(r);
}

// v = t1 + t2 + t3 (+ O(2^-33 |v|)), each part exact in tf32
__device__ __forceinline__ void split3(double v, float &t1, float &t2, float &t3) {
    t1 = tf32_rna((float)v);
    const double r1 = v - (double)t1;
    t2 = tf32_rna((float)r1);
    t3 = tf32_rna((float)(r1 - (double)t2));
}
__device__ __forceinline__ void split3(float v, float &t1, float &t2, float &t3) {
    t1 = tf32_rna(v);
    const float r1 = v - t1;
    t2 = tf32_rna(r1);
    t3 = tf32_rna(r1 - t2);
}

// programmatic dependent launch: let the next kernel in the stream start its
// prologue now / wait until the previous kernel has completed and flushed
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void arrive_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

// window of one tile: start sample and the bulk-copyable range [lo, hi)
struct Win {
    long long c, n0, start, lo, hi;
};
__device__ __forceinline__ Win win(long long tile, long long C, long long N, int H, int W, int vec_x) {
    Win g;
    g.c = (long long)((unsigned)tile % (unsigned)C);
    g.n0 = (long long)((unsigned)tile / (unsigned)C) * (long long)CT_TOUT;
    g.start = g.n0 - H;
    g.lo = g.start > 0 ? g.start : 0;
    const long long nv = vec_x ? (N & ~3LL) : 0;
    long long hi = g.start + W;
    if (hi > nv) hi = nv;
    g.hi = hi > g.lo ? hi : g.lo;
    return g;
}

// out += M v, M block lower triangular (2x2 blocks): one FMA chain per row
// (independent rows / segments give the ILP)
template <int D, typename TS, typename F>
__device__ __forceinline__ void matvec_fma(TS (&out)[D], const TS (&v)[D], F m) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
        const int nj = 2 * ((i >> 1) + 1);
#pragma unroll
        for (int j = 0; j < D; ++j)
            if (j < nj) out[i] = fma(m(i, j), v[j], out[i]);
    }
}

template <typename TS, int D>
__device__ __forceinline__ void store_vec(TS *dst, const TS (&v)[D]) {
    if constexpr ((sizeof(TS) * D) % 16 == 0) {
#pragma unroll
        for (int q = 0; q < (int)(sizeof(TS) * D / 16); ++q)
            reinterpret_cast<uint4 *>(dst)[q] = reinterpret_cast<const uint4 *>(v)[q];
    } else {
#pragma unroll
        for (int d = 0; d < D; ++d) dst[d] = v[d];
    }
}

template <typename TS, int D>
__device__ __forceinline__ void load_vec(TS (&v)[D], const TS *src) {
    if constexpr ((sizeof(TS) * D) % 16 == 0) {
#pragma unroll
        for (int q = 0; q < (int)(sizeof(TS) * D / 16); ++q)
            reinterpret_cast<uint4 *>(v)[q] = __ldcg(reinterpret_cast<const uint4 *>(src) + q);
    } else {
#pragma unroll
        for (int d = 0; d < D; ++d) v[d] = ldcg(src + d);
    }
}

}  // namespace c3d

// ---------------------------------------------------------------------------
// chain_rows: one warp per tile (persistent, static stride over tiles), no CTA
// barrier. Lane l owns rows 4l..4l+3: four independent e accumulations (every
// coefficient read from shared memory feeds four rows), a serial scan over its
// four rows, one Kogge-Stone over the lanes, and the rows' exclusive prefixes.
// The samples stream through a per-warp ring of RSTG shared-memory stages
// (8 samples x 128 rows each) filled by cp.async, RSTG - 1 steps ahead: four
// stages at 3 CTAs/SM for the fp64 scan (register-bound), three stages at 4
// CTAs/SM for fp32 (measured best for each).
template <typename TS>
__host__ __device__ constexpr int c3_rstg() { return sizeof(TS) == 8 ? 4 : 3; }
template <typename TS>
__host__ __device__ constexpr int c3_rows_ctas() { return sizeof(TS) == 8 ? 3 : 4; }
template <typename TS>
__host__ __device__ constexpr int c3_rows_smem() { return (C3_ROWS_THREADS / 32) * c3_rstg<TS>() * 4096; }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// byte offset of (row, 16-byte half h) inside a stage: rows of 32 B, four rows
// per 128-B line; the 16-B chunk position is XOR-swizzled by the line index so
// that lanes reading rows 4l + g (g fixed) hit distinct banks
__device__ __forceinline__ uint32_t rs_off(int row, int h) {
    return (uint32_t)((row >> 2) * 128 + 16 * ((((row & 3) << 1) | h) ^ ((row >> 2) & 7)));
}

// edge / unaligned tiles: guarded loads straight into the stage (kept out of
// line so the hot loop's code stays small)
static __device__ __noinline__ void rows_fill_slow(unsigned char *stage, const float *xr, long long t0, int q, int lane,
                                            long long N, int vec_x) {
#pragma unroll 1
    for (int j = 0; j < 8; ++j) {
        const int row = (lane >> 1) + 16 * j;
        const long long pos = t0 + 64LL * row + 8 * q + 4 * (lane & 1);
        *reinterpret_cast<float4 *>(stage + rs_off(row, lane & 1)) = load_region4(xr, pos, N, vec_x);
    }
}

template <typename TS, int S>
__global__ void __launch_bounds__(C3_ROWS_THREADS, c3_rows_ctas<TS>()) chain_rows_kernel(const C3RowsArgs a,
                                                                        const C3RowsTables<TS, 2 * S> tb) {
    constexpr int D = 2 * S;
    constexpr int NWR = C3_ROWS_THREADS / 32;
    __shared__ __align__(16) TS Ks[64][D];
    constexpr int C3_RSTG = c3_rstg<TS>();
    extern __shared__ __align__(16) unsigned char ring[];  // [NWR][C3_RSTG][128 rows x 32 B]
    const int tid = threadIdx.x, lane = tid & 31, wr = tid >> 5;
    c3d::pdl_trigger();  // chain_carry may be scheduled; it waits for this grid to finish
    for (int i = tid; i < 64 * D; i += C3_ROWS_THREADS) Ks[i / D][i % D] = tb.K[i / D][i % D];
    __syncthreads();
    TS *rows = reinterpret_cast<TS *>(a.rows);
    TS *aggs = reinterpret_cast<TS *>(a.aggs);
    unsigned char *myring = ring + (size_t)wr * C3_RSTG * 4096;
    const uint32_t ring0 = wptc::smem_u32(myring);
    // this lane's copy chunks: rows (lane >> 1) + 16 j, half lane & 1
    uint32_t soff[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) soff[j] = rs_off((lane >> 1) + 16 * j, lane & 1);
    const long long nwarps = (long long)gridDim.x * NWR;
    auto mt1 = [&](int r, int q) { return tb.P[0][r][q]; };  // M: one row
    for (long long tile = (long long)blockIdx.x * NWR + wr; tile < a.total_tiles; tile += nwarps) {
        const long long c = (long long)((unsigned long long)tile % (unsigned long long)a.C);
        const long long k = (long long)((unsigned long long)tile / (unsigned long long)a.C);
        const float *xr = a.x + c * a.ldx;
        const long long t0 = k * CT_TOUT - a.H;
        const bool fast = a.vec_x && t0 >= 0 && t0 + CT_TOUT <= a.N;
        const float *gp = xr + t0 + 64 * (lane >> 1) + 4 * (lane & 1);
        auto fill = [&](int q) {
            const uint32_t so = (uint32_t)(q % C3_RSTG) * 4096u;
            if (fast) {
#pragma unroll
                for (int j = 0; j < 8; ++j) cp_async16(ring0 + so + soff[j], gp + 1024 * j + 8 * q);
            } else {
                rows_fill_slow(myring + so, xr, t0, q, lane, a.N, a.vec_x);
            }
        };
        __syncwarp();  // the previous tile's reads of the ring are done
#pragma unroll
        for (int q = 0; q < C3_RSTG - 1; ++q) {
            fill(q);
            cp_async_commit();
        }
        // lane l: rows 4 l + g
        TS e[4][D];
#pragma unroll
        for (int g = 0; g < 4; ++g)
#pragma unroll
            for (int d = 0; d < D; ++d) e[g][d] = TS(0);
#pragma unroll 1
        for (int q = 0; q < 8; ++q) {
            if (q + C3_RSTG - 1 < 8) fill(q + C3_RSTG - 1);
            cp_async_commit();
            cp_async_wait<C3_RSTG - 1>();
            __syncwarp();
            const unsigned char *stg = myring + (q % C3_RSTG) * 4096;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float4 xv4[4];
#pragma unroll
                for (int g = 0; g < 4; ++g) xv4[g] = *reinterpret_cast<const float4 *>(stg + rs_off(4 * lane + g, h));
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    TS xv[4];
#pragma unroll
                    for (int g = 0; g < 4; ++g)
                        xv[g] = (TS)(u == 0 ? xv4[g].x : u == 1 ? xv4[g].y : u == 2 ? xv4[g].z : xv4[g].w);
                    const TS *kr = &Ks[8 * q + 4 * h + u][0];
#pragma unroll
                    for (int d = 0; d < D; ++d) {
                        const TS kc = kr[d];
#pragma unroll
                        for (int g = 0; g < 4; ++g) e[g][d] = fma(kc, xv[g], e[g][d]);
                    }
                }
            }
            __syncwarp();  // stage q is refilled C3_RSTG - 1 steps later
        }
        // serial scan over the lane's 4 rows (zero carry), then a Kogge-Stone over
        // lanes with M^(4 2^i), then the rows' exclusive prefixes
        TS t[D];
#pragma unroll
        for (int d = 0; d < D; ++d) t[d] = e[0][d];
#pragma unroll
        for (int g = 1; g < 4; ++g) {
            TS nt[D];
#pragma unroll
            for (int d = 0; d < D; ++d) nt[d] = e[g][d];
            c3d::matvec_fma<D, TS>(nt, t, mt1);
#pragma unroll
            for (int d = 0; d < D; ++d) t[d] = nt[d];
        }
#pragma unroll
        for (int stp = 0; stp < 5; ++stp) {
            const int off = 1 << stp;
            TS prev[D];
#pragma unroll
            for (int d = 0; d < D; ++d) prev[d] = shfl_up(t[d], off);
            if (lane >= off) c3d::matvec_fma<D, TS>(t, prev, [&](int r, int q) { return tb.P[stp + 2][r][q]; });
        }
        if (lane == 31) c3d::store_vec<TS, D>(aggs + (size_t)tile * D, t);
        TS Lm[D];
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const TS u = shfl_up(t[d], 1);
            Lm[d] = lane == 0 ? TS(0) : u;
        }
        TS *dst = rows + ((size_t)tile * CT_ROWS + 4 * lane) * D;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            c3d::store_vec<TS, D>(dst + g * D, Lm);
            if (g < 3) {
                TS nl[D];
#pragma unroll
                for (int d = 0; d < D; ++d) nl[d] = e[g][d];
                c3d::matvec_fma<D, TS>(nl, Lm, mt1);
#pragma unroll
                for (int d = 0; d < D; ++d) Lm[d] = nl[d];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// chain_carry: one CTA per channel over its T tiles; thread t owns tiles
// [t B, (t+1) B).
template <typename TS, int S>
__global__ void __launch_bounds__(C3_CARRY_THREADS) chain_carry_kernel(const C3CarryArgs a,
                                                                       const C3CarryTables<TS, 2 * S> tb) {
    constexpr int D = 2 * S;
    constexpr int NWC = C3_CARRY_THREADS / 32;
    __shared__ TS wt[NWC][D];
    const int tid = threadIdx.x, lane = tid & 31, wq = tid >> 5;
    const long long c = blockIdx.x;
    const long long j0 = (long long)tid * a.B;
    const long long j1 = j0 + a.B < a.T ? j0 + a.B : a.T;
    const TS *aggs = reinterpret_cast<const TS *>(a.aggs);
    TS *carry = reinterpret_cast<TS *>(a.carry);
    auto seg = [&](long long j) { return (size_t)(j * a.C + c) * D; };
    auto stamp = [&](int ev) {
        if (a.trace && tid == C3_CARRY_THREADS - 1) a.trace[c * 8 + ev] = ctd::gtimer();
    };
    stamp(0);
    c3d::pdl_trigger();  // chain_gemm may start its main GEMMs
    c3d::pdl_wait();     // chain_rows' aggregates are complete
    stamp(1);
    auto mt = [&](int r, int q) { return tb.MT[r][q]; };
    // local inclusive prefix of this thread's segments (zero carry)
    TS loc[D];
#pragma unroll
    for (int d = 0; d < D; ++d) loc[d] = TS(0);
    {
        TS nxt[D];
        if (j0 < j1) c3d::load_vec<TS, D>(nxt, aggs + seg(j0));
#pragma unroll 1
        for (long long j = j0; j < j1; ++j) {
            TS cur[D];
#pragma unroll
            for (int d = 0; d < D; ++d) cur[d] = nxt[d];
            if (j + 1 < j1) c3d::load_vec<TS, D>(nxt, aggs + seg(j + 1));
            c3d::matvec_fma<D, TS>(cur, loc, mt);
#pragma unroll
            for (int d = 0; d < D; ++d) loc[d] = cur[d];
        }
    }
    stamp(2);
    // warp scan over threads (blocks of exactly B segments before any short one)
    TS incl[D];
#pragma unroll
    for (int d = 0; d < D; ++d) incl[d] = loc[d];
#pragma unroll
    for (int stp = 0; stp < 5; ++stp) {
        const int off = 1 << stp;
        TS prev[D];
#pragma unroll
        for (int d = 0; d < D; ++d) prev[d] = shfl_up(incl[d], off);
        if (lane >= off) ctd::matvec_tree<D, TS>(incl, prev, [&](int r, int q) { return tb.Q[stp][r][q]; });
    }
    if (lane == 31) {
#pragma unroll
        for (int d = 0; d < D; ++d) wt[wq][d] = incl[d];
    }
    __syncthreads();
    stamp(3);
    TS ex[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const TS u = shfl_up(incl[d], 1);
        ex[d] = lane == 0 ? TS(0) : u;
    }
    {
        // carry entering this warp (Horner): wc = MT^(32 B) wc + wt_u, u < wq
        TS wc[D];
#pragma unroll
        for (int d = 0; d < D; ++d) wc[d] = TS(0);
#pragma unroll 1
        for (int u = 0; u < wq; ++u) {
            TS nw[D];
#pragma unroll
            for (int d = 0; d < D; ++d) nw[d] = wt[u][d];
            ctd::matvec_tree<D, TS>(nw, wc, [&](int r, int q) { return tb.R[r][q]; });
#pragma unroll
            for (int d = 0; d < D; ++d) wc[d] = nw[d];
        }
        // ex += MT^(B lane) wc: apply the Q powers by the bits of lane
#pragma unroll
        for (int b = 0; b < 5; ++b) {
            if ((lane >> b) & 1) {
                TS z[D];
#pragma unroll
                for (int d = 0; d < D; ++d) z[d] = TS(0);
                ctd::matvec_tree<D, TS>(z, wc, [&](int r, int q) { return tb.Q[b][r][q]; });
#pragma unroll
                for (int d = 0; d < D; ++d) wc[d] = z[d];
            }
        }
#pragma unroll
        for (int d = 0; d < D; ++d) ex[d] += wc[d];
    }
    stamp(4);
    // replay: carry of each owned segment
    {
        TS nxt[D];
        if (j0 < j1) c3d::load_vec<TS, D>(nxt, aggs + seg(j0));
#pragma unroll 1
        for (long long j = j0; j < j1; ++j) {
            TS cur[D];
#pragma unroll
            for (int d = 0; d < D; ++d) cur[d] = nxt[d];
            if (j + 1 < j1) c3d::load_vec<TS, D>(nxt, aggs + seg(j + 1));
            // state entering rows 0, 32, 64, 96 of tile j
            TS *cq = carry + seg(j) * 4;
            c3d::store_vec<TS, D>(cq, ex);
#pragma unroll
            for (int w = 0; w < 3; ++w) {
                TS vq[D];
#pragma unroll
                for (int d = 0; d < D; ++d) vq[d] = TS(0);
                c3d::matvec_fma<D, TS>(vq, ex, [&](int r, int q) { return tb.W[w][r][q]; });
                c3d::store_vec<TS, D>(cq + (w + 1) * D, vq);
            }
            c3d::matvec_fma<D, TS>(cur, ex, mt);
#pragma unroll
            for (int d = 0; d < D; ++d) ex[d] = cur[d];
        }
    }
    stamp(5);
}

// ---------------------------------------------------------------------------
// chain_gemm: persistent, one CTA per SM, warp-specialized.
struct C3Layout {
    uint32_t opBytes, bBytes;
    uint32_t rawBytes;
    uint32_t bimg, eimg, op, sop, raw, g, stg, misc, bars;
    uint32_t total;
    __host__ __device__ C3Layout(int W, int K, int D, int ts, int nop) {
        opBytes = ((uint32_t)W * 2u + 1023u) & ~1023u;
        bBytes = (uint32_t)((K + 63) / 64) * 8192u;  // one part; the image is [atom][hi rows | lo rows]
        bimg = 0;
        eimg = bimg + 2 * bBytes;
        op = eimg + 3 * 2048u;
        sop = op + 2u * (uint32_t)nop * opBytes;  // op: [nop stages][hi, lo]
        raw = sop + 2u * 3u * 4096u;        // sop: [2 stages][3 parts][128 rows x 32 B]
        rawBytes = ((uint32_t)W * 4u + 1023u) & ~1023u;
        g = raw + rawBytes;                 // raw: one fp32 window (bulk copy)
        stg = (g + (uint32_t)(ts * lt_size(D) * 32) + 15u) & ~15u;
        misc = stg + 4u * 32u * CT_STG_PITCH;  // scl[8] f32, red[8] f32, stag[8] i32
        bars = (misc + 96u + 15u) & ~15u;
        total = bars + 20 * 8 + 16 + 1024;  // + alignment slack
    }
};

template <typename TS, int S, int NOP>
__global__ void __launch_bounds__(C3_THREADS, 1) chain_gemm_kernel(const C3GemmArgs a) {
    static_assert(NOP == 2 || NOP == 3, "two or three fp16 operand stages");
    constexpr int D = 2 * S;
    static_assert(D <= 8, "state operand holds K = 8 columns");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024u - (wptc::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nk = a.K / 16;
    const C3Layout lay(a.W, a.K, D, (int)sizeof(TS), NOP);
#define C3TR(tile, ev) \
    do {                                                                              \
        if (a.trace) a.trace[(long long)(tile) * C3_TRACE_EV + (ev)] = ctd::gtimer(); \
    } while (0)
    unsigned char *bimg = smem + lay.bimg;
    unsigned char *op = smem + lay.op;
    unsigned char *sop = smem + lay.sop;
    TS *gsm = reinterpret_cast<TS *>(smem + lay.g);
    unsigned char *stg = smem + lay.stg;
    float *scl = reinterpret_cast<float *>(smem + lay.misc);  // [8] ring by local tile
    float *red = scl + 8;                                     // [8]
    int *stag = reinterpret_cast<int *>(red + 8);             // [8] local tile index of scl[]
    unsigned long long *bars = reinterpret_cast<unsigned long long *>(smem + lay.bars);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 20);
    const uint32_t bar0 = wptc::smem_u32(bars);
    // barriers: OP_FULL, OP_EMPTY, SOP_FULL, SOP_EMPTY x 2 stages; ACC_FULL, ACC_EMPTY x 4 stages
#define OPF(s) (bar0 + 8u * (uint32_t)(0 + (s)))
#define OPE(s) (bar0 + 8u * (uint32_t)(3 + (s)))
#define SOF(s) (bar0 + 8u * (uint32_t)(6 + (s)))
#define SOE(s) (bar0 + 8u * (uint32_t)(8 + (s)))
#define ACF(s) (bar0 + 8u * (uint32_t)(10 + (s)))
#define ACE(s) (bar0 + 8u * (uint32_t)(14 + (s)))
#define RWF (bar0 + 8u * 18u)
#define RWE (bar0 + 8u * 19u)

    if (warp == 0) wptc::tmem_alloc(wptc::smem_u32(tmem_slot), 128 * C3_NA);
    if (tid == 32) {
        for (int s = 0; s < NOP; ++s) {
            wptc::mbar_init(OPF(s), 1);
            wptc::mbar_init(OPE(s), 1);
        }
        for (int s = 0; s < 2; ++s) {
            wptc::mbar_init(SOF(s), CT_ROWS);
            wptc::mbar_init(SOE(s), 1);
        }
        for (int s = 0; s < C3_NA; ++s) {
            wptc::mbar_init(ACF(s), 1);
            wptc::mbar_init(ACE(s), CT_ROWS);
        }
        wptc::mbar_init(RWF, 1);
        wptc::mbar_init(RWE, 1);
        wptc::mbar_fence_init();
    }
    for (int i = tid; i < (int)(2 * lay.bBytes / 16); i += C3_THREADS)
        reinterpret_cast<uint4 *>(bimg)[i] = reinterpret_cast<const uint4 *>(a.Bimg)[i];
    for (int i = tid; i < 3 * 2048 / 16; i += C3_THREADS)
        reinterpret_cast<uint4 *>(smem + lay.eimg)[i] = reinterpret_cast<const uint4 *>(a.Eimg)[i];
    for (int i = tid; i < 2 * 3 * 4096 / 16; i += C3_THREADS)  // state columns >= D stay zero
        reinterpret_cast<uint4 *>(sop)[i] = make_uint4(0u, 0u, 0u, 0u);
    if (tid < 8) stag[tid] = -1;
    {
        const TS *G = reinterpret_cast<const TS *>(a.G);
        for (int i = tid; i < D * D * 32; i += C3_THREADS) {
            const int r = i / (D * 32), q = (i / 32) % D, l = i % 32;
            if (q < lt_nj(r)) gsm[(lt_off(r) + q) * 32 + l] = G[(r * D + q) * 33 + l];
        }
    }
    wptc::fence_proxy_async_smem();
    wptc::fence_before_sync();
    __syncthreads();
    wptc::fence_after_sync();
    const uint32_t tmem = *tmem_slot;
    const long long first = blockIdx.x, stride = gridDim.x;
    const int ntiles = first < a.total_tiles ? (int)((a.total_tiles - 1 - first) / stride + 1) : 0;

    if (warp == 0) {
        // ================= MMA issuer =================
        if (lane == 0) {
            const uint32_t idesc = wptc::idesc_f16(128, 64), idesc2 = wptc::idesc_f16(128, 128);
            const uint32_t idt = c3d::idesc_tf32(128, 64);
            const uint32_t op0 = wptc::smem_u32(op), b0 = wptc::smem_u32(bimg);
            const uint32_t sop0 = wptc::smem_u32(sop), e0 = wptc::smem_u32(smem + lay.eimg);
            for (int i = 0; i < ntiles; ++i) {
                const int s = i & 1;  // state operand stage
                const uint32_t par = (uint32_t)((i >> 1) & 1);
                const int so = i % NOP;  // fp16 operand stage
                const uint32_t paro = (uint32_t)((i / NOP) & 1);
                const int sa = i % C3_NA;
                const uint32_t para = (uint32_t)((i / C3_NA) & 1);
                C3TR(first + (long long)i * stride, 8);
                wptc::mbar_wait(OPF(so), paro);
                C3TR(first + (long long)i * stride, 9);
                wptc::mbar_wait(ACE(sa), para ^ 1u);
                wptc::fence_after_sync();
                C3TR(first + (long long)i * stride, 2);
                // columns [0, 64): x_hi g_hi + x_lo g_hi (+ state term); [64, 128): x_hi g_lo
                const uint32_t dm = tmem + 128u * sa;
                const uint32_t ahi = op0 + (2u * so) * lay.opBytes, alo = ahi + lay.opBytes;
                const uint64_t ah0 = ctd::desc_sw128(ahi), al0 = ctd::desc_sw128(alo);
#pragma unroll 1
                for (int kk = 0; kk < nk; ++kk) {
                    const uint64_t ka = 2u * kk;  // +32 B per K step, across rows (Hankel)
                    const uint64_t bb = ctd::desc_sw128(b0 + 16384u * (kk >> 2) + 32u * (kk & 3));
                    wptc::mma_f16(dm, ah0 + ka, bb, idesc2, kk > 0);
                    wptc::mma_f16(dm, al0 + ka, bb, idesc, 1u);
                }
                wptc::mma_commit(OPE(so));  // the operand stage is free once the main GEMM has read it
                C3TR(first + (long long)i * stride, 3);
                wptc::mbar_wait(SOF(s), par);
                wptc::fence_after_sync();
                if (!(a.dbg & 4)) {
                    // state term: parts (i, j) with i + j < 3 of s' x E
#pragma unroll
                    for (int pr = 0; pr < 6; ++pr) {
                        // (s' part, E part): (0,0) (0,1) (1,0) (0,2) (1,1) (2,0)
                        const int ia = pr == 2 || pr == 4 ? 1 : pr == 5 ? 2 : 0;
                        const int ib = pr == 1 || pr == 4 ? 1 : pr == 3 ? 2 : 0;
                        c3d::mma_tf32(dm, c3d::desc32(sop0 + (uint32_t)(s * 3 + ia) * 4096u),
                                      c3d::desc32(e0 + (uint32_t)ib * 2048u), idt);
                    }
                }
                wptc::mma_commit(SOE(s));
                wptc::mma_commit(ACF(sa));
            }
        }
    } else if (warp == 1) {
        // ================= bulk-copy producer: fp32 window -> smem =================
        if (lane == 0) {
            const uint32_t raw0 = wptc::smem_u32(smem + lay.raw);
            for (int i = 0; i < ntiles; ++i) {
                wptc::mbar_wait(RWE, (uint32_t)(i & 1) ^ 1u);
                const c3d::Win g = c3d::win(first + (long long)i * stride, a.C, a.N, a.H, a.W, a.vec_x);
                const uint32_t bytes = (uint32_t)(4 * (g.hi - g.lo));
                if (bytes > 0) {
                    c3d::arrive_tx(RWF, bytes);
                    const float *src = a.x + g.c * a.ldx + g.lo;
                    const uint32_t dst = raw0 + 4u * (uint32_t)(g.lo - g.start);
                    // pieces of <= 16 KB
                    for (uint32_t o = 0; o < bytes; o += 16384u) {
                        const uint32_t nb = bytes - o < 16384u ? bytes - o : 16384u;
                        c3d::bulk_g2s(dst + o, reinterpret_cast<const unsigned char *>(src) + o, nb, RWF);
                    }
                } else {
                    ctd::arrive(RWF);
                }
                // warm L2 with the window after next
                const long long nt = first + (long long)(i + 2) * stride;
                if (i + 2 < ntiles) {
                    const c3d::Win g2 = c3d::win(nt, a.C, a.N, a.H, a.W, a.vec_x);
                    const uint32_t b2 = (uint32_t)(4 * (g2.hi - g2.lo));
                    if (b2 > 0) ctd::prefetch_l2(a.x + g2.c * a.ldx + g2.lo, b2);
                }
            }
        }
    } else if (warp >= 2 && warp <= 7) {
        // ================= converters (warps 2..7): fp32 window -> SW128 fp16 hi / lo =================
        const int ct = tid - 64;
        const int cw = ct >> 5;
        const int nq = a.W / 4;
        const float4 *raw4 = reinterpret_cast<const float4 *>(smem + lay.raw);
        for (int i = 0; i < ntiles; ++i) {
            const int s = i % NOP;
            const uint32_t par = (uint32_t)((i / NOP) & 1);
            const c3d::Win g = c3d::win(first + (long long)i * stride, a.C, a.N, a.H, a.W, a.vec_x);
            const float *xr = a.x + g.c * a.ldx;
            const bool interior = g.start >= g.lo && g.start + a.W <= g.hi;
            wptc::mbar_wait(RWF, (uint32_t)(i & 1));
            if (ct == 0) C3TR(first + (long long)i * stride, 0);
            float4 v[C3_QMAX];
            float m = 0.f;
            if (interior) {
#pragma unroll
                for (int j = 0; j < C3_QMAX; ++j)
                    v[j] = (ct + j * C3_CONV < nq) ? raw4[ct + j * C3_CONV] : make_float4(0.f, 0.f, 0.f, 0.f);
            } else {
#pragma unroll 1
                for (int j = 0; j < C3_QMAX; ++j) {
                    const int q = ct + j * C3_CONV;
                    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (q < nq) {
                        const long long p0 = g.start + 4LL * q;
                        if (p0 >= g.lo && p0 + 4 <= g.hi) {
                            t = raw4[q];
                        } else {
                            t.x = (p0 + 0 >= 0 && p0 + 0 < a.N) ? __ldg(xr + p0 + 0) : 0.f;
                            t.y = (p0 + 1 >= 0 && p0 + 1 < a.N) ? __ldg(xr + p0 + 1) : 0.f;
                            t.z = (p0 + 2 >= 0 && p0 + 2 < a.N) ? __ldg(xr + p0 + 2) : 0.f;
                            t.w = (p0 + 3 >= 0 && p0 + 3 < a.N) ? __ldg(xr + p0 + 3) : 0.f;
                        }
                    }
#pragma unroll
                    for (int jj = 0; jj < C3_QMAX; ++jj)
                        if (jj == j) v[jj] = t;
                }
            }
#pragma unroll
            for (int j = 0; j < C3_QMAX; ++j)
                m = fmaxf(m, fmaxf(fmaxf(fabsf(v[j].x), fabsf(v[j].y)), fmaxf(fabsf(v[j].z), fabsf(v[j].w))));
            const unsigned mb = __reduce_max_sync(0xffffffffu, __float_as_uint(m));
            if (lane == 0) red[cw] = __uint_as_float(mb);
            ctd::named_sync(1, C3_CONV);
            if (ct == 0) ctd::arrive(RWE);  // the window is in registers: free it
            float tmax = red[0];
#pragma unroll
            for (int w = 1; w < C3_CONV / 32; ++w) tmax = fmaxf(tmax, red[w]);
            int ex = 0;
            if (tmax > 0.f) frexpf(tmax, &ex);
            const float sc = ldexpf(1.f, tmax > 0.f ? 14 - ex : 0);
            wptc::mbar_wait(OPE(s), par ^ 1u);
            unsigned char *ohi = op + (2 * s) * lay.opBytes, *olo = ohi + lay.opBytes;
#pragma unroll
            for (int j = 0; j < C3_QMAX; ++j) {
                const int q = ct + j * C3_CONV;
                if (q < nq) {
                    const float2 f01 = make_float2(v[j].x * sc, v[j].y * sc);
                    const float2 f23 = make_float2(v[j].z * sc, v[j].w * sc);
                    const __half2 h01 = __float22half2_rn(f01), h23 = __float22half2_rn(f23);
                    const float2 b01 = __half22float2(h01), b23 = __half22float2(h23);
                    const __half2 l01 = __floats2half2_rn(f01.x - b01.x, f01.y - b01.y);
                    const __half2 l23 = __floats2half2_rn(f23.x - b23.x, f23.y - b23.y);
                    uint2 hv, lv;
                    hv.x = *reinterpret_cast<const uint32_t *>(&h01);
                    hv.y = *reinterpret_cast<const uint32_t *>(&h23);
                    lv.x = *reinterpret_cast<const uint32_t *>(&l01);
                    lv.y = *reinterpret_cast<const uint32_t *>(&l23);
                    const uint32_t off = ctd::swz128(8u * (uint32_t)q);
                    *reinterpret_cast<uint2 *>(ohi + off) = hv;
                    *reinterpret_cast<uint2 *>(olo + off) = lv;
                }
            }
            if (ct == 0) {
                scl[i & 7] = sc;
                __threadfence_block();
                *reinterpret_cast<volatile int *>(stag + (i & 7)) = i;
            }
            wptc::fence_proxy_async_smem();
            ctd::named_sync(2, C3_CONV);
            if (ct == 0) {
                ctd::arrive(OPF(s));
                C3TR(first + (long long)i * stride, 1);
            }
        }
    } else if (warp >= 8 && warp <= 11) {
        // ================= state operand (warps 8..11), one tile row per thread =================
        const int wq = warp & 3;
        const int row = 32 * wq + lane;
        const TS *rows = reinterpret_cast<const TS *>(a.rows);
        const TS *carry = reinterpret_cast<const TS *>(a.carry);
        TS Ln[D], Cn[D];
        c3d::pdl_wait();  // row prefixes and carries of chain_rows / chain_carry are complete
        if (ntiles > 0) {
            c3d::load_vec<TS, D>(Ln, rows + ((size_t)first * CT_ROWS + row) * D);
            c3d::load_vec<TS, D>(Cn, carry + ((size_t)first * 4 + wq) * D);
        }
        for (int i = 0; i < ntiles; ++i) {
            const int s = i & 1;
            const uint32_t par = (uint32_t)((i >> 1) & 1);
            TS sv[D], cv[D];
#pragma unroll
            for (int d = 0; d < D; ++d) sv[d] = Ln[d], cv[d] = Cn[d];
            if (i + 1 < ntiles) {
                const long long nt = first + (long long)(i + 1) * stride;
                c3d::load_vec<TS, D>(Ln, rows + ((size_t)nt * CT_ROWS + row) * D);
                c3d::load_vec<TS, D>(Cn, carry + ((size_t)nt * 4 + wq) * D);
            }
            // s_m = L_m + M^lane (M^(32 wq) carry)
            ctd::matvec_tree<D, TS>(sv, cv, [&](int r, int q) { return gsm[(lt_off(r) + q) * 32 + lane]; });
            if (row == 0) C3TR(first + (long long)i * stride, 4);
            // the tile's input scale: tagged ring slot (absolute local tile index,
            // so no barrier-phase aliasing however far the converters run ahead)
            for (int spins = 0; *reinterpret_cast<volatile int *>(stag + (i & 7)) != i; ++spins) {
                __nanosleep(32);
                if (spins > (1 << 28)) __trap();  // watchdog
            }
            __threadfence_block();
            const TS f = (TS)scl[i & 7] * (TS)a.st_scale;
            wptc::mbar_wait(SOE(s), par ^ 1u);
            unsigned char *dst = sop + (size_t)s * 3 * 4096;
#pragma unroll
            for (int d = 0; d < D; ++d) {
                float t1, t2, t3;
                c3d::split3(sv[d] * f, t1, t2, t3);
                const uint32_t o = c3d::off32(row, d);
                *reinterpret_cast<float *>(dst + o) = t1;
                *reinterpret_cast<float *>(dst + 4096 + o) = t2;
                *reinterpret_cast<float *>(dst + 8192 + o) = t3;
            }
            wptc::fence_proxy_async_smem();
            ctd::arrive(SOF(s));
            if (row == 0) C3TR(first + (long long)i * stride, 5);
        }
    } else if (warp >= 12) {
        // ================= epilogue (warps 12..15): TMEM -> scale -> coalesced stores =================
        const int wq = warp & 3;
        const uint32_t trow = (uint32_t)(32 * wq) << 16;
        unsigned char *mystg = stg + (size_t)wq * 32 * CT_STG_PITCH;
        for (int i = 0; i < ntiles; ++i) {
            const int sa = i % C3_NA;
            const long long tile = first + (long long)i * stride;
            const long long c = (long long)((unsigned)tile % (unsigned)a.C);
            const long long n0 = (long long)((unsigned)tile / (unsigned)a.C) * (long long)CT_TOUT;
            wptc::mbar_wait(ACF(sa), (uint32_t)((i / C3_NA) & 1));
            wptc::fence_after_sync();
            if (tid == 384) C3TR(tile, 6);
            const float osc = a.out_scale / scl[i & 7];
            const uint32_t tbase = tmem + 128u * sa + trow;
            float *yr = a.y + c * a.ldy + n0;
            const long long tleft = a.N - n0;
            const bool full = a.vec_y && tleft >= CT_TOUT;
#pragma unroll 1
            for (int ch = 0; ch < 4; ++ch) {
                const int h = ch >> 1, hh = ch & 1;
                float t16[16], u16[16];
                ctd::tmem_ld16(tbase + 16u * ch, t16);
                ctd::tmem_ld16(tbase + 64u + 16u * ch, u16);
                wptc::tmem_wait_ld();
                if (ch == 3) {
                    wptc::fence_before_sync();
                    ctd::arrive(ACE(sa));
                }
                float4 *dst = reinterpret_cast<float4 *>(mystg + lane * CT_STG_PITCH + 64 * hh);
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4)
                    dst[q4] = make_float4((t16[4 * q4] + u16[4 * q4]) * osc, (t16[4 * q4 + 1] + u16[4 * q4 + 1]) * osc,
                                          (t16[4 * q4 + 2] + u16[4 * q4 + 2]) * osc,
                                          (t16[4 * q4 + 3] + u16[4 * q4 + 3]) * osc);
                if (hh == 1) {
                    __syncwarp();
                    if (full) {
#pragma unroll
                        for (int r = 0; r < 8; ++r) {
                            const int q = lane + 32 * r;
                            const int rr = q >> 3, c4 = q & 7;
                            const float4 v = *reinterpret_cast<const float4 *>(mystg + rr * CT_STG_PITCH + 16 * c4);
                            __stcs(reinterpret_cast<float4 *>(yr + 64 * (32 * wq + rr) + 32 * h + 4 * c4), v);
                        }
                    } else {
#pragma unroll 1
                        for (int r = 0; r < 8; ++r) {
                            const int q = lane + 32 * r;
                            const int rr = q >> 3, c4 = q & 7;
                            const float4 v = *reinterpret_cast<const float4 *>(mystg + rr * CT_STG_PITCH + 16 * c4);
                            const int o = 64 * (32 * wq + rr) + 32 * h + 4 * c4;
                            const long long left = tleft - o;
                            if (a.vec_y && left >= 4) {
                                __stcs(reinterpret_cast<float4 *>(yr + o), v);
                            } else {
                                if (left > 0) yr[o + 0] = v.x;
                                if (left > 1) yr[o + 1] = v.y;
                                if (left > 2) yr[o + 2] = v.z;
                                if (left > 3) yr[o + 3] = v.w;
                            }
                        }
                    }
                    __syncwarp();
                }
            }
            if (tid == 384) C3TR(tile, 7);
        }
    }
#undef C3TR
#undef OPF
#undef OPE
#undef SOF
#undef SOE
#undef ACF
#undef ACE
#undef RWF
#undef RWE
    wptc::fence_before_sync();
    __syncthreads();
    wptc::fence_after_sync();
    if (warp == 0) wptc::tmem_dealloc(tmem, 128 * C3_NA);
}

}  // namespace wpk
