// Instantiations and launchers of the decoupled tensor-core chain
// (wp_chain3.cuh): scan dtype float64 or float32, 1..4 SOS sections.
#include <algorithm>
#include <atomic>

#include "wp_chain3.cuh"
#include "wp_internal.h"

namespace wp {

namespace {

template <typename TS, int S>
wpk::C3RowsTables<TS, 2 * S> c3_rows_tables(const HostTables &t) {
    constexpr int D = 2 * S;
    wpk::C3RowsTables<TS, D> tb{};
    for (int n = 0; n < 64; ++n)
        for (int i = 0; i < D; ++i) tb.K[n][i] = TS(t.K[n * D + i]);
    // P[q] = M^(2^q), q < 7 (the host tables hold q < 5)
    std::vector<double> m(t.P.begin() + 4 * D * D, t.P.begin() + 5 * D * D);
    for (int q = 0; q < 7; ++q) {
        if (q >= 5) {
            std::vector<double> m2((size_t)D * D, 0.0);
            for (int i = 0; i < D; ++i)
                for (int j = 0; j < D; ++j) {
                    long double acc = 0;
                    for (int l = 0; l < D; ++l) acc += (long double)m[i * D + l] * m[l * D + j];
                    m2[i * D + j] = (double)acc;
                }
            m = m2;
        }
        for (int i = 0; i < D; ++i)
            for (int j = 0; j < D; ++j) tb.P[q][i][j] = TS(q < 5 ? t.P[(q * D + i) * D + j] : m[i * D + j]);
    }
    for (int w = 0; w < 4; ++w)
        for (int i = 0; i < D; ++i)
            for (int j = 0; j < D; ++j) tb.W[w][i][j] = TS(t.W[(w * D + i) * D + j]);
    return tb;
}

template <typename TS, int S>
cudaError_t c3_launch_one(const Chain3Launch &L, const HostTables &t, cudaStream_t st) {
    static_assert(sizeof(TS) >= 4, "scan dtype");
    constexpr int D = 2 * S;
    const wpk::C3RowsTables<TS, D> tb = c3_rows_tables<TS, S>(t);
    // chain_rows: persistent, as many CTAs as fit
    static std::atomic<int> rows_occ[64];  // per device; benign races write the same value
    int dev = 0;
    cudaGetDevice(&dev);
    dev = dev < 0 || dev >= 64 ? 0 : dev;
    cudaError_t e = cudaFuncSetAttribute(wpk::chain_rows_kernel<TS, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         wpk::c3_rows_smem<TS>());
    if (e != cudaSuccess) return e;
    if (!rows_occ[dev].load(std::memory_order_relaxed)) {
        int occ = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, wpk::chain_rows_kernel<TS, S>, wpk::C3_ROWS_THREADS,
                                                          wpk::c3_rows_smem<TS>());
        if (e != cudaSuccess) return e;
        rows_occ[dev].store(std::max(occ, 1), std::memory_order_relaxed);
    }
    const long long rg =
        std::min<long long>(L.rows.total_tiles, (long long)rows_occ[dev].load(std::memory_order_relaxed) * sm_count());
    wpk::chain_rows_kernel<TS, S><<<(unsigned)rg, wpk::C3_ROWS_THREADS, wpk::c3_rows_smem<TS>(), st>>>(L.rows, tb);
    count_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // chain_carry and chain_gemm use programmatic dependent launch: their CTAs
    // may start while the previous kernel drains; they wait (griddepcontrol)
    // before reading its output
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;
    // chain_carry: one CTA per channel
    wpk::C3CarryTables<TS, D> ct{};
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) {
            ct.MT[i][j] = TS(L.carry_mats[i * D + j]);
            for (int q = 0; q < 5; ++q) ct.Q[q][i][j] = TS(L.carry_mats[((1 + q) * D + i) * D + j]);
            ct.R[i][j] = TS(L.carry_mats[(6 * D + i) * D + j]);
            for (int w = 0; w < 3; ++w) ct.W[w][i][j] = TS(t.W[((w + 1) * D + i) * D + j]);
        }
    {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)L.carry.C);
        cfg.blockDim = dim3(wpk::C3_CARRY_THREADS);
        cfg.stream = st;
        cfg.attrs = pdl;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, wpk::chain_carry_kernel<TS, S>, L.carry, ct);
        if (e != cudaSuccess) return e;
    }
    count_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // chain_gemm: one CTA per SM
    auto kern = L.nop == 3 ? wpk::chain_gemm_kernel<TS, S, 3> : wpk::chain_gemm_kernel<TS, S, 2>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
    if (e != cudaSuccess) return e;
    {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)L.gemm_grid);
        cfg.blockDim = dim3(wpk::C3_THREADS);
        cfg.dynamicSmemBytes = L.smem;
        cfg.stream = st;
        cfg.attrs = pdl;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, kern, L.gemm);
        if (e != cudaSuccess) return e;
    }
    count_launch();
    return cudaGetLastError();
}

template <typename TS>
cudaError_t c3_dispatch(int S, const Chain3Launch &L, const HostTables &t, cudaStream_t st) {
    switch (S) {
        case 1: return c3_launch_one<TS, 1>(L, t, st);
        case 2: return c3_launch_one<TS, 2>(L, t, st);
        case 3: return c3_launch_one<TS, 3>(L, t, st);
        case 4: return c3_launch_one<TS, 4>(L, t, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

size_t chain3_smem_bytes(int W, int K, int S, bool f64, int nop) {
    return wpk::C3Layout(W, K, 2 * S, f64 ? 8 : 4, nop).total;
}

cudaError_t launch_chain3(bool f64, int S, const Chain3Launch &L, const HostTables &t, cudaStream_t st) {
    return f64 ? c3_dispatch<double>(S, L, t, st) : c3_dispatch<float>(S, L, t, st);
}

}  // namespace wp
