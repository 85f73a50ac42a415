// Instantiations and launchers of the tensor-core chain kernel
// (wp_chain_tc.cuh): scan dtype float64 or float32, 1..4 SOS sections.
#include "wp_chain_tc.cuh"
#include "wp_internal.h"

namespace wp {

namespace {

template <typename TS, int S>
wpk::IirTables<TS, S> ct_tables(const HostTables &t) {
    wpk::IirTables<TS, S> tb{};
    constexpr int D = 2 * S;
    for (int s = 0; s < S; ++s)
        for (int j = 0; j < 5; ++j) tb.sos[s][j] = TS(t.sos[s * 5 + j]);
    for (int n = 0; n < wpk::L; ++n)
        for (int i = 0; i < D; ++i) tb.K[n][i] = TS(t.K[n * D + i]);
    for (int q = 0; q < 5; ++q)
        for (int i = 0; i < D; ++i)
            for (int j = 0; j < D; ++j) tb.P[q][i][j] = TS(t.P[(q * D + i) * D + j]);
    for (int w = 0; w < wpk::NW; ++w)
        for (int i = 0; i < D; ++i)
            for (int j = 0; j < D; ++j) tb.W[w][i][j] = TS(t.W[(w * D + i) * D + j]);
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) tb.MT[i][j] = TS(t.MT[i * D + j]);
    return tb;
}

template <typename TS, int S>
cudaError_t ct_launch_one(const wpk::ChainTcArgs &a, const HostTables &t, const std::vector<double> &E, int grid,
                          size_t smem, cudaStream_t st) {
    constexpr int D = 2 * S;
    auto kern = wpk::chain_tc_kernel<TS, S>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const wpk::IirTables<TS, S> tb = ct_tables<TS, S>(t);
    wpk::ETable<TS, D> et{};
    for (int p = 0; p < 64; ++p)
        for (int i = 0; i < D; ++i) et.E[p][i] = TS(E[p * D + i]);
    kern<<<grid, wpk::CT_THREADS, smem, st>>>(a, tb, et);
    count_launch();
    return cudaGetLastError();
}

template <typename TS>
cudaError_t ct_dispatch(int S, const wpk::ChainTcArgs &a, const HostTables &t, const std::vector<double> &E, int grid,
                        size_t smem, cudaStream_t st) {
    switch (S) {
        case 1: return ct_launch_one<TS, 1>(a, t, E, grid, smem, st);
        case 2: return ct_launch_one<TS, 2>(a, t, E, grid, smem, st);
        case 3: return ct_launch_one<TS, 3>(a, t, E, grid, smem, st);
        case 4: return ct_launch_one<TS, 4>(a, t, E, grid, smem, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

size_t chain_tc_smem_bytes(int W, int K, int S, bool f64) {
    return wpk::CtLayout(W, K, 2 * S, f64 ? 8 : 4).total;
}

cudaError_t launch_chain_tc(bool f64, int S, const wpk::ChainTcArgs &a, const HostTables &t,
                            const std::vector<double> &E, int grid, size_t smem, cudaStream_t st) {
    return f64 ? ct_dispatch<double>(S, a, t, E, grid, smem, st) : ct_dispatch<float>(S, a, t, E, grid, smem, st);
}

}  // namespace wp
