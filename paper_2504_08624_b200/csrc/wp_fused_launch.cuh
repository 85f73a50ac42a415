// Template launcher for the fused kernel: converts float64 host tables into
// the by-value kernel parameter block of the requested scan dtype.
#pragma once

#include "wp_internal.h"

namespace wp {

template <typename TS, int S>
static wpk::IirTables<TS, S> make_tables(const HostTables &t) {
    wpk::IirTables<TS, S> tb{};
    if constexpr (S > 0) {
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
    }
    return tb;
}

template <typename TS, int S, bool FIR>
static cudaError_t launch_one(const wpk::FusedArgs &a, const HostTables &t, int grid, size_t smem, cudaStream_t st) {
    auto kern = wpk::fused_chain_kernel<TS, S, FIR>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const wpk::IirTables<TS, S> tb = make_tables<TS, S>(t);
    kern<<<grid, wpk::NT, smem, st>>>(a, tb);
    count_launch();
    return cudaGetLastError();
}

template <typename TS, int S, bool FIR>
static int occupancy_one(size_t smem) {
    auto kern = wpk::fused_chain_kernel<TS, S, FIR>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, wpk::NT, smem) != cudaSuccess) return 0;
    return n;
}

template <typename TS>
static cudaError_t launch_dispatch(int S, bool fir, const wpk::FusedArgs &a, const HostTables &t, int grid,
                                   size_t smem, cudaStream_t st) {
#define WP_CASE(SS)                                                                        \
    case SS:                                                                               \
        return fir ? launch_one<TS, SS, true>(a, t, grid, smem, st)                        \
                   : launch_one<TS, SS, false>(a, t, grid, smem, st);
    switch (S) {
        WP_CASE(1)
        WP_CASE(2)
        WP_CASE(3)
        WP_CASE(4)
        default:
            return cudaErrorInvalidValue;
    }
#undef WP_CASE
}

template <typename TS>
static int occupancy_dispatch(int S, bool fir, size_t smem) {
#define WP_CASE(SS) \
    case SS:        \
        return fir ? occupancy_one<TS, SS, true>(smem) : occupancy_one<TS, SS, false>(smem);
    switch (S) {
        WP_CASE(1)
        WP_CASE(2)
        WP_CASE(3)
        WP_CASE(4)
        default:
            return 0;
    }
#undef WP_CASE
}

}  // namespace wp
