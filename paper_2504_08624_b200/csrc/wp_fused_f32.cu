// fp32 instantiations of the fused chain kernel (scan and recurrence in fp32),
// plus the IIR-free variants (FIR only / gain only).
#include "wp_fused_launch.cuh"

namespace wp {

cudaError_t launch_fused_f32(int S, bool fir, const wpk::FusedArgs &a, const HostTables &t, int grid, size_t smem,
                             cudaStream_t st) {
    if (S == 0) {
        return fir ? launch_one<float, 0, true>(a, t, grid, smem, st) : launch_one<float, 0, false>(a, t, grid, smem, st);
    }
    return launch_dispatch<float>(S, fir, a, t, grid, smem, st);
}

int fused_occupancy_f32(int S, bool fir, size_t smem) {
    if (S == 0) return fir ? occupancy_one<float, 0, true>(smem) : occupancy_one<float, 0, false>(smem);
    return occupancy_dispatch<float>(S, fir, smem);
}

size_t fused_smem_bytes_f32(int S, int tpad) {
    switch (S) {
        case 0: return wpk::SmemLayout<float, 0>::total(tpad);
        case 1: return wpk::SmemLayout<float, 1>::total(tpad);
        case 2: return wpk::SmemLayout<float, 2>::total(tpad);
        case 3: return wpk::SmemLayout<float, 3>::total(tpad);
        default: return wpk::SmemLayout<float, 4>::total(tpad);
    }
}

}  // namespace wp
