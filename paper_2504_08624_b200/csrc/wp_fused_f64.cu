// fp64 instantiations of the fused chain kernel: used for IIR blocks with a
// pole radius above 0.98 (fp32 DF2T state fails the 1e-4
// bar on the 100 Hz high-pass of cfg3 with low-frequency input).
#include "wp_fused_launch.cuh"

namespace wp {

cudaError_t launch_fused_f64(int S, bool fir, const wpk::FusedArgs &a, const HostTables &t, int grid, size_t smem,
                             cudaStream_t st) {
    return launch_dispatch<double>(S, fir, a, t, grid, smem, st);
}

int fused_occupancy_f64(int S, bool fir, size_t smem) { return occupancy_dispatch<double>(S, fir, smem); }

size_t fused_smem_bytes_f64(int S, int tpad) {
    switch (S) {
        case 1: return wpk::SmemLayout<double, 1>::total(tpad);
        case 2: return wpk::SmemLayout<double, 2>::total(tpad);
        case 3: return wpk::SmemLayout<double, 3>::total(tpad);
        default: return wpk::SmemLayout<double, 4>::total(tpad);
    }
}

}  // namespace wp
