// fp64 (complex128) instantiations of the fused overlap-save kernel.
#include "kernels_impl.cuh"

namespace fcvbw_gpu {
template <>
bool plan_info<double>(int N, LaunchInfo* out) { return plan_info_impl<double>(N, out); }
template <>
cudaError_t launch_ols<double>(int N, int mode, const OlsArgs<double>& a, size_t smem_extra, int max_grid,
                              cudaStream_t s, int* grid_used) {
    return launch_ols_impl<double>(N, mode, a, smem_extra, max_grid, s, grid_used);
}
}  // namespace fcvbw_gpu
