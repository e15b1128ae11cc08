// fp32 (complex64) instantiations of the fused overlap-save kernel.
#include "kernels_impl.cuh"

namespace fcvbw_gpu {
template <>
bool plan_info<float>(int N, LaunchInfo* out) { return plan_info_impl<float>(N, out); }
template <>
cudaError_t launch_ols<float>(int N, int mode, const OlsArgs<float>& a, size_t smem_extra, int max_grid,
                              cudaStream_t s, int* grid_used) {
    return launch_ols_impl<float>(N, mode, a, smem_extra, max_grid, s, grid_used);
}
}  // namespace fcvbw_gpu
