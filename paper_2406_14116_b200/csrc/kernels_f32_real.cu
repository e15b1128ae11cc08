// real-input f32 instantiations of the fused overlap-save kernel (IO = 1: raw tables, one real
// channel per transform; IO = 2: structured engines, block pairs per transform).
#include "kernels_impl.cuh"

namespace fcvbw_gpu {
template <>
cudaError_t launch_ols_io<float, 1>(int N, int mode, const OlsArgs<float>& a, size_t smem_extra, int max_grid,
                                  cudaStream_t s, int* grid_used) {
    return launch_ols_impl<float, 1>(N, mode, a, smem_extra, max_grid, s, grid_used);
}
template <>
cudaError_t launch_ols_io<float, 2>(int N, int mode, const OlsArgs<float>& a, size_t smem_extra, int max_grid,
                                  cudaStream_t s, int* grid_used) {
    return launch_ols_impl<float, 2>(N, mode, a, smem_extra, max_grid, s, grid_used);
}
}  // namespace fcvbw_gpu
