// complex fp64 instantiations of the fused overlap-save kernel (one translation unit per sample
// type and I/O layout so that nvcc compiles them in parallel).
#include "kernels_impl.cuh"

namespace fcvbw_gpu {
template <>
bool plan_info<double>(int N, LaunchInfo* out) { return plan_info_impl<double>(N, out); }
template <>
cudaError_t launch_ols_io<double, 0>(int N, int mode, const OlsArgs<double>& a, size_t smem_extra, int max_grid,
                                  cudaStream_t s, int* grid_used) {
    return launch_ols_impl<double, 0>(N, mode, a, smem_extra, max_grid, s, grid_used);
}
}  // namespace fcvbw_gpu
