// f64 mask-dump instantiations of the fused overlap-save kernel (IO = 3: the complex kernel plus
// the write of the mask every item applies, for fcvbw_gpu_mask_dump; own translation unit so that
// nvcc compiles it in parallel and the production kernels carry no dump code).
#include "kernels_impl.cuh"

namespace fcvbw_gpu {
template <>
cudaError_t launch_ols_io<double, 3>(int N, int mode, const OlsArgs<double>& a, size_t smem_extra, int max_grid,
                                   cudaStream_t s, int* grid_used) {
    return launch_ols_impl<double, 3>(N, mode, a, smem_extra, max_grid, s, grid_used);
}
}  // namespace fcvbw_gpu
