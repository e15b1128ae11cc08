// Synthetic workload generator on the device (bench / test utility, not part of the reference
// interface): the unit-variance complex Gaussian stream of paper_2406_14116_b200/workload.py
// (complex_gaussian), regenerated on the GPU so that the 2^30- and 2^31-sample BASELINE inputs are
// produced in milliseconds instead of minutes of host Box-Muller, identically at every GPU count:
// sample i of channel c depends only on (seed_base + c, i), never on how channels or block ranges
// are split across ranks.
//
//   key = splitmix64(seed), h1 = splitmix64(key ^ 2i), h2 = splitmix64(key ^ (2i + 1))
//   u1 = ((h1 >> 11) + 1) 2^-53 in (0, 1], u2 = (h2 >> 11) 2^-53 in [0, 1)
//   x_i = sqrt(-ln u1) (cos 2 pi u2 + j sin 2 pi u2)     (Re, Im ~ N(0, 1/2): E|x|^2 = 1)
//
// Device log / sin / cos are within 1-2 ulp of the host libm the Python generator uses, so the two
// streams agree to ~1e-16 relative in fp64 (and almost always bitwise after rounding to fp32);
// parity tests feed the oracle the samples the GPU actually consumed.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/fcvbw_gpu.h"

namespace fcvbw_gpu_detail {
void set_last_error(const std::string& m);
}

namespace {

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

template <class R>
__global__ void gaussian_kernel(R* x, int64_t S, int channels, int64_t ch_stride, uint64_t seed_base,
                                int64_t ch_first, int64_t start) {
    const int64_t total = S * int64_t(channels);
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t c = e / S, i = e - c * S;
        const uint64_t key = splitmix64(seed_base + uint64_t(ch_first + c));
        const uint64_t idx = uint64_t(start + i);
        const uint64_t h1 = splitmix64(key ^ (idx * 2ULL));
        const uint64_t h2 = splitmix64(key ^ (idx * 2ULL + 1ULL));
        const double u1 = (double(h1 >> 11) + 1.0) * 0x1.0p-53;
        const double u2 = double(h2 >> 11) * 0x1.0p-53;
        const double r = sqrt(-log(u1));
        const double ang = 2.0 * 3.141592653589793 * u2;
        R* p = x + 2 * (c * ch_stride + i);
        p[0] = static_cast<R>(r * cos(ang));
        p[1] = static_cast<R>(r * sin(ang));
    }
}

}  // namespace

extern "C" int fcvbw_gpu_fill_gaussian(void* x_dev, int dtype, int64_t S, int channels, int64_t ch_stride,
                                       uint64_t seed_base, int64_t ch_first, int64_t start, void* stream) {
    if (S < 0 || channels < 0 || ch_stride < S || (S > 0 && channels > 0 && !x_dev) ||
        (dtype != FCVBW_GPU_C64 && dtype != FCVBW_GPU_C128)) {
        fcvbw_gpu_detail::set_last_error("fill_gaussian: bad arguments");
        return FCVBW_GPU_VALIDATION;
    }
    if (S == 0 || channels == 0) return FCVBW_GPU_OK;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dtype == FCVBW_GPU_C64)
        gaussian_kernel<float><<<sms * 8, 256, 0, st>>>(static_cast<float*>(x_dev), S, channels, ch_stride, seed_base,
                                                       ch_first, start);
    else
        gaussian_kernel<double><<<sms * 8, 256, 0, st>>>(static_cast<double*>(x_dev), S, channels, ch_stride,
                                                        seed_base, ch_first, start);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fcvbw_gpu_detail::set_last_error(std::string("fill_gaussian: ") + cudaGetErrorString(e));
        return FCVBW_GPU_ERROR;
    }
    return FCVBW_GPU_OK;
}
