// Template launchers behind launch.cuh; included once per sample type.
#pragma once

#include "launch.cuh"

namespace fcvbw_gpu {

template <class R, int N, int MODE, int IO>
cudaError_t launch_one(const OlsArgs<R>& a, size_t smem_extra, int max_grid, cudaStream_t s,
                       int* grid_used) {
    using CH = Choice<R, N>;
    // the real block-pair path stages the pair's union segment in the exchange buffer wherever the
    // complex plan prefetches
    // IO = 3 (mask dump) is the IO = 0 kernel plus the dump. The real-input kernels keep the
    // twiddle table in shared memory (the block-pair code needs the registers) and prefetch into
    // the exchange buffer.
    constexpr int TMA = IO == 1 ? 0 : ((IO == 2 && CH::TMA == 1) ? 2 : CH::TMA);
    constexpr int TWK = (IO == 1 || IO == 2) && CH::TWK == 3 ? 1 : CH::TWK;
    auto kern = ols_fused<R, N, CH::E, MODE, CH::GROUPS, TMA, TWK, CH::MINB, IO>;
    using PLK = Plan<N, CH::E, CH::TWF>;
    const size_t smem = info_for<R, N>().smem + smem_extra +
                        (TWK != CH::TWK ? sizeof(cx_t<R>) * size_t(PLK::TW_PER_THREAD) * CH::T : 0);
    cudaError_t err;
    int dev = 0;
    if ((err = cudaGetDevice(&dev)) != cudaSuccess) return err;
    // residency per (device, smem) is cached: the launch path is then one kernel launch
    static thread_local int c_dev = -1, c_sms = 0, c_per_sm = 0;
    static thread_local size_t c_smem = 0;
    if (c_dev != dev || c_smem != smem) {
        if (smem > 48 * 1024) {
            err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
            if (err != cudaSuccess) return err;
        }
        int sms = 0, per_sm = 0;
        if ((err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return err;
        if ((err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, CH::THREADS, smem)) != cudaSuccess)
            return err;
        if (per_sm < 1) return cudaErrorInvalidConfiguration;
        c_dev = dev;
        c_smem = smem;
        c_sms = sms;
        c_per_sm = per_sm;
    }
    const int sms = c_sms, per_sm = c_per_sm;
    int64_t grid = (a.total + CH::GROUPS - 1) / CH::GROUPS;
    const int64_t resident = int64_t(sms) * per_sm;
    if (grid > resident) grid = resident;
    if (max_grid > 0 && grid > max_grid) grid = max_grid;
    if (grid < 1) grid = 1;
    if (grid_used) *grid_used = int(grid);
    // small launches: when the items of a CTA need R rounds of its warps, use just enough warps
    // that all R rounds are equally full (the last round of a 16 + 3 split runs latency-bound)
    OlsArgs<R> args = a;
    {
        constexpr int GPW = CH::T >= 32 ? 1 : 32 / CH::T;
        constexpr int UPC = CH::GROUPS / GPW;
        const int64_t per_cta = (a.total + grid - 1) / grid;
        const int64_t units = (per_cta + GPW - 1) / GPW;  // warp-steps of work per CTA
        const int64_t rounds = (units + UPC - 1) / UPC;
        args.units = rounds > 0 ? int((units + rounds - 1) / rounds) : UPC;
    }
    // programmatic dependent launch: the kernel's prologue overlaps the previous launch's tail
    // (griddepcontrol.wait in ols_fused orders its global accesses after it)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(CH::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args);
}

template <class R, int N, int IO>
cudaError_t launch_modes(int mode, const OlsArgs<R>& a, size_t smem_extra, int max_grid, cudaStream_t s,
                         int* grid_used) {
    // real I/O: IO = 1 (one real channel per transform) serves raw tables; IO = 2 (block pairs)
    // serves structured engines
    if constexpr (IO == 3) {  // mask dump: structured modes, complex buffers
        switch (mode) {
            case COEF_SHIFT: return launch_one<R, N, COEF_SHIFT, 3>(a, smem_extra, max_grid, s, grid_used);
            case COEF_PHASE: return launch_one<R, N, COEF_PHASE, 3>(a, smem_extra, max_grid, s, grid_used);
            case COEF_SHIFT_Q:
                if constexpr (Choice<R, N>::E % 8 == 0)
                    return launch_one<R, N, COEF_SHIFT_Q, 3>(a, smem_extra, max_grid, s, grid_used);
                else
                    return launch_one<R, N, COEF_SHIFT, 3>(a, smem_extra, max_grid, s, grid_used);
        }
        return cudaErrorInvalidValue;
    } else if constexpr (IO == 1) {
        if (mode != COEF_RAW) return cudaErrorInvalidValue;
        return launch_one<R, N, COEF_RAW, 1>(a, smem_extra, max_grid, s, grid_used);
    } else if constexpr (IO == 2) {
        switch (mode) {
            case COEF_SHIFT: return launch_one<R, N, COEF_SHIFT, 2>(a, smem_extra, max_grid, s, grid_used);
            case COEF_PHASE: return launch_one<R, N, COEF_PHASE, 2>(a, smem_extra, max_grid, s, grid_used);
            case COEF_SHIFT_Q:
                if constexpr (Choice<R, N>::E % 8 == 0)
                    return launch_one<R, N, COEF_SHIFT_Q, 2>(a, smem_extra, max_grid, s, grid_used);
                else
                    return launch_one<R, N, COEF_SHIFT, 2>(a, smem_extra, max_grid, s, grid_used);
        }
        return cudaErrorInvalidValue;
    }
    switch (mode) {
        case COEF_SHIFT: return launch_one<R, N, COEF_SHIFT, IO>(a, smem_extra, max_grid, s, grid_used);
        case COEF_PHASE: return launch_one<R, N, COEF_PHASE, IO>(a, smem_extra, max_grid, s, grid_used);
        case COEF_RAW: return launch_one<R, N, COEF_RAW, IO>(a, smem_extra, max_grid, s, grid_used);
        case COEF_SHIFT_Q:
            if constexpr (Choice<R, N>::E % 8 == 0)
                return launch_one<R, N, COEF_SHIFT_Q, IO>(a, smem_extra, max_grid, s, grid_used);
            else
                return launch_one<R, N, COEF_SHIFT, IO>(a, smem_extra, max_grid, s, grid_used);
    }
    return cudaErrorInvalidValue;
}

#define FCVBW_FOR_EACH_N(X) X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096) X(8192)

template <class R>
bool plan_info_impl(int N, LaunchInfo* out) {
    switch (N) {
#define FCVBW_CASE(n) \
    case n: *out = info_for<R, n>(); return true;
        FCVBW_FOR_EACH_N(FCVBW_CASE)
#undef FCVBW_CASE
    }
    return false;
}

template <class R, int IO>
cudaError_t launch_ols_impl(int N, int mode, const OlsArgs<R>& a, size_t smem_extra, int max_grid,
                            cudaStream_t s, int* grid_used) {
    switch (N) {
#define FCVBW_CASE(n) \
    case n: return launch_modes<R, n, IO>(mode, a, smem_extra, max_grid, s, grid_used);
        FCVBW_FOR_EACH_N(FCVBW_CASE)
#undef FCVBW_CASE
    }
    return cudaErrorInvalidValue;
}

}  // namespace fcvbw_gpu
