// Plan selection and type-erased launchers for the fused OLS kernel (one translation unit per
// sample type instantiates every N, see kernels_f32.cu / kernels_f64.cu).
#pragma once

#include <cuda_runtime.h>

#include "ols_kernel.cuh"

namespace fcvbw_gpu {

// Elements per thread E for each N: register-resident pass 0 of E points, remaining radices <= E.
// fp32 keeps 32 complex (64 registers) per thread from N = 512 up so that N = 1024 is exactly two
// 32-point passes with one warp per block; fp64 uses 16 (64 registers).
#ifndef FCVBW_E32_MAX
#define FCVBW_E32_MAX 32  // elements per thread cap for fp32 plans (experiment knob)
#endif
#ifdef FCVBW_E64_BIG  // experiment knob: elements per thread of every fp64 plan with N >= 512
#define FCVBW_E64_FOR(n) FCVBW_E64_BIG
#else  // measured (profiles/r01_sweep.md): 32 elements (two passes) win at 512 / 1024 / 8192
#define FCVBW_E64_FOR(n) (((n) == 512 || (n) == 1024 || (n) == 8192) ? 32 : 16)
#endif
#ifdef FCVBW_E32_BIG  // experiment knob: elements per thread of fp32 plans with N >= 2048
#define FCVBW_E32_FOR(n) ((n) >= 2048 ? FCVBW_E32_BIG : 32)
#else  // measured (profiles/r01_sweep.md): 64 elements (two 64-point passes) win at N = 4096 only
#define FCVBW_E32_FOR(n) ((n) == 4096 ? 64 : 32)
#endif
template <class R, int N>
struct Choice {
    static constexpr int E0 = sizeof(R) == 4
                                  ? (N <= 16 ? N : (N == 64 ? 8 : (N <= 256 ? 16 : FCVBW_E32_FOR(N))))
                                  : (N <= 16 ? N : (N == 64 ? 8 : (N < 512 ? 16 : FCVBW_E64_FOR(N))));
    static constexpr int E = (sizeof(R) == 4 && E0 > FCVBW_E32_MAX && E0 <= 32) ? FCVBW_E32_MAX : E0;
    static constexpr int T = N / E;
    // Multi-warp transforms (T >= 64): the full twiddle table lives in shared memory once per CTA
    // and several groups share it (12 warps per CTA, one CTA per SM) when it fits.
    static constexpr size_t EXB = sizeof(cx_t<R>) * size_t(padded<R, E>(N));
    static constexpr size_t TWB_FULL = sizeof(cx_t<R>) * size_t(Plan<N, E, true>::TW_PER_THREAD) * T;
#ifdef FCVBW_NO_BIG
    static constexpr bool BIG = false;
#else
    // measured (profiles/r01_sweep.md): wins for T = 64 / 128 (3-6 groups share the table); the
    // single-group T = 256 plans keep the factored table and the TMA staging buffer instead
    static constexpr bool BIG = T >= 64 && T <= 128 && EXB + TWB_FULL <= 200 * 1024;
#endif
    // 384 threads per CTA, except the 64-element plans: 256 threads (two warps per SMSP) so that
    // ptxas may give them the 243 registers they need without spilling
#ifdef FCVBW_BIG_THREADS
    static constexpr int BIG_THREADS = FCVBW_BIG_THREADS;
#else
#ifndef FCVBW_BIG32_THREADS
#define FCVBW_BIG32_THREADS 512  // CTA size of the fp32 32-element BIG plan (N = 2048): 8 groups, 16 warps (vs 384 threads: +3 %)
#endif
    static constexpr int BIG_THREADS = E0 >= 64 ? 256 : (sizeof(R) == 4 ? FCVBW_BIG32_THREADS : 384);
#endif
    static constexpr int GROUPS_BIG0 = BIG_THREADS / T > 1 ? BIG_THREADS / T : 1;
    static constexpr int GROUPS_FIT = BIG ? int((200 * 1024 - TWB_FULL) / EXB) : 1;
#ifdef FCVBW_MB
    static constexpr int MINB = FCVBW_MB;
#else
    static constexpr int MINB = sizeof(R) == 4 ? ((N <= 1024 || N == 8192) ? 4 : 3)
                                               : (E0 == 32 ? 1 : ((N <= 256 || N == 1024 || N == 4096) ? 4 : 3));
#endif
    // Single-warp-or-smaller transforms: ONE CTA per SM holds all 128 * MINB threads (MINB groups
    // of warps that used to be MINB separate 128-thread CTAs). Measured at N = 1024 fp32 (c3): four
    // 128-thread CTAs per SM averaged only 12 of their 16 warps resident (ncu sm__warps_active),
    // one 512-thread CTA keeps 15.8 resident and shares one twiddle table: 0.707 -> 0.770
    // (profiles/r01_sweep.md, "One CTA per SM"). Multi-warp groups (T >= 128) keep one group per
    // CTA (measured 2 % slower as one CTA of two groups).
#ifndef FCVBW_CTA_THREADS
#define FCVBW_CTA_THREADS 0  // experiment knob: threads per CTA of the small plans (0: 128 * MINB)
#endif
    // (fp32 N = 64, four 8-thread groups per warp, measured 4 % faster with 128-thread CTAs; the
    // MINB = 1 plan fp64 N = 512 runs one 256-thread CTA instead of two 128-thread ones: +5 %)
    static constexpr int CTA_T = FCVBW_CTA_THREADS > 0 ? FCVBW_CTA_THREADS
                                                       : ((sizeof(R) == 4 && N == 64) ? 128
                                                          : (MINB == 1 ? 256 : 128 * MINB));
    static constexpr int GROUPS = BIG ? (GROUPS_BIG0 < GROUPS_FIT ? GROUPS_BIG0 : GROUPS_FIT)
                                      : (T >= 128 ? 1 : CTA_T / T);
    static constexpr int THREADS = GROUPS * T;
    // TMA bulk prefetch of the next segment, and the register budget (resident 128-thread CTAs
    // requested from ptxas), chosen per plan from the measured sweeps (profiles/r01_sweep.md):
    // direct coalesced loads with more resident warps win for the small transforms (several groups
    // per warp), the exchange-buffer prefetch wins at N = 1024 fp32, and the largest transforms,
    // whose one-CTA-per-SM residency cannot hide DRAM latency, need the dedicated staging buffer.
#if defined(FCVBW_NO_TMA)
    static constexpr int TMA = 0;

#elif defined(FCVBW_TMA_MODE)
    static constexpr int TMA = (N >= 64 && size_t(GROUPS) * N * sizeof(cx_t<R>) <= 64 * 1024) ? FCVBW_TMA_MODE : 0;
#else
    // mode 2 (prefetch into the idle exchange buffer, no extra shared memory) for the one-warp-per-
    // block N = 1024 fp32 plan; mode 1 (dedicated staging buffer) for the largest transforms
#ifndef FCVBW_BIG_TMA
#define FCVBW_BIG_TMA 2  // exchange-buffer prefetch (measured: +0-6 %)
#endif
    // (fp32 N = 2048, the 32-element BIG plan: direct loads measured +3.7 %; fp32 N = 8192 and
    // fp64 N = 4096: the exchange-buffer prefetch frees the staging buffer so that, with the
    // 4-CTA register budget, two CTAs fit per SM: +13 % / +19 %)
#ifndef FCVBW_TMA_1024
#define FCVBW_TMA_1024 2  // fp32 N = 1024 complex: 2 = staging in the exchange buffer; 3 = L2-only prefetch (measured equal)
#endif
    static constexpr int TMA = BIG ? ((sizeof(R) == 4 && E0 == 32) ? 0 : FCVBW_BIG_TMA)
                               : (sizeof(R) == 4 && N == 1024) ? FCVBW_TMA_1024
                               : ((sizeof(R) == 4 ? (N == 1024 || N == 8192) : N == 4096) ? 2
                               : (((sizeof(R) == 4 ? N > 8192 : N == 4096) &&
                                   size_t(GROUPS) * N * sizeof(cx_t<R>) <= 64 * 1024) ? 1 : 0));
#endif
    // full twiddle table in shared memory when small; otherwise the factored table from L1
#ifndef FCVBW_BIG_TWK
#define FCVBW_BIG_TWK 2  // factored table staged in shared memory (measured: +0.5-2.5 % over the full table)
#endif
#ifdef FCVBW_NO_TWF
    static constexpr int TWK = 0;
#else
    // twiddle table: 1 = full table in shared memory, 2 = factored table in shared memory,
    // 0 = factored table read through L1
    // (the 64-element plan measured +3.5 % with the full table: profiles/r01_sweep.md)
#ifndef FCVBW_E64_TWK
#define FCVBW_E64_TWK 1
#endif
    static constexpr int TWK = BIG ? (E0 >= 64 ? FCVBW_E64_TWK : FCVBW_BIG_TWK) : (TWB_FULL <= 16 * 1024 ? 1 : 0);
#endif
    static constexpr bool TWF = TWK == 1;
};

struct LaunchInfo {
    int N = 0, E = 0, T = 0, groups = 0, threads = 0, passes = 0, tw_per_thread = 0;
    int radix[8] = {0};
    size_t smem = 0;  // dynamic shared memory excluding the profile table
    bool tma = false;
    bool twf = false;  // full (unfactored) twiddle table
    bool twt = false;  // full table stored in tangent form {t, wr}
    bool twp = false;  // factored fp32 table in the paired layout (tw_paired)
};

template <class R, int N, int TMA_USED = Choice<R, N>::TMA>
LaunchInfo info_for() {
    using CH = Choice<R, N>;
    using PL = Plan<N, CH::E, CH::TWF>;
    LaunchInfo li;
    li.N = N;
    li.E = CH::E;
    li.T = CH::T;
    li.groups = CH::GROUPS;
    li.threads = CH::THREADS;
    li.passes = PL::P;
    li.tw_per_thread = PL::TW_PER_THREAD;
    for (int p = 0; p < PL::P && p < 8; ++p) li.radix[p] = PL::radix(p);
    li.smem = sizeof(cx_t<R>) * size_t(CH::GROUPS) * padded<R, CH::E>(N) +
              (TMA_USED == 1 ? sizeof(cx_t<R>) * size_t(CH::GROUPS) * N : 0) +
              (TMA_USED ? sizeof(uint64_t) * CH::GROUPS : 0) +
              (CH::TWK ? sizeof(cx_t<R>) * size_t(PL::TW_PER_THREAD) * CH::T : 0);
    li.tma = CH::TMA != 0;
    li.twf = CH::TWF;
    li.twt = tw_tangent<R, N>(CH::TWF);
    li.twp = tw_paired<R, N, CH::E, CH::TWF>();
    return li;
}

// Implemented in kernels_f32.cu / kernels_f64.cu.
template <class R>
bool plan_info(int N, LaunchInfo* out);
// io = 0: complex interleaved buffers; io = 1: real buffers, one real channel per transform;
// io = 2: real buffers, block pairs (see OlsArgs::xr / nblk_real)
template <class R, int IO>
cudaError_t launch_ols_io(int N, int mode, const OlsArgs<R>& args, size_t smem_extra, int max_grid,
                          cudaStream_t stream, int* grid_used);
template <class R>
inline cudaError_t launch_ols(int N, int mode, int io, const OlsArgs<R>& args, size_t smem_extra, int max_grid,
                              cudaStream_t stream, int* grid_used) {
    return io == 2   ? launch_ols_io<R, 2>(N, mode, args, smem_extra, max_grid, stream, grid_used)
           : io == 1 ? launch_ols_io<R, 1>(N, mode, args, smem_extra, max_grid, stream, grid_used)
                     : launch_ols_io<R, 0>(N, mode, args, smem_extra, max_grid, stream, grid_used);
}
template <class R>
cudaError_t launch_coeff_dump(int N, const int* b_dev, int n_b, int half_dn, const double* v_dev,
                              const double2* phase_dev, int8_t* region, int16_t* vidx, double2* H,
                              cudaStream_t stream);

}  // namespace fcvbw_gpu
