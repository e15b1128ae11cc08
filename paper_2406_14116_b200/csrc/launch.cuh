// Plan selection and type-erased launchers for the fused OLS kernel (one translation unit per
// sample type instantiates every N, see kernels_f32.cu / kernels_f64.cu).
#pragma once

#include <cuda_runtime.h>

#include "ols_kernel.cuh"

namespace fcvbw_gpu {

// Per-(sample type, N) plan, every choice measured (profiles/r01_sweep.md; round-2 changes in
// profiles/r02_sweep.md):
//   E       elements (complex registers) per thread: pass 0 is an E-point register DFT, the
//           remaining radices are <= E. fp32 keeps 32 from N = 512 up so that N = 1024 is exactly
//           two 32-point passes with one warp per block; the 64-element plan {64, 64} wins at
//           fp32 N = 4096; fp64 uses 32 at N = 512 / 1024 / 8192 and 16 elsewhere.
//   BIG     multi-warp transforms (T = 64 / 128 threads per block): several groups per CTA share
//           one twiddle table in shared memory (wins over one group per CTA).
//   GROUPS  blocks in flight per CTA. Single-warp-or-smaller transforms run ONE CTA of 128 x MINB
//           threads per SM (one 512-thread CTA keeps 15.8 of 16 warp slots busy at N = 1024 where
//           four 128-thread CTAs averaged 12: c3 0.707 -> 0.770); fp32 N = 64 runs 128-thread CTAs
//           (+4 %), the MINB = 1 plans one 256-thread CTA (+5 %).
//   MINB    register budget as resident 128-thread CTAs per SM (123 registers at N = 1024 fp32).
//   TMA     2 = the next segment is bulk-copied into the idle exchange buffer (N = 1024 / 8192
//           fp32, fp64 N = 4096, the fp32 64-element plan); 0 = direct coalesced loads.
//   TWK     twiddles: 1 = full per-thread table in shared memory (<= 16 KB, and the 64-element
//           plan: +3.5 %), 2 = factored table in shared memory (BIG 32-element plans: +0.5-2.5 %),
//           0 = factored table through L1.
template <class R, int N>
struct Choice {
    static constexpr bool F32 = sizeof(R) == 4;
#ifndef FCVBW_E_F64_512
#define FCVBW_E_F64_512 32
#endif
#ifndef FCVBW_E64_F32
#define FCVBW_E64_F32 ((1 << 11) | (1 << 12))
#endif
    static constexpr bool E64F = (FCVBW_E64_F32 >> ilog2(N)) & 1;
    static constexpr int E0 = F32 ? (N <= 16 ? N : (N == 64 ? 8 : (N <= 256 ? 16 : (E64F ? 64 : 32))))
                                  : (N <= 16 ? N : (N == 64 ? 8 : (N < 512 ? 16 : (N == 512 ? FCVBW_E_F64_512 : ((N == 1024 || N == 8192) ? 32 : 16)))));
    static constexpr int E = E0;
    static constexpr int T = N / E;
    static constexpr size_t EXB = sizeof(cx_t<R>) * size_t(padded<R, E>(N));
    static constexpr size_t TWB_FULL = sizeof(cx_t<R>) * size_t(Plan<N, E, true>::TW_PER_THREAD) * T;
#ifndef FCVBW_TWC_F32
#define FCVBW_TWC_F32 0
#endif
#ifndef FCVBW_TWC_F64
#define FCVBW_TWC_F64 0
#endif
    static constexpr int LOGN = ilog2(N);
    static constexpr bool bit(long long mask) { return (mask >> LOGN) & 1; }
    // TWC: full tangent-form table in the compact (pass, i, k) layout, shared by the CTA's groups
    static constexpr bool TWC = bit(F32 ? FCVBW_TWC_F32 : FCVBW_TWC_F64) && Plan<N, E, true>::P >= 3;
    static constexpr size_t TWB_C = sizeof(cx_t<R>) * size_t(Plan<N, E, true>::TW_COMPACT);
    static constexpr size_t TWB_USE = TWC ? TWB_C : TWB_FULL;
    static constexpr bool BIG = T >= 64 && T <= 128 && EXB + TWB_USE <= 200 * 1024;
    // CTA size of the BIG plans: 256 threads for the 64-element plan (two warps per SMSP, so that its
    // 243 registers fit), 512 for the fp32 32-element plan (8 groups, 16 warps: +3 % over 384)
    static constexpr int BIG_THREADS = E0 >= 64 ? 256 : (F32 ? 512 : 384);
    static constexpr int GROUPS_BIG0 = BIG_THREADS / T > 1 ? BIG_THREADS / T : 1;
    static constexpr int GROUPS_FIT = BIG ? int((200 * 1024 - TWB_USE) / EXB) : 1;
    // T >= 128 with the compact table: up to 512 threads per CTA sharing it
    static constexpr int GROUPS_WIDE0 = int((220 * 1024 - TWB_C) / EXB) < 512 / T ? int((220 * 1024 - TWB_C) / EXB)
                                                                                    : 512 / T;
    static constexpr int GROUPS_WIDE = GROUPS_WIDE0 >= 1 ? GROUPS_WIDE0 : 1;
// Per-N plan switches as bit masks over log2 N (experiments override them with -D; the defaults
// are the measured choices, profiles/r02_sweep.md):
//   TWREG: inter-pass twiddle table held in registers (TWK = 3, two-pass plans only)
//   TMA1:  dedicated staging buffer per group, next segment prefetched a whole block ahead
//   MINB3: register budget of three 128-thread CTAs per SM (168 registers at <= 128 threads)
#ifndef FCVBW_TWREG_F32
#define FCVBW_TWREG_F32 (1 << 10)
#endif
#ifndef FCVBW_TWREG_F64
#define FCVBW_TWREG_F64 0
#endif
#ifndef FCVBW_TMA1_F32
#define FCVBW_TMA1_F32 (1 << 10)
#endif
#ifndef FCVBW_TMA1_F64
#define FCVBW_TMA1_F64 0
#endif
#ifndef FCVBW_MINB3_F32
#define FCVBW_MINB3_F32 (1 << 10)
#endif
#ifndef FCVBW_MINB3_F64
#define FCVBW_MINB3_F64 0
#endif
    static constexpr int MINB0 = F32 ? (E0 >= 64 && N != 4096 ? 2 : ((N <= 1024 || N == 8192) ? 4 : 3))
                                     : (E0 == 32 ? 1 : ((N <= 256 || N == 1024 || N == 4096) ? 4 : 3));
    static constexpr int MINB = bit(F32 ? FCVBW_MINB3_F32 : FCVBW_MINB3_F64) ? 3 : MINB0;
    static constexpr int CTA_T = (F32 && N == 64) ? 128 : (MINB == 1 ? 256 : 128 * MINB);
    static constexpr int GROUPS = BIG ? (GROUPS_BIG0 < GROUPS_FIT ? GROUPS_BIG0 : GROUPS_FIT)
                                      : (T >= 128 ? (TWC ? GROUPS_WIDE : 1) : CTA_T / T);
    static constexpr int THREADS = GROUPS * T;
    // (fp32 N = 2048, the 32-element BIG plan: direct loads measured +3.7 %; fp32 N = 8192 and fp64
    // N = 4096: the exchange-buffer prefetch lets two CTAs fit per SM: +13 % / +19 %)
    static constexpr bool TMA1 = !BIG && T <= 32 && bit(F32 ? FCVBW_TMA1_F32 : FCVBW_TMA1_F64) &&
                                 size_t(GROUPS) * (EXB + sizeof(cx_t<R>) * N) <= 220 * 1024;
#ifndef FCVBW_TMA2_F32
#define FCVBW_TMA2_F32 ((1 << 11) | (1 << 13))
#endif
#ifndef FCVBW_TMA2_F64
#define FCVBW_TMA2_F64 ((1 << 10) | (1 << 12))
#endif
    static constexpr int TMA = BIG ? ((F32 && E0 == 32) ? 0 : 2)
                                   : (TMA1 ? 1 : (bit(F32 ? FCVBW_TMA2_F32 : FCVBW_TMA2_F64) ? 2 : 0));
    static constexpr bool TWREG = bit(F32 ? FCVBW_TWREG_F32 : FCVBW_TWREG_F64) && Plan<N, E, true>::P == 2 &&
                                  Plan<N, E, true>::TW_PER_THREAD <= 32 && T <= 32;
    static constexpr int TWK = BIG ? (TWC ? 4 : (E0 >= 64 ? 1 : 2))
                                   : (TWB_FULL <= 16 * 1024 ? (TWREG ? 3 : 1) : (TWC ? 4 : 0));
    static constexpr bool TWF = TWK == 1 || TWK == 3 || TWK == 4;
};

struct LaunchInfo {
    int N = 0, E = 0, T = 0, groups = 0, threads = 0, passes = 0, tw_per_thread = 0, tw_compact = 0;
    int radix[8] = {0};
    size_t smem = 0;  // dynamic shared memory excluding the profile table
    bool tma = false;
    bool twf = false;  // full (unfactored) twiddle table
    bool twt = false;  // full table stored in tangent form {t, wr}
    bool twp = false;  // factored fp32 table in the paired layout (tw_paired)
    bool twc = false;  // full table in the compact (pass, i, k) layout (TWK = 4)
    bool mask_table = false;  // structured modes keep the b-independent mask table behind V (MaskGen)
    bool mask_table4 = false;  // ... transposed in four shifted copies (vector loads)
};

template <class R, int N>
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
    li.smem = sizeof(cx_t<R>) * size_t(CH::GROUPS) * padded<R, CH::E>(N) + sizeof(uint64_t) * CH::GROUPS +
              (CH::TMA == 1 ? sizeof(cx_t<R>) * size_t(CH::GROUPS) * N : 0) +
              ((CH::TWK == 1 || CH::TWK == 2) ? sizeof(cx_t<R>) * size_t(PL::TW_PER_THREAD) * CH::T : 0) +
              (CH::TWK == 4 ? sizeof(cx_t<R>) * size_t(PL::TW_COMPACT) : 0);
    li.twc = CH::TWK == 4;
    li.mask_table = mask_table<R, N>();
    li.mask_table4 = mask_table4<R, N>();
    li.tw_compact = PL::TW_COMPACT;
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
// io = 2: real buffers, block pairs (see OlsArgs::xr / nblk_real); io = 3: io = 0 plus the mask dump
template <class R, int IO>
cudaError_t launch_ols_io(int N, int mode, const OlsArgs<R>& args, size_t smem_extra, int max_grid,
                          cudaStream_t stream, int* grid_used);
template <class R>
inline cudaError_t launch_ols(int N, int mode, int io, const OlsArgs<R>& args, size_t smem_extra, int max_grid,
                              cudaStream_t stream, int* grid_used) {
    return io == 3   ? launch_ols_io<R, 3>(N, mode, args, smem_extra, max_grid, stream, grid_used)
           : io == 2 ? launch_ols_io<R, 2>(N, mode, args, smem_extra, max_grid, stream, grid_used)
           : io == 1 ? launch_ols_io<R, 1>(N, mode, args, smem_extra, max_grid, stream, grid_used)
                     : launch_ols_io<R, 0>(N, mode, args, smem_extra, max_grid, stream, grid_used);
}
template <class R>
cudaError_t launch_coeff_dump(int N, const int* b_dev, int n_b, int half_dn, const double* v_dev,
                              const double2* phase_dev, int8_t* region, int16_t* vidx, double2* H,
                              cudaStream_t stream);

}  // namespace fcvbw_gpu
