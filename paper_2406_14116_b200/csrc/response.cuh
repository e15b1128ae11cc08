// Device evaluation of PTVIR responses in the reference's exact operation order (shared by
// design.cu and analyze.cu): std::complex<double> products without FMA contraction, sums in
// index order. With host-libm tables (grid.h) the results are bit-identical to the reference's
// base_response_idft (ptvir.hpp:100-115) and response_from_row (ptvir.hpp:355-361).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace fcvbw_resp {

// std::complex<double> arithmetic in the reference's order, without contraction.
__device__ __forceinline__ double2 cmul_x(double2 a, double2 b) {
    return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                        __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

// base_response_idft (ptvir.hpp:100-115) for T tables: base[t][q] = Re(sum_k table[t][k] root(qk)) / N,
// k ascending. bad[t] set when the imaginary residue exceeds 1e-12 N.
static __global__ void base_rows_kernel(int N, int T, const double2* __restrict__ tables, const double2* __restrict__ roots,
                                 double* base, int* bad) {
    const int t = blockIdx.y;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T || q >= N) return;
    const double2* tab = tables + size_t(t) * N;
    double re = 0.0, im = 0.0;
    for (int k = 0; k < N; ++k) {
        const double2 p = cmul_x(tab[k], roots[int((int64_t(q) * k) & (N - 1))]);
        re = __dadd_rn(re, p.x);
        im = __dadd_rn(im, p.y);
    }
    if (fabs(im) > 1e-12 * N) atomicExch(bad, 1);
    base[size_t(t) * N + q] = __ddiv_rn(re, double(N));
}

// response_from_row (ptvir.hpp:355-361) on the PTVIR row n of a base row: d_n(q) = base((q + s) mod N).
__device__ __forceinline__ double2 row_response(const double* __restrict__ base, int N, int shift,
                                                const double2* __restrict__ ph, double2 pre) {
    double re = 0.0, im = 0.0;
    for (int q = 0; q < N; ++q) {
        const double d = base[(q + shift) & (N - 1)];
        const double2 f = ph[q];
        re = __dadd_rn(re, __dmul_rn(d, f.x));
        im = __dadd_rn(im, __dmul_rn(d, f.y));
    }
    return cmul_x(pre, make_double2(re, im));
}

// |z| exactly as the host's libm computes it: glibc 2.35+ __hypot (sysdeps/ieee754/dbl-64/e_hypot.c,
// the non-FMA kernel x86-64 builds use: one sqrt plus a correction step), restated with explicit
// round-to-nearest operations. std::abs(std::complex<double>) calls it, so every |H| / |E| the
// reference compares or prints goes through this algorithm; CUDA's own hypot differs by up to an
// ulp. Pinned against the host libm on random inputs by tests/test_host_logic.py
// (test_glibc_hypot_restatement) through the same formula in Python.
__device__ __forceinline__ double glibc_hypot_kernel(double ax, double ay) {
    double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
    double t1, t2;
    if (h <= __dmul_rn(2.0, ay)) {
        const double delta = __dsub_rn(h, ay);
        t1 = __dmul_rn(ax, __dsub_rn(__dmul_rn(2.0, delta), ax));
        t2 = __dmul_rn(__dsub_rn(delta, __dmul_rn(2.0, __dsub_rn(ax, ay))), delta);
    } else {
        const double delta = __dsub_rn(h, ax);
        t1 = __dmul_rn(__dmul_rn(2.0, delta), __dsub_rn(ax, __dmul_rn(2.0, ay)));
        t2 = __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(4.0, delta), ay), ay), __dmul_rn(delta, delta));
    }
    return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), __dmul_rn(2.0, h)));
}

__device__ __forceinline__ double glibc_hypot(double x, double y) {
    if (isinf(x) || isinf(y)) return INFINITY;
    if (isnan(x) || isnan(y)) return x + y;
    x = fabs(x);
    y = fabs(y);
    const double ax = x < y ? y : x, ay = x < y ? x : y;
    constexpr double kScale = 0x1p-600, kLarge = 0x1p+511, kTiny = 0x1p-511, kEps = 0x1p-54;
    if (ax > kLarge) {
        if (ay <= __dmul_rn(ax, kEps)) return __dadd_rn(ax, ay);
        return __ddiv_rn(glibc_hypot_kernel(__dmul_rn(ax, kScale), __dmul_rn(ay, kScale)), kScale);
    }
    if (ay < kTiny) {
        if (ax >= __ddiv_rn(ay, kEps)) return __dadd_rn(ax, ay);
        return __dmul_rn(glibc_hypot_kernel(__ddiv_rn(ax, kScale), __ddiv_rn(ay, kScale)), kScale);
    }
    if (ay <= __dmul_rn(ax, kEps)) return __dadd_rn(ax, ay);
    return glibc_hypot_kernel(ax, ay);
}

}  // namespace fcvbw_resp
