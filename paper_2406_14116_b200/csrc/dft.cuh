// Register-resident DFT codelets (radix-2/4 building blocks composed by the four-step rule).
//
// Replaces the per-stage butterfly loop of the reference's Radix2Fft::run
// (proj/include/fcvbw/fft.hpp:95-108) inside one thread: the R inputs live in registers, every
// array index is a compile-time constant after unrolling, and the bit-reversal of the reference
// (fft.hpp:40-45, :57) disappears into compile-time register renaming. Twiddles inside a codelet
// are literals (twiddle64.cuh); trivial ones (1, -j, -1, +j) cost nothing because the swap/negate
// folds into the FADD2 operand selectors of the consumer.
//
// Convention matches fft.hpp:16-19: forward X[k] = sum_n x[n] e^{-j 2 pi n k / R}, unnormalised;
// INV uses e^{+j...} (the 1/N of the inverse is folded into the spectral coefficients).
#pragma once

#include "cplx.cuh"
#include "twiddle64.cuh"

namespace fcvbw_gpu {

// v * W_R^m (forward kernel); the INV caller passes m -> R - m.
template <int R, int M, class C>
__device__ __forceinline__ C twiddle_const(C v) {
    constexpr int m = ((M % R) + R) % R;
    if constexpr (m == 0) {
        return v;
    } else if constexpr (4 * m == R) {
        return cmul_mj(v);  // * (-j)
    } else if constexpr (2 * m == R) {
        return cneg(v);
    } else if constexpr (4 * m == 3 * R) {
        return cneg(cmul_mj(v));  // * (+j)
    } else {
        constexpr int t = m * (64 / R);
        return cmul(v, cmake<C>(cos64(t), -sin64(t)));
    }
}

template <bool INV, class C>
__device__ __forceinline__ void bfly2(C& a0, C& a1) {
    C s = cadd(a0, a1);
    a1 = csub(a0, a1);
    a0 = s;
}

template <bool INV, class C>
__device__ __forceinline__ void bfly4(C& a0, C& a1, C& a2, C& a3) {
    C s0 = cadd(a0, a2), d0 = csub(a0, a2);
    C s1 = cadd(a1, a3), d1 = csub(a1, a3);
    a0 = cadd(s0, s1);
    a2 = csub(s0, s1);
    if constexpr (!INV) {
        a1 = cadd_mj(d0, d1);  // d0 + (-j) d1
        a3 = csub_mj(d0, d1);
    } else {
        a1 = csub_mj(d0, d1);  // d0 + (+j) d1
        a3 = cadd_mj(d0, d1);
    }
}

#ifndef FCVBW_DFT32_A
#define FCVBW_DFT32_A 4
#endif
template <int R>
struct dft_split {
    // R = A * B; the B-point sub-DFTs run first (stride A), then A-point DFTs across them.
    static constexpr int A = R == 32 ? FCVBW_DFT32_A : ((R >= 16) ? 4 : 2);
    static constexpr int B = R / A;
};

template <int R, int A, int B, bool INV, int a = 1, int kb = 1, class C>
__device__ __forceinline__ void twiddle_rows(C (&u)[A][B]) {
    if constexpr (a < A) {
        if constexpr (kb < B) {
            constexpr int m = INV ? (R - (a * kb) % R) : (a * kb);
            u[a][kb] = twiddle_const<R, m>(u[a][kb]);
            twiddle_rows<R, A, B, INV, a, kb + 1>(u);
        } else {
            twiddle_rows<R, A, B, INV, a + 1, 1>(u);
        }
    }
}

struct no_pre {
    template <class C>
    __device__ __forceinline__ C operator()(int, C x) const {
        return x;
    }
};

// In-place DFT of R values held in registers, natural order in and out. `pre(i, x)` is applied
// to input i immediately before its first use (the inter-pass twiddle of a Stockham pass), so
// the twiddles of one B-point sub-DFT are live only while that sub-DFT runs.
template <int R, bool INV, class C, class Pre = no_pre>
__device__ __forceinline__ void dft(C (&v)[R], Pre pre = Pre{}) {
    if constexpr (R == 1) {
        v[0] = pre(0, v[0]);
    } else if constexpr (R == 2) {
        v[1] = pre(1, v[1]);
        bfly2<INV>(v[0], v[1]);
    } else if constexpr (R == 4) {
#pragma unroll
        for (int i = 1; i < 4; ++i) v[i] = pre(i, v[i]);
        bfly4<INV>(v[0], v[1], v[2], v[3]);
    } else {
        constexpr int A = dft_split<R>::A;
        constexpr int B = dft_split<R>::B;
        C u[A][B];
#pragma unroll
        for (int a = 0; a < A; ++a) {
#pragma unroll
            for (int b = 0; b < B; ++b) u[a][b] = pre(a + A * b, v[a + A * b]);
            dft<B, INV>(u[a]);
        }
        // u[a][kb] *= W_R^{a kb}
        twiddle_rows<R, A, B, INV>(u);
#pragma unroll
        for (int kb = 0; kb < B; ++kb) {
            C w[A];
#pragma unroll
            for (int a = 0; a < A; ++a) w[a] = u[a][kb];
            dft<A, INV>(w);
#pragma unroll
            for (int ka = 0; ka < A; ++ka) v[kb + B * ka] = w[ka];
        }
    }
}

}  // namespace fcvbw_gpu
