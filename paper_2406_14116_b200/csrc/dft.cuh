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

struct no_pre {
    template <class C>
    __device__ __forceinline__ C operator()(int, C x) const {
        return x;
    }
};
// Real per-input scale s(i) fused into the first butterfly level (x0 s0 + x1 s1 = FMUL2 + FFMA2
// instead of two FMUL2 and an FADD2): the spectral mask feeding the inverse transform.
struct no_scale {
    static constexpr bool active = false;
    __device__ __forceinline__ float operator()(int) const { return 1.f; }
};
template <class F>
struct scale_by {
    static constexpr bool active = true;
    F f;
    __device__ __forceinline__ auto operator()(int i) const { return f(i); }
};
template <class F>
__device__ __forceinline__ scale_by<F> make_scale(F f) {
    return scale_by<F>{f};
}

template <int R, bool INV, class C, class Pre = no_pre, class Sc = no_scale>
__device__ __forceinline__ void dft(C (&v)[R], Pre pre = Pre{}, Sc sc = Sc{});

template <class C>
struct re_of;
template <>
struct re_of<float2> {
    using type = float;
};
template <>
struct re_of<double2> {
    using type = double;
};

// W8-type twiddles. W_R^m with 8 m / R = m' odd equals c (sx + j sy), c = 1/sqrt(2), sx, sy = +-1:
// v W_R^m = sx c (v + s' j v) with s' = sx sy. The kernel keeps p = v + s' j v (ONE add: the
// swap and negation fold into the FADD2 operand selectors) and carries the real factor sx c into
// the butterfly that consumes the value, where a +- (sx c) p is one FFMA2 instead of the FMUL2 of
// the scale plus an FADD2. Returns m' (1, 3, 5, 7) or 0.
__host__ __device__ constexpr int w8_index(int R, int m) {
    return (R % 8 == 0 && (8 * m) % R == 0 && (((8 * m) / R) & 1)) ? (8 * m) / R : 0;
}
// sign sx of the pending factor: m' = 1 -> c(1 - j), 3 -> c(-1 - j), 5 -> c(-1 + j), 7 -> c(1 + j)
__host__ __device__ constexpr int w8_sign(int mp) { return (mp == 1 || mp == 7) ? 1 : -1; }
// twiddle exponent of element (a, kb) of the four-step split (the INV caller conjugates)
__host__ __device__ constexpr int tw_exp(int R, int a, int kb, bool inv) {
    return inv ? (R - (a * kb) % R) % R : (a * kb) % R;
}
// pending-scale code of element (a, kb): 0 none, +-1 = sign of the pending factor c
__host__ __device__ constexpr int w8_code(int R, int a, int kb, bool inv) {
    return w8_index(R, tw_exp(R, a, kb, inv)) ? w8_sign(w8_index(R, tw_exp(R, a, kb, inv))) : 0;
}

template <int R, int M, class C>
__device__ __forceinline__ C twiddle_w8_unscaled(C v) {
    constexpr int mp = w8_index(R, M);
    static_assert(mp != 0, "not a W8-type twiddle");
    if constexpr (mp == 1 || mp == 5)
        return cadd_mj(v, v);  // v + (-j) v
    else
        return csub_mj(v, v);  // v + j v
}

// column kb of the four-step split: twiddle u[a][kb] (W8-type ones left pending), then the
// A-point DFT consuming them
template <int R, int A, int B, bool INV, int kb, int a = 1, class C>
__device__ __forceinline__ void load_col(C (&u)[A][B], C (&w)[A]) {
    if constexpr (a == 1) w[0] = u[0][kb];
    if constexpr (a < A) {
        constexpr int m = tw_exp(R, a, kb, INV);
        if constexpr (w8_code(R, a, kb, INV) != 0)
            w[a] = twiddle_w8_unscaled<R, m>(u[a][kb]);
        else
            w[a] = twiddle_const<R, m>(u[a][kb]);
        load_col<R, A, B, INV, kb, a + 1>(u, w);
    }
}

template <bool INV, int C1, class C>
__device__ __forceinline__ void dft2_pend(C (&w)[2]) {
    using Rr = typename re_of<C>::type;
    if constexpr (C1 == 0) {
        bfly2<INV>(w[0], w[1]);
    } else {
        const Rr k = Rr(C1) * Rr(cos64(8));
        const C o0 = cfma(w[1], k, w[0]);
        w[1] = cfma(w[1], -k, w[0]);
        w[0] = o0;
    }
}

template <bool INV, int C1, int C2, int C3, class C>
__device__ __forceinline__ void dft4_pend(C (&w)[4]) {
    using Rr = typename re_of<C>::type;
    const Rr cc = Rr(cos64(8));
    C s0, d0;
    if constexpr (C2 == 0) {
        s0 = cadd(w[0], w[2]);
        d0 = csub(w[0], w[2]);
    } else {
        s0 = cfma(w[2], Rr(C2) * cc, w[0]);
        d0 = cfma(w[2], -Rr(C2) * cc, w[0]);
    }
    if constexpr (C1 != 0 && C3 != 0) {
        // C1 c p1 + C3 c p3 = (C1 c) (p1 + (C3 / C1) p3)
        const C q = C1 == C3 ? cadd(w[1], w[3]) : csub(w[1], w[3]);
        const C r = C1 == C3 ? csub(w[1], w[3]) : cadd(w[1], w[3]);
        const Rr k = Rr(C1) * cc;
        w[0] = cfma(q, k, s0);
        w[2] = cfma(q, -k, s0);
        // d1 = k r; forward: d0 + (-j) d1 = d0 + k (r.y, -r.x); inverse: d0 + j d1 = d0 + k (-r.y, r.x)
        if constexpr (!INV) {
            w[1] = cfma_swap(r, k, -k, d0);
            w[3] = cfma_swap(r, -k, k, d0);
        } else {
            w[1] = cfma_swap(r, -k, k, d0);
            w[3] = cfma_swap(r, k, -k, d0);
        }
    } else {
        const C x1 = C1 != 0 ? cscale(w[1], Rr(C1) * cc) : w[1];
        const C x3 = C3 != 0 ? cscale(w[3], Rr(C3) * cc) : w[3];
        const C s1 = cadd(x1, x3), d1 = csub(x1, x3);
        w[0] = cadd(s0, s1);
        w[2] = csub(s0, s1);
        if constexpr (!INV) {
            w[1] = cadd_mj(d0, d1);
            w[3] = csub_mj(d0, d1);
        } else {
            w[1] = csub_mj(d0, d1);
            w[3] = cadd_mj(d0, d1);
        }
    }
}

template <int R, int A, int B, bool INV, int kb, class C>
__device__ __forceinline__ void dft_cols(C (&u)[A][B], C (&v)[R]) {
    if constexpr (kb < B) {
        C w[A];
        load_col<R, A, B, INV, kb>(u, w);
        if constexpr (A == 2) {
            dft2_pend<INV, w8_code(R, 1, kb, INV)>(w);
        } else if constexpr (A == 4) {
            dft4_pend<INV, w8_code(R, 1, kb, INV), w8_code(R, 2, kb, INV), w8_code(R, 3, kb, INV)>(w);
        } else {
            using Rr = typename re_of<C>::type;
#pragma unroll
            for (int a = 1; a < A; ++a)
                if (w8_code(R, a, kb, INV) != 0) w[a] = cscale(w[a], Rr(w8_code(R, a, kb, INV)) * Rr(cos64(8)));
            dft<A, INV>(w);
        }
#pragma unroll
        for (int ka = 0; ka < A; ++ka) v[kb + B * ka] = w[ka];
        dft_cols<R, A, B, INV, kb + 1>(u, v);
    }
}

// In-place DFT of R values held in registers, natural order in and out. `pre(i, x)` is applied
// to input i immediately before its first use (the inter-pass twiddle of a Stockham pass), so
// the twiddles of one B-point sub-DFT are live only while that sub-DFT runs; `sc(i)` (when
// active) is a real factor on input i, applied inside the first butterfly level.
template <int R, bool INV, class C, class Pre, class Sc>
__device__ __forceinline__ void dft(C (&v)[R], Pre pre, Sc sc) {
    if constexpr (R == 1) {
        v[0] = pre(0, v[0]);
        if constexpr (Sc::active) v[0] = cscale(v[0], sc(0));
    } else if constexpr (R == 2) {
        v[1] = pre(1, v[1]);
        if constexpr (Sc::active) {
            const C t = cscale(v[0], sc(0));
            const auto g1 = sc(1);
            v[0] = cfma(v[1], g1, t);
            v[1] = cfma(v[1], -g1, t);
        } else {
            bfly2<INV>(v[0], v[1]);
        }
    } else if constexpr (R == 4) {
#pragma unroll
        for (int i = 1; i < 4; ++i) v[i] = pre(i, v[i]);
        if constexpr (Sc::active) {
            const C t0 = cscale(v[0], sc(0)), t1 = cscale(v[1], sc(1));
            const auto g2 = sc(2), g3 = sc(3);
            const C s0 = cfma(v[2], g2, t0), d0 = cfma(v[2], -g2, t0);
            const C s1 = cfma(v[3], g3, t1), d1 = cfma(v[3], -g3, t1);
            v[0] = cadd(s0, s1);
            v[2] = csub(s0, s1);
            if constexpr (!INV) {
                v[1] = cadd_mj(d0, d1);
                v[3] = csub_mj(d0, d1);
            } else {
                v[1] = csub_mj(d0, d1);
                v[3] = cadd_mj(d0, d1);
            }
        } else {
            bfly4<INV>(v[0], v[1], v[2], v[3]);
        }
    } else {
        constexpr int A = dft_split<R>::A;
        constexpr int B = dft_split<R>::B;
        C u[A][B];
#pragma unroll
        for (int a = 0; a < A; ++a) {
#pragma unroll
            for (int b = 0; b < B; ++b) u[a][b] = pre(a + A * b, v[a + A * b]);
            if constexpr (Sc::active)
                dft<B, INV>(u[a], no_pre{}, make_scale([&](int b) { return sc(a + A * b); }));
            else
                dft<B, INV>(u[a]);
        }
        // u[a][kb] *= W_R^{a kb}, then the A-point DFTs across the columns
        dft_cols<R, A, B, INV, 0>(u, v);
    }
}

}  // namespace fcvbw_gpu
