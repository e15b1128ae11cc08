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

// Codelet twiddles with a pending real factor. A non-trivial W = W_R^m = wr + j wi is split as
//   |wr| >= |wi|:  W = wr (1 + j t),  t = wi / wr      (kind 1: pending real factor wr)
//   |wr| <  |wi|:  W = j wi (1 - j u), u = wr / wi     (kind 2: pending factor j wi)
// The element keeps p = v (1 + j t) (or v (1 - j u)): ONE FFMA2 with the component swap in the
// operand selector, or one FADD2 for the W8-type angles (t = +-1, p = v +- j v). The pending
// factor is applied inside the butterfly that consumes the element (a +- f p, a +- j f p: one
// FFMA2 each), saving the FMUL2 of a full complex multiply. Trivial twiddles (1, -j, -1, +j) stay
// free (twiddle_const).
__host__ __device__ constexpr int w8_index(int R, int m) {
    return (R % 8 == 0 && (8 * m) % R == 0 && (((8 * m) / R) & 1)) ? (8 * m) / R : 0;
}
// twiddle exponent of element (a, kb) of the four-step split (the INV caller conjugates)
__host__ __device__ constexpr int tw_exp(int R, int a, int kb, bool inv) {
    return inv ? (R - (a * kb) % R) % R : (a * kb) % R;
}
__host__ __device__ constexpr double tw_re(int R, int m) { return cos64(m * (64 / R)); }
__host__ __device__ constexpr double tw_im(int R, int m) { return -sin64(m * (64 / R)); }
__host__ __device__ constexpr double cabs_(double x) { return x < 0 ? -x : x; }
// 0: trivial (or m = 0), 1: pending real factor, 2: pending factor j * f
__host__ __device__ constexpr int pend_kind(int R, int m) {
    return (4 * m) % R == 0 ? 0 : ((w8_index(R, m) != 0 || cabs_(tw_re(R, m)) >= cabs_(tw_im(R, m))) ? 1 : 2);
}
__host__ __device__ constexpr double pend_fac(int R, int m) {
    return pend_kind(R, m) == 1 ? tw_re(R, m) : (pend_kind(R, m) == 2 ? tw_im(R, m) : 1.0);
}
// t (kind 1) or u (kind 2)
__host__ __device__ constexpr double pend_arg(int R, int m) {
    return pend_kind(R, m) == 1 ? tw_im(R, m) / tw_re(R, m) : (pend_kind(R, m) == 2 ? tw_re(R, m) / tw_im(R, m) : 0.0);
}

template <int R, int M, class C>
__device__ __forceinline__ C twiddle_pending(C v) {
    using Rr = typename re_of<C>::type;
    constexpr int mp = w8_index(R, M);
    if constexpr (pend_kind(R, M) == 0) {
        return twiddle_const<R, M>(v);
    } else if constexpr (mp != 0) {
        // W8-type: t = +-1
        if constexpr (pend_arg(R, M) < 0)
            return cadd_mj(v, v);  // v (1 - j)
        else
            return csub_mj(v, v);  // v (1 + j)
    } else if constexpr (pend_kind(R, M) == 1) {
        constexpr double t = pend_arg(R, M);  // v (1 + j t) = (v.x - t v.y, v.y + t v.x)
        return cfma_swap(v, Rr(-t), Rr(t), v);
    } else {
        constexpr double u = pend_arg(R, M);  // v (1 - j u) = (v.x + u v.y, v.y - u v.x)
        return cfma_swap(v, Rr(u), Rr(-u), v);
    }
}

// b + s f p, s = +-1, for a pending element p of kind K with factor f
template <int K, int S, class C, class Rr>
__device__ __forceinline__ C pend_fma(C p, Rr f, C b) {
    if constexpr (K == 0)
        return S > 0 ? cadd(b, p) : csub(b, p);
    else if constexpr (K == 1)
        return cfma(p, Rr(S) * f, b);
    else  // b + s j f p = (b.x - s f p.y, b.y + s f p.x)
        return cfma_swap(p, -Rr(S) * f, Rr(S) * f, b);
}
// f p materialized
template <int K, class C, class Rr>
__device__ __forceinline__ C pend_apply(C p, Rr f) {
    if constexpr (K == 0)
        return p;
    else if constexpr (K == 1)
        return cscale(p, f);
    else
        return cscale_swap(p, -f, f);
}

template <int R, int A, int B, bool INV, int kb, int a = 1, class C>
__device__ __forceinline__ void load_col(C (&u)[A][B], C (&w)[A]) {
    if constexpr (a == 1) w[0] = u[0][kb];
    if constexpr (a < A) {
        w[a] = twiddle_pending<R, tw_exp(R, a, kb, INV)>(u[a][kb]);
        load_col<R, A, B, INV, kb, a + 1>(u, w);
    }
}

template <int R, int kb, bool INV, class C>
__device__ __forceinline__ void dft2_pend(C (&w)[2]) {
    using Rr = typename re_of<C>::type;
    constexpr int m1 = tw_exp(R, 1, kb, INV);
    constexpr int K1 = pend_kind(R, m1);
    const Rr f1 = Rr(pend_fac(R, m1));
    const C o0 = pend_fma<K1, 1>(w[1], f1, w[0]);
    w[1] = pend_fma<K1, -1>(w[1], f1, w[0]);
    w[0] = o0;
}

template <int R, int kb, bool INV, class C>
__device__ __forceinline__ void dft4_pend(C (&w)[4]) {
    using Rr = typename re_of<C>::type;
    constexpr int m1 = tw_exp(R, 1, kb, INV), m2 = tw_exp(R, 2, kb, INV), m3 = tw_exp(R, 3, kb, INV);
    constexpr int K1 = pend_kind(R, m1), K2 = pend_kind(R, m2), K3 = pend_kind(R, m3);
    constexpr double F1 = pend_fac(R, m1), F3 = pend_fac(R, m3);
    const C s0 = pend_fma<K2, 1>(w[2], Rr(pend_fac(R, m2)), w[0]);
    const C d0 = pend_fma<K2, -1>(w[2], Rr(pend_fac(R, m2)), w[0]);
    if constexpr (K1 != 0 && K1 == K3 && (F1 == F3 || F1 == -F3)) {
        // f p1 + (+-f) p3 = f (p1 +- p3): the common factor is applied in the outputs
        const C q = F1 == F3 ? cadd(w[1], w[3]) : csub(w[1], w[3]);
        const C r = F1 == F3 ? csub(w[1], w[3]) : cadd(w[1], w[3]);
        const Rr f = Rr(F1);
        w[0] = pend_fma<K1, 1>(q, f, s0);
        w[2] = pend_fma<K1, -1>(q, f, s0);
        // out1 = d0 + (-j) f r (forward) / d0 + j f r (inverse); out3 with the opposite sign.
        // (-j) times a kind-1 factor is a kind-2 factor -f; (-j)(j f) = f is kind 1.
        constexpr int KJ = K1 == 1 ? 2 : 1;
        const Rr fj = K1 == 1 ? -f : f;  // (-j) * factor, as a factor of kind KJ
        if constexpr (!INV) {
            w[1] = pend_fma<KJ, 1>(r, fj, d0);
            w[3] = pend_fma<KJ, -1>(r, fj, d0);
        } else {
            w[1] = pend_fma<KJ, -1>(r, fj, d0);
            w[3] = pend_fma<KJ, 1>(r, fj, d0);
        }
    } else {
        const C x1 = pend_apply<K1>(w[1], Rr(F1));
        const C s1 = pend_fma<K3, 1>(w[3], Rr(F3), x1);
        const C d1 = pend_fma<K3, -1>(w[3], Rr(F3), x1);
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

template <int R, int A, int B, bool INV, int kb, int a = 1, class C>
__device__ __forceinline__ void apply_col(C (&w)[A]) {
    if constexpr (a < A) {
        using Rr = typename re_of<C>::type;
        constexpr int m = tw_exp(R, a, kb, INV);
        w[a] = pend_apply<pend_kind(R, m)>(w[a], Rr(pend_fac(R, m)));
        apply_col<R, A, B, INV, kb, a + 1>(w);
    }
}

template <int R, int A, int B, bool INV, int kb, class C>
__device__ __forceinline__ void dft_cols(C (&u)[A][B], C (&v)[R]) {
    if constexpr (kb < B) {
        C w[A];
        load_col<R, A, B, INV, kb>(u, w);
        if constexpr (A == 2) {
            dft2_pend<R, kb, INV>(w);
        } else if constexpr (A == 4) {
            dft4_pend<R, kb, INV>(w);
        } else {
            apply_col<R, A, B, INV, kb>(w);
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
