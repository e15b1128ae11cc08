// Complex arithmetic for the overlap-save kernels, written for sm_100a.
//
// fp32: a complex sample is a float2 held in an even/odd register pair, and every complex add,
// subtract, real scale and multiply goes through Blackwell's packed FP32x2 pipe
// (`add/sub/mul/fma.rn.f32x2`, SASS FADD2/FMUL2/FFMA2). ptxas folds the component swap and the
// half-negation of a*(+-j) into the operand selectors (`.F32x2.LO_HI.NP`), so:
//   complex add/sub          -> 1 instruction (scalar: 2)
//   a +- (-j) b              -> 1 instruction (scalar: 2)
//   complex multiply         -> 2 instructions (FMUL2 + FFMA2; scalar: 4)
// fp64: plain DADD/DFMA (there is no packed FP64 pipe).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fcvbw_gpu {

template <class R>
struct cx_of;
template <>
struct cx_of<float> {
    using type = float2;
};
template <>
struct cx_of<double> {
    using type = double2;
};
template <class R>
using cx_t = typename cx_of<R>::type;

__device__ __forceinline__ uint64_t pk(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float2 upk(uint64_t r) {
    float2 a;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
    return a;
}
__device__ __forceinline__ uint64_t pk(float2 a) { return pk(a.x, a.y); }

// ---------------------------------------------------------------- fp32 (packed)
__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
    return upk(r);
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
    return upk(r);
}
// a * s, s real
__device__ __forceinline__ float2 cscale(float2 a, float s) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(s, s)));
    return upk(r);
}
// a * w
__device__ __forceinline__ float2 cmul(float2 a, float2 w) {
    uint64_t t, r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(pk(a)), "l"(pk(w.x, w.x)));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(a.y, a.x)), "l"(pk(-w.y, w.y)), "l"(t));
    return upk(r);
}
// a * conj(w)
__device__ __forceinline__ float2 cmulc(float2 a, float2 w) {
    uint64_t t, r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(pk(a)), "l"(pk(w.x, w.x)));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(a.y, a.x)), "l"(pk(w.y, -w.y)), "l"(t));
    return upk(r);
}
// a * s + b, s real (one FFMA2)
__device__ __forceinline__ float2 cfma(float2 a, float s, float2 b) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(a)), "l"(pk(s, s)), "l"(pk(b)));
    return upk(r);
}
// (a.x * s0 + b.x, a.y * s1 + b.y) (one FFMA2)
__device__ __forceinline__ float2 cfma2(float2 a, float s0, float s1, float2 b) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(a)), "l"(pk(s0, s1)), "l"(pk(b)));
    return upk(r);
}
// (a.y * s0 + b.x, a.x * s1 + b.y): a times a real multiple of +-j, plus b (one FFMA2; the
// component swap folds into the operand selector as in cmul)
__device__ __forceinline__ float2 cfma_swap(float2 a, float s0, float s1, float2 b) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(a.y, a.x)), "l"(pk(s0, s1)), "l"(pk(b)));
    return upk(r);
}
// (a.y * s0, a.x * s1) (one FMUL2)
__device__ __forceinline__ float2 cscale_swap(float2 a, float s0, float s1) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a.y, a.x)), "l"(pk(s0, s1)));
    return upk(r);
}
// a + (-j) b  and  a - (-j) b
__device__ __forceinline__ float2 cadd_mj(float2 a, float2 b) { return cadd(a, make_float2(b.y, -b.x)); }
__device__ __forceinline__ float2 csub_mj(float2 a, float2 b) { return cadd(a, make_float2(-b.y, b.x)); }
__device__ __forceinline__ float2 cmul_mj(float2 a) { return make_float2(a.y, -a.x); }
__device__ __forceinline__ float2 cneg(float2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ float2 czero(float2) { return make_float2(0.f, 0.f); }

// ---------------------------------------------------------------- fp64 (scalar pipe)
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cmul(double2 a, double2 w) {
    return make_double2(fma(a.x, w.x, -a.y * w.y), fma(a.x, w.y, a.y * w.x));
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 w) {
    return make_double2(fma(a.x, w.x, a.y * w.y), fma(a.y, w.x, -a.x * w.y));
}
__device__ __forceinline__ double2 cfma(double2 a, double s, double2 b) {
    return make_double2(fma(a.x, s, b.x), fma(a.y, s, b.y));
}
__device__ __forceinline__ double2 cfma2(double2 a, double s0, double s1, double2 b) {
    return make_double2(fma(a.x, s0, b.x), fma(a.y, s1, b.y));
}
__device__ __forceinline__ double2 cfma_swap(double2 a, double s0, double s1, double2 b) {
    return make_double2(fma(a.y, s0, b.x), fma(a.x, s1, b.y));
}
__device__ __forceinline__ double2 cscale_swap(double2 a, double s0, double s1) {
    return make_double2(a.y * s0, a.x * s1);
}
__device__ __forceinline__ double2 cadd_mj(double2 a, double2 b) { return make_double2(a.x + b.y, a.y - b.x); }
__device__ __forceinline__ double2 csub_mj(double2 a, double2 b) { return make_double2(a.x - b.y, a.y + b.x); }
__device__ __forceinline__ double2 cmul_mj(double2 a) { return make_double2(a.y, -a.x); }
__device__ __forceinline__ double2 cneg(double2 a) { return make_double2(-a.x, -a.y); }
__device__ __forceinline__ double2 czero(double2) { return make_double2(0.0, 0.0); }

template <class C>
__device__ __forceinline__ C cmake(double re, double im);
template <>
__device__ __forceinline__ float2 cmake<float2>(double re, double im) {
    return make_float2(static_cast<float>(re), static_cast<float>(im));
}
template <>
__device__ __forceinline__ double2 cmake<double2>(double re, double im) {
    return make_double2(re, im);
}

}  // namespace fcvbw_gpu
