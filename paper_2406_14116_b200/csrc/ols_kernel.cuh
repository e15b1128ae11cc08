// Fused overlap-save kernel: framing -> FFT_N -> x H(k; b_N[block]) -> IFFT_N -> discard, for
// every block of every channel, in ONE launch. Replaces OlsEngine::run_block
// (proj/include/fcvbw/engine.hpp:139-172) together with the Radix2Fft calls it makes
// (proj/include/fcvbw/fft.hpp:55-108) and the CLI block loop that drives it
// (proj/tools/fcvbw_cli.cpp:100-113).
//
// Work decomposition. One "group" of T = N/E threads owns one block at a time; thread j of the
// group holds E complex values in registers, always in the "q-layout": register q <-> sequence
// index j + T*q. The FFT is a Stockham auto-sort transform over the radix plan
// {E, r_1, ..., r_{P-1}}: pass 0 is an E-point register DFT over exactly what the coalesced load
// delivered, later passes exchange through padded shared memory. The forward transform ends, and
// the inverse transform begins, in the q-layout, so the spectral multiply needs no reordering and
// there is no bit reversal anywhere. Groups are persistent: each warp walks ONE contiguous run of
// (channel, block) work items, its groups side by side, so the (N-M)-sample halo of a block is the
// tail of a segment the same warp fetched one step earlier and its re-read is served by L2.
// Launches are chained with programmatic dependent launch: the next launch's prologue (table
// staging, barrier init) overlaps this launch's tail, and griddepcontrol.wait orders its first
// global access after this launch completes.
//
// Coefficients (SURVEY.md section 8(a) contract), built on the fly per block from the integer
// b_N only (set_bandwidth, engine.hpp:70-80, is pure index arithmetic):
//   k1 = b - dN/2 + 1, k2 = b + dN/2 - 1, f = min(k, N - k)
//   g(k) = 1 if f < k1; V[f - k1] if f <= k2; 0 otherwise      (spectrum.hpp:170-202)
//   P(k) = phase_table(N, L)[k]                                  (spectrum.hpp:208-219)
// COEF_SHIFT (L odd, i.e. L-1 even): P(k) = W_N^{k (L-1)/2} exactly for every k, so multiplying
//   by P is an exact circular delay of (L-1)/2 samples; it is applied as an index rotation at the
//   store, removing the complex multiply altogether.
// COEF_PHASE (L even): P(k) is multiplied explicitly from the reference phase table.
// COEF_RAW: arbitrary table H(k) (the raw-table engine, engine.hpp:47-56, 163-165).
// The inverse transform's 1/N (fft.hpp:75-76) is folded into g (power of two: exact).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "cplx.cuh"
#include "dft.cuh"
#include "sm100.cuh"


__host__ __device__ constexpr int minb_for(int threads, int mb) { return (mb * 128) / threads > 0 ? (mb * 128) / threads : 1; }
namespace fcvbw_gpu {

// COEF_SHIFT_Q is COEF_SHIFT at the BASELINE geometry L - 1 = N/4 (delay N/8): the stored output
// registers are then a compile-time range, so the discard costs nothing.
enum CoefMode : int { COEF_SHIFT = 0, COEF_PHASE = 1, COEF_RAW = 2, COEF_SHIFT_Q = 3 };

template <class R>
struct OlsArgs {
    const cx_t<R>* x;  // x[ch * x_cs + (i - x_first)] holds input sample i of channel ch
    cx_t<R>* y;        // y[ch * y_cs + (i - y_first)] receives output sample i
    int64_t x_first, y_first, x_cs, y_cs;
    int64_t S;                    // samples per channel (global stream length)
    int64_t blk_begin;            // global block range [blk_begin, blk_begin + nblk)
    int nblk;
    int total;                    // channels * nblk work items (< 2^31; the host splits larger runs)
    int tma_lo, tma_hi;           // relative blocks whose whole segment is in range and 16B-aligned
                                  // (TMA-eligible: tma_lo <= bl <= tma_hi; tma_lo > tma_hi disables)
    const int* bsched;            // b per (channel, global block), or null -> b_const
    int64_t b_cs;                 // channel stride of bsched (0: one schedule for all channels)
    int b_const;
    int M, half_dn, LV, shift;    // shift = (L-1)/2 for COEF_SHIFT
    const R* V;                   // LV profile values, pre-scaled by 1/N
    const cx_t<R>* coef;          // COEF_PHASE: phase table; COEF_RAW: table / N
    const cx_t<R>* tw;            // per-thread twiddle table (plan_twiddles layout)
    R inv_n;
    // real-input I/O: x/y are real [channels][...] buffers (xr / yr).
    //   IO = 1: one real block per transform, zero imaginary part (raw tables, which may be
    //           asymmetric: the reference keeps Re(IFFT), fft.hpp:68-78);
    //   IO = 2: work item p covers real blocks 2p and 2p + 1 of one channel, carried as (re, im)
    //           of ONE transform when both use the same b (exact: structured H is conjugate-
    //           symmetric); blk_begin / nblk then count PAIRS and nblk_real counts real blocks.
    const R* xr;
    R* yr;
    int64_t nblk_real;
    // IO = 2: 1 pairs blocks that share b; 0 runs every real block as its own transform with a
    // zero imaginary part (the streaming entry points: a block's output then never depends on the
    // block it would have been paired with, so caller batching stays bit-identical, and it equals
    // the complex path on x + 0j bit for bit)
    int pair_real;
    // parity (IO = 3 instantiation only): every work item w writes the mask g(k)/N it applies to
    // gdump[w * N + k] (fcvbw_gpu_mask_dump)
    R* gdump;
    // warps (units) per CTA that take items (0: all); set by the launcher for small launches
    int units;
};

// ------------------------------------------------------------------ radix plan
__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n / 2); }

template <int N, int E, bool TWF = false>
struct Plan {
    static_assert((N & (N - 1)) == 0 && (E & (E - 1)) == 0 && E <= N, "powers of two");
    static constexpr int T = N / E;
    static constexpr int LE = ilog2(E);
    static constexpr int LREM = ilog2(N / E);
    static constexpr int NP1 = LREM == 0 ? 0 : (LREM + LE - 1) / LE;  // passes after the first
    static constexpr int P = 1 + NP1;
    __host__ __device__ static constexpr int radix(int p) {
        return p == 0 ? E
                      : (1 << (LREM / (NP1 ? NP1 : 1) + ((p - 1) < (LREM % (NP1 ? NP1 : 1)) ? 1 : 0)));
    }
    __host__ __device__ static constexpr int ns(int p) { return p == 0 ? 1 : ns(p - 1) * radix(p - 1); }
    // Inter-pass twiddles W^{i k}, i in [1, r), are factored along the codelet's own four-step
    // split (i = i0 + LO i1, LO = its stride A): W^{i0 k} W^{LO i1 k}. Per butterfly the thread
    // loads (LO - 1) + (HI - 1) base values instead of r - 1 and forms each product right before
    // the sub-DFT that consumes it.
    __host__ __device__ static constexpr int tw_lo(int r) { return r == 32 ? FCVBW_DFT32_A : (r >= 16 ? 4 : (r == 8 ? 2 : r)); }
    __host__ __device__ static constexpr int tw_hi(int r) { return (r + tw_lo(r) - 1) / tw_lo(r); }
    // TWF (full table, kept in shared memory): all r - 1 twiddles per butterfly, no products
    __host__ __device__ static constexpr int tw_cnt(int r) {
        return TWF ? r - 1 : (tw_lo(r) - 1) + (tw_hi(r) - 1);
    }
    // base-table entries (per thread) before pass p
    __host__ __device__ static constexpr int tw_off(int p) {
        return p <= 1 ? 0 : tw_off(p - 1) + (E / radix(p - 1)) * tw_cnt(radix(p - 1));
    }
    static constexpr int TW_PER_THREAD = tw_off(P);
    // compact full table (TWK = 4): pass p holds W_{ns r}^{i k} at [(i - 1) ns + k], k in [0, ns)
    __host__ __device__ static constexpr int tw_coff(int p) {
        return p <= 1 ? 0 : tw_coff(p - 1) + (radix(p - 1) - 1) * ns(p - 1);
    }
    static constexpr int TW_COMPACT = tw_coff(P);
    __host__ __device__ static constexpr bool cnt_even(int p) {
        return p >= P ? true : ((tw_cnt(radix(p)) % 2 == 0) && cnt_even(p + 1));
    }
    // fp32 factored tables stored as pairs of consecutive entries per thread (one 16-byte load
    // brings two twiddles): every pass's per-butterfly entry count must be even
    static constexpr bool PAIRABLE = !TWF && cnt_even(1);
};

template <class R, int N, int E, bool TWF>
__host__ __device__ constexpr bool tw_paired() {
    return sizeof(R) == 4 && Plan<N, E, TWF>::PAIRABLE;
}

// Shared-memory padding: one element per P elements, P = min(E, one 128-byte row = 32 fp32 /
// 16 fp64 elements). The first Stockham write has stride E inside a group and the groups of a
// warp sit padded(N) apart, so P = E spreads a warp's 32 stores over all bank pairs (2 wavefronts)
// while the q-layout reads stay contiguous. Small-E plans with P = 32 ran 2-4-way conflicted
// (ncu N = 64 fp32: l1tex 94 %); P = E measured N = 64 / 128 / 256 fp32 0.58 / 0.56 / 0.66 ->
// 0.74 / 0.72 / 0.73 (profiles/r01_sweep.md). For the fp32 E = 64 plan a 64-element row would make
// its stride-64 writes conflict-free too (store conflicts 425 M -> 48 M per c4 launch); it measured
// 5 % slower with the early kernel (c4 0.527 vs 0.553) but 4.5 % FASTER once the fused-factor
// codelets cut the FMA work (c4 0.582 -> 0.608), so the 64-element plan pads per 64. fp64 plans
// with E = 32 pad per 32 elements: with a 16-element row the stride-E writes (34 16-byte words per
// lane) were 2-way conflicted (ncu c5_512_f64: 363 M excess store wavefronts per launch).
template <class R, int E>
__host__ __device__ constexpr int pad_log() {
    return sizeof(R) == 4 ? (E >= 64 ? 6 : (E < 32 ? ilog2(E) : 5)) : (E < 16 ? ilog2(E) : (E >= 32 ? 5 : 4));
}
template <class R, int E>
__device__ __forceinline__ int padi(int a) {
    return a + (a >> pad_log<R, E>());
}
template <class R, int E>
__host__ __device__ constexpr int padded(int n) {
    return n + (n >> pad_log<R, E>());
}
template <class R, int E>
__host__ __device__ constexpr int row_len() {
    return 1 << pad_log<R, E>();
}

// Coefficient-region rule shared by the fused kernel and the parity dump (bin_region,
// spectrum.hpp:194-202): f = min(k, N - k) against [k1, k1 + span].
__device__ __forceinline__ int bin_region_of(int f, int k1, int span) {
    const int idx = f - k1;
    return idx < 0 ? 0 : (idx <= span ? 1 : 2);
}

template <int T>
__device__ __forceinline__ void group_sync(int g) {
    if constexpr (T <= 32) {
        __syncwarp();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(T) : "memory");
    }
}

// Inter-pass twiddle source: the table in memory (shared or global, `const C*`, entry idx of
// thread j at tw[idx * T + j]) or the thread's whole table held in registers (TwRegs), loaded once
// per kernel and used by the forward AND the inverse transform of every block (the inverse reads
// the same entries, conjugated).
template <class C, int K>
struct TwRegs {
    C r[K > 0 ? K : 1];
};
template <int T, class C>
__device__ __forceinline__ C tw_get(const C* tw, int idx, int j) {
    return tw[idx * T + j];
}
template <int T, class C, int K>
__device__ __forceinline__ C tw_get(const TwRegs<C, K>& tw, int idx, int) {
    return tw.r[idx];
}
// compact full table (TWK = 4), indexed by (pass, i, k) instead of (entry, thread): tables whose
// twiddles repeat across threads (k = (j + m T) mod ns with ns < T E / r) shrink by T E / (r ns)
template <class C>
struct TwCompact {
    const C* p;
};
template <class X>
struct is_compact : std::false_type {};
template <class C>
struct is_compact<TwCompact<C>> : std::true_type {};

// Full twiddle tables in tangent form {t, wr} (W = wr (1 + j t), Pass::run), except fp64 N = 256
// where the fused form measured 4 % slower (profiles/r01_sweep.md); that plan keeps {wr, wi}.
template <class R, int N>
__host__ __device__ constexpr bool tw_tangent(bool twf) {
    return twf && !(sizeof(R) == 8 && N == 256);
}

// ------------------------------------------------------------------ Stockham passes
template <class R, int N, int E, bool INV, int p, bool TWF>
struct Pass {
    using C = cx_t<R>;
    using PL = Plan<N, E, TWF>;
    static constexpr int T = PL::T;
    // pass p-1 results (registers, q-layout) -> shared memory in Stockham output order.
    // Both special cases that occur in every plan keep the address a per-thread base plus a
    // compile-time offset: ns == 1 (r divides the padded row) and ns a multiple of the row.
    __device__ __forceinline__ static void write_prev(C (&v)[E], C* buf, int j) {
        constexpr int r = PL::radix(p - 1);
        constexpr int ns = PL::ns(p - 1);
        constexpr int LEN = row_len<R, E>();
        constexpr bool linear = (ns == 1 && LEN % r == 0) || (ns % LEN == 0);
#pragma unroll
        for (int m = 0; m < E / r; ++m) {
            const int jp = j + m * T;
            const int idxd = (jp / ns) * ns * r + (jp % ns);
            if constexpr (linear) {
                C* base = buf + padi<R, E>(idxd);
#pragma unroll
                for (int i = 0; i < r; ++i) base[padded<R, E>(i * ns)] = v[m + i * (E / r)];
            } else {
#pragma unroll
                for (int i = 0; i < r; ++i) buf[padi<R, E>(idxd + i * ns)] = v[m + i * (E / r)];
            }
        }
    }

    template <class TW, class AfterRead>
    __device__ __forceinline__ static void run(C (&v)[E], C* buf, const TW& tw, int j, int g, AfterRead&& after_read) {
        if constexpr (p < PL::P) {
            constexpr int r = PL::radix(p);
            group_sync<T>(g);  // previous readers of buf are done
            write_prev(v, buf, j);
            group_sync<T>(g);
            const C* rb = buf + padi<R, E>(j);  // pad(j + Tq) = pad(j) + pad(Tq)
#pragma unroll
            for (int q = 0; q < E; ++q) v[q] = rb[padded<R, E>(T * q)];
            if constexpr (p == PL::P - 1) after_read();  // buf is idle from here to the next transform
            // twiddles W_{ns r}^{i k}, k = (j + mT) mod ns: either the full per-thread table in
            // shared memory (TWF) or the factored base table (shared memory or L1-resident global)
            constexpr int LO = PL::tw_lo(r), HI = PL::tw_hi(r), CNT = PL::tw_cnt(r);
            constexpr int TO = PL::tw_off(p);
            constexpr int NS = PL::ns(p);
            // full-table entry i (1 <= i < r) of butterfly m
            auto twe = [&](int m, int i) -> C {
                if constexpr (is_compact<TW>::value)
                    return tw.p[PL::tw_coff(p) + (i - 1) * NS + ((j + m * T) & (NS - 1))];
                else
                    return tw_get<T>(tw, TO + m * CNT + i - 1, j);
            };
#pragma unroll
            for (int m = 0; m < E / r; ++m) {
                C t[r];
#pragma unroll
                for (int i = 0; i < r; ++i) t[i] = v[m + i * (E / r)];
                if constexpr (TWF && !tw_tangent<R, N>(TWF)) {
                    auto pre = [&](int i, C x) -> C {
                        if (i == 0) return x;
                        const C w = twe(m, i);
                        return INV ? cmulc(x, w) : cmul(x, w);
                    };
                    dft<r, INV>(t, pre);
                } else if constexpr (TWF) {
                    // table entry {t, wr}: W = wr (1 + j t). The input keeps p = x (1 +- j t) (one
                    // FFMA2, conjugate for the inverse) and wr is applied as a real factor inside
                    // the first butterfly level (dft scale hook)
                    auto pre = [&](int i, C x) -> C {
                        if (i == 0) return x;
                        const R tt = twe(m, i).x;
                        return INV ? cfma_swap(x, tt, -tt, x) : cfma_swap(x, -tt, tt, x);
                    };
                    auto wr = [&](int i) -> R { return i == 0 ? R(1) : twe(m, i).y; };
                    dft<r, INV>(t, pre, make_scale(wr));
                } else {
                    const C* twp = tw + TO * T + j;
                    C lo[LO], hi[HI];
                    if constexpr (tw_paired<R, N, E, TWF>()) {
                        // entries (2c, 2c + 1) of butterfly m are one float4 per thread
                        const float4* tp = reinterpret_cast<const float4*>(tw) + (PL::tw_off(p) / 2) * T + j;
                        C e[CNT];
#pragma unroll
                        for (int c = 0; c < CNT; c += 2) {
                            const float4 q4 = tp[(m * CNT / 2 + c / 2) * T];
                            e[c] = cmake<C>(q4.x, q4.y);
                            e[c + 1] = cmake<C>(q4.z, q4.w);
                        }
#pragma unroll
                        for (int i0 = 1; i0 < LO; ++i0) lo[i0] = e[i0 - 1];
#pragma unroll
                        for (int i1 = 1; i1 < HI; ++i1) hi[i1] = e[LO - 1 + i1 - 1];
                    } else {
#pragma unroll
                        for (int i0 = 1; i0 < LO; ++i0) lo[i0] = twp[(m * CNT + i0 - 1) * T];
#pragma unroll
                        for (int i1 = 1; i1 < HI; ++i1) hi[i1] = twp[(m * CNT + LO - 1 + i1 - 1) * T];
                    }
                    auto pre = [&](int i, C x) -> C {
                        const int i0 = i % LO, i1 = i / LO;
                        if (i == 0) return x;
                        const C w = i1 == 0 ? lo[i0] : (i0 == 0 ? hi[i1] : cmul(hi[i1], lo[i0]));
                        return INV ? cmulc(x, w) : cmul(x, w);
                    };
                    dft<r, INV>(t, pre);
                }
#pragma unroll
                for (int i = 0; i < r; ++i) v[m + i * (E / r)] = t[i];
            }
            Pass<R, N, E, INV, p + 1, TWF>::run(v, buf, tw, j, g, after_read);
        }
    }
};

struct nothing {
    __device__ __forceinline__ void operator()() const {}
};

// passes 1 .. P-1 (pass 0, the register DFT, is the caller's)
template <class R, int N, int E, bool INV, bool TWF, class TW, class AfterRead = nothing>
__device__ __forceinline__ void fft_rest(cx_t<R> (&v)[E], cx_t<R>* buf, const TW& tw, int j, int g,
                                         AfterRead after_read = AfterRead{}) {
    if constexpr (Plan<N, E, TWF>::P > 1)
        Pass<R, N, E, INV, 1, TWF>::run(v, buf, tw, j, g, after_read);
    else
        after_read();
}

template <class R, int N, int E, bool INV, bool TWF, class TW, class AfterRead = nothing>
__device__ __forceinline__ void fft_q(cx_t<R> (&v)[E], cx_t<R>* buf, const TW& tw, int j, int g,
                                      AfterRead after_read = AfterRead{}) {
    dft<E, INV>(v);  // pass 0: ns = 1, no twiddles
    fft_rest<R, N, E, INV, TWF>(v, buf, tw, j, g, after_read);
}

// ------------------------------------------------------------------ the fused kernel
// Spectral mask g(k)/N for the bins k = j + T q a thread holds (q-layout), built from the integer
// b only: f = min(k, N - k); 1 if f < k1, V[f - k1] if f <= k2, 0 otherwise (bin_region /
// magnitude_samples, spectrum.hpp:170-202), with the inverse transform's 1/N folded in. FAST
// (span < T): at most one transition register per half-spectrum of the thread, located once per
// block by two integer divisions, so each register costs two compares and two selects. The SAME
// object feeds the inverse transform's first butterfly level and the mask dump (OlsArgs::gdump).
// TABLE (mask_table<R, N>()): g depends on (f - k1) only, so one b-independent table per CTA in
// shared memory, gt[d + MASK_OFF] = 1/N for d < 0, V[d]/N for 0 <= d <= span, 0 beyond, turns the
// mask of register q into ONE shared-memory load at a per-thread base plus a compile-time offset
// (lower half f = j + T q, upper half f = N - j - T q; lanes read consecutive words). It replaces
// the two compares and two selects per register of FAST (ncu c3: ISETP + FSEL were 141 of the
// 1402 warp-instructions per block).
// Measured per plan (profiles/r02_sweep.md, "Mask table"): fp32 N = 512 .. 4096 and fp64 N = 512 /
// 1024 gain (N = 2048 fp32: +11 %), the small-N plans (several groups per warp read different
// table rows) and the largest plans (shared memory is their bottleneck) lose 1-5 % and keep the
// compare / select form. Bit masks over log2 N.
#ifndef FCVBW_MASKT_F32
#define FCVBW_MASKT_F32 ((1 << 9) | (1 << 10) | (1 << 11) | (1 << 12))
#endif
#ifndef FCVBW_MASKT_F64
#define FCVBW_MASKT_F64 ((1 << 9) | (1 << 10))
#endif
template <class R, int N>
__host__ __device__ constexpr bool mask_table() {
    return ((sizeof(R) == 4 ? (long long)(FCVBW_MASKT_F32) : (long long)(FCVBW_MASKT_F64)) >> ilog2(N)) & 1;
}
// table index of d = f - k1: k1 is clamped to [-half_dn, N/2 + 1], f is in [0, N/2]
template <int N>
__host__ __device__ constexpr int mask_off() { return N / 2 + 1; }
__host__ __device__ constexpr int mask_table_len(int N, int half_dn) { return N + half_dn + 2; }

// TABLE4 (mask_table4<R, N>(), fp32): the same table TRANSPOSED with period T and kept in four
// shifted copies, C_s[r][m] = G[r + T (m + s)]. A thread's E/2 masks of one half-spectrum are
// G[u + T m], m = 0 .. E/2-1 (u = r + T a its first table index), i.e. E/2 CONSECUTIVE words of
// row r of copy s = a mod 4 starting at the 16-byte aligned column a - s: E/8 LDS.128 per
// half-spectrum instead of E/2 LDS.32. With the flat table the register-starved N = 1024 kernel
// issued each mask load right before its use (ncu: 13 % of all stall samples on those 32
// load-use pairs); one vector load feeds four butterflies. The upper half runs over q' = E-1-q,
// which ascends in the table like the lower half.
// Measured (profiles/r02_sweep.md, "Transposed mask table"): c3 / c5_1024_f32 +1.7 %, c2 +0.8 %,
// c5_2048_f32 +0.9 %, c5_512_f32 +2.7 %, mixed real pairs +1 %.
#ifndef FCVBW_MASKT4_F32
#define FCVBW_MASKT4_F32 ((1 << 9) | (1 << 10) | (1 << 11))
#endif
template <class R, int N>
__host__ __device__ constexpr bool mask_table4() {
    return sizeof(R) == 4 && mask_table<R, N>() && (((long long)(FCVBW_MASKT4_F32) >> ilog2(N)) & 1);
}
// row length of the transposed copies: first index u <= OFF + T + half_dn, E/2 columns from the
// aligned start, rounded up to a multiple of 4 with an odd number of 16-byte words per row (rows of
// consecutive r then fall into distinct bank groups)
__host__ __device__ constexpr int mask4_row(int N, int T, int E, int half_dn) {
    const int need = (N / 2 + 1 + T + half_dn) / T + E / 2 + 1;
    const int w = (need + 3) / 4;
    return 4 * (w | 1);
}
// table words behind V (flat or transposed), plus alignment slack for the vector form
__host__ __device__ constexpr int mask_table_words(int N, int T, int E, int half_dn, bool t4) {
    return t4 ? 4 * T * mask4_row(N, T, E, half_dn) : ((mask_table_len(N, half_dn) + 3) & ~3);
}
// The table sits in front of V in shared memory (16-byte aligned): gt = vs - words.
template <class R, int N, int E>
__device__ __forceinline__ const R* mask_table_of(const R* vs, int half_dn) {
    return vs - mask_table_words(N, N / E, E, half_dn, mask_table4<R, N>());
}

enum MaskKind : int { MASK_GENERAL = 0, MASK_FAST = 1, MASK_TABLE = 2, MASK_TABLE4 = 3 };

template <class R, int N, int E, int KIND>
struct MaskGen {
    static constexpr int T = N / E;
    static constexpr bool FAST = KIND == MASK_FAST;
    const R* vs;
    R inv_n;
    int j, k1, span;
    int qt, qu;  // FAST: transition register of the lower / upper half-spectrum
    R vt, vu;
    const R *pl, *pu;  // TABLE: bases of the lower / upper half-spectrum reads
    __device__ __forceinline__ MaskGen(const R* vs_, const R* gt, R inv_n_, int j_, int b, int half_dn)
        : vs(vs_), inv_n(inv_n_), j(j_), k1(b - half_dn + 1), span(2 * half_dn - 2) {  // spectrum.hpp:161-165
        if constexpr (KIND == MASK_TABLE) {
            const int k1c = min(max(k1, -half_dn), N / 2 + 1);
            pl = gt + (mask_off<N>() + j - k1c);
            pu = pl + (N - 2 * j);
        } else if constexpr (KIND == MASK_TABLE4) {
            const int k1c = min(max(k1, -half_dn), N / 2 + 1);
            const int rl = mask4_row(N, T, E, half_dn);
            auto row = [&](int u) -> const R* {  // first table index u = r + T a of a half-spectrum
                const int r = u & (T - 1), a_ = u / T;
                return gt + (((a_ & 3) * T + r) * rl + (a_ & ~3));
            };
            pl = row(mask_off<N>() + j - k1c);      // lower half: f = j + T q
            pu = row(mask_off<N>() + T - j - k1c);  // upper half, q' = E-1-q: f = T - j + T q'
        } else if constexpr (FAST) {
            // lower half (q < E/2): f = j + T q; passband while T q < d1
            const int d1 = k1 - j;
            qt = d1 <= 0 ? 0 : (d1 + T - 1) / T;
            const int it = T * qt - d1;
            vt = (qt < E / 2 && it <= span) ? vs[it] : R(0);
            // upper half (q >= E/2): f = N - j - T q; passband while T q > e1
            const int e1 = N - j - k1;
            qu = e1 >= 0 ? e1 / T : -1;
            const int iu = e1 - T * qu;
            vu = (qu >= E / 2 && iu <= span) ? vs[iu] : R(0);
        }
    }
    __device__ __forceinline__ R operator()(int q) const {
        if constexpr (KIND == MASK_TABLE) {
            return q < E / 2 ? pl[T * q] : pu[-T * q];
        } else if constexpr (KIND == MASK_TABLE4) {
            const int m = q < E / 2 ? q : E - 1 - q;
            const float4 w4 = reinterpret_cast<const float4*>(q < E / 2 ? pl : pu)[m / 4];
            return (m & 3) == 0 ? w4.x : ((m & 3) == 1 ? w4.y : ((m & 3) == 2 ? w4.z : w4.w));
        } else if constexpr (FAST) {
            if (q < E / 2) return q < qt ? inv_n : (q == qt ? vt : R(0));
            return q > qu ? inv_n : (q == qu ? vu : R(0));
        } else {
            const int f = (q < E / 2) ? (j + T * q) : (N - j - T * q);  // min(k, N - k)
            const int region = bin_region_of(f, k1, span);
            return region == 0 ? inv_n : (region == 1 ? vs[f - k1] : R(0));
        }
    }
    // mask dump (parity): the g(k)/N this thread applies, at row[k]
    __device__ __forceinline__ void dump(R* row) const {
        if (row) {
#pragma unroll
            for (int q = 0; q < E; ++q) row[j + T * q] = (*this)(q);
        }
    }
};

// The mask generator of a block: the table form when the plan carries the table, else FAST when
// at most one transition register per half-spectrum lands in a thread (span < T), else the
// general per-register rule. f(mg) runs with the chosen generator.
template <class R, int N, int E, class F>
__device__ __forceinline__ void with_mask(const OlsArgs<R>& a, const R* vs, int j, int b, F&& f) {
    constexpr int T = N / E;
    if constexpr (mask_table4<R, N>())
        f(MaskGen<R, N, E, MASK_TABLE4>(vs, mask_table_of<R, N, E>(vs, a.half_dn), a.inv_n, j, b, a.half_dn));
    else if constexpr (mask_table<R, N>())
        f(MaskGen<R, N, E, MASK_TABLE>(vs, mask_table_of<R, N, E>(vs, a.half_dn), a.inv_n, j, b, a.half_dn));
    else if (2 * a.half_dn - 2 < T)
        f(MaskGen<R, N, E, MASK_FAST>(vs, nullptr, a.inv_n, j, b, a.half_dn));
    else
        f(MaskGen<R, N, E, MASK_GENERAL>(vs, nullptr, a.inv_n, j, b, a.half_dn));
}
template <class R, int N, int E, class F>
__device__ __forceinline__ void with_mask2(const OlsArgs<R>& a, const R* vs, int j, int b0, int b1, F&& f) {
    constexpr int T = N / E;
    if constexpr (mask_table4<R, N>())
        f(MaskGen<R, N, E, MASK_TABLE4>(vs, mask_table_of<R, N, E>(vs, a.half_dn), a.inv_n, j, b0, a.half_dn),
          MaskGen<R, N, E, MASK_TABLE4>(vs, mask_table_of<R, N, E>(vs, a.half_dn), a.inv_n, j, b1, a.half_dn));
    else if constexpr (mask_table<R, N>())
        f(MaskGen<R, N, E, MASK_TABLE>(vs, mask_table_of<R, N, E>(vs, a.half_dn), a.inv_n, j, b0, a.half_dn),
          MaskGen<R, N, E, MASK_TABLE>(vs, mask_table_of<R, N, E>(vs, a.half_dn), a.inv_n, j, b1, a.half_dn));
    else if (2 * a.half_dn - 2 < T)
        f(MaskGen<R, N, E, MASK_FAST>(vs, nullptr, a.inv_n, j, b0, a.half_dn),
          MaskGen<R, N, E, MASK_FAST>(vs, nullptr, a.inv_n, j, b1, a.half_dn));
    else
        f(MaskGen<R, N, E, MASK_GENERAL>(vs, nullptr, a.inv_n, j, b0, a.half_dn),
          MaskGen<R, N, E, MASK_GENERAL>(vs, nullptr, a.inv_n, j, b1, a.half_dn));
}

// Spectral multiply by g(k) (and P(k) for COEF_PHASE) in the q-layout, k = j + T q.
template <class R, int N, int E, int MODE>
__device__ __forceinline__ void spectral_multiply(cx_t<R> (&v)[E], const OlsArgs<R>& a, const R* vs, int j,
                                                  int b, R* gdump_row) {
    constexpr int T = N / E;
    if constexpr (MODE == COEF_RAW) {
#pragma unroll
        for (int q = 0; q < E; ++q) v[q] = cmul(v[q], __ldg(a.coef + j + T * q));
    } else {
        auto apply = [&](const auto& mg) {
            mg.dump(gdump_row);
#pragma unroll
            for (int q = 0; q < E; ++q) v[q] = cscale(v[q], mg(q));
        };
        with_mask<R, N, E>(a, vs, j, b, apply);
        if constexpr (MODE == COEF_PHASE) {
#pragma unroll
            for (int q = 0; q < E; ++q) v[q] = cmul(v[q], __ldg(a.coef + j + T * q));
        }
    }
}

// Spectral multiply followed by the inverse transform. For the structured modes of single-warp
// (or smaller) groups the mask g(k) is a real factor per register, fused into the first butterfly
// level of the inverse pass-0 DFT (x0 g0 + x1 g1 = FMUL2 + FFMA2); the phase is an index rotation
// at the store. Multi-warp groups multiply first (spectral_multiply), same MaskGen.
template <class R, int N, int E, int MODE, bool TWF, class TW, class AfterRead = nothing>
__device__ __forceinline__ void multiply_inverse(cx_t<R> (&v)[E], const OlsArgs<R>& a, const R* vs, int j, int b,
                                                 cx_t<R>* buf, const TW& tw, int g, R* gdump_row,
                                                 AfterRead after_read = AfterRead{}) {
    constexpr int T = N / E;
    if constexpr ((MODE == COEF_SHIFT || MODE == COEF_SHIFT_Q) && T <= 32) {
        auto fused = [&](const auto& mg) {
            mg.dump(gdump_row);
            dft<E, true>(v, no_pre{}, make_scale(mg));
        };
        with_mask<R, N, E>(a, vs, j, b, fused);
        fft_rest<R, N, E, true, TWF>(v, buf, tw, j, g, after_read);
    } else {
        spectral_multiply<R, N, E, MODE>(v, a, vs, j, b, gdump_row);
        fft_q<R, N, E, true, TWF>(v, buf, tw, j, g, after_read);
    }
}

// Spectral multiply of a real block pair carried as x0 + j x1 whose blocks use different b:
// Y(k) = Z(k) (g0 + g1)/2 + conj(Z(N - k)) (g0 - g1)/2 (times P(k) for COEF_PHASE), g = the real
// masks of MaskGen (1/N included). The mirrored bins come through the group's exchange buffer,
// idle between the forward transform's last read and the inverse transform's first write: thread
// j writes its bins k = j + T q in natural order and reads N - k = (T - j) + T (E - 1 - q)
// (the same conflict-free q-layout pattern from base T - j; bin 0 of thread 0 is its own mirror).
template <class R, int N, int E, int MODE>
__device__ __forceinline__ void mixed_pair_multiply(cx_t<R> (&v)[E], const OlsArgs<R>& a, const R* vs, int j,
                                                    int b0, int b1, cx_t<R>* buf, int g) {
    using C = cx_t<R>;
    constexpr int T = N / E;
    group_sync<T>(g);  // the forward transform's last exchange reads are done
    {
        C* wb = buf + padi<R, E>(j);
#pragma unroll
        for (int q = 0; q < E; ++q) wb[padded<R, E>(T * q)] = v[q];
    }
    group_sync<T>(g);
    // pad(a + T q') = pad(a) + pad(T q') for 0 < a < T (as for the q-layout reads); thread 0's
    // mirrors T (E - q) need base 0 when T is shorter than a padded row
    constexpr int ROW = row_len<R, E>();
    const C* rb = buf + padi<R, E>(T - j);
    auto combine = [&](const auto& m0, const auto& m1) {
#pragma unroll
        for (int q = 0; q < E; ++q) {
            C m;
            if constexpr (T % ROW == 0)
                m = rb[padded<R, E>(T * (E - 1 - q))];
            else
                m = j == 0 ? buf[padded<R, E>(T * ((E - q) % E))] : rb[padded<R, E>(T * (E - 1 - q))];
            if (q == 0 && j == 0) m = v[0];
            const R g0 = m0(q), g1 = m1(q);
            const R sp = R(0.5) * (g0 + g1), dm = R(0.5) * (g0 - g1);
            // Z sp + conj(m) dm = (Z.x sp + m.x dm, Z.y sp - m.y dm)
            v[q] = cfma2(m, dm, -dm, cscale(v[q], sp));
        }
    };
    with_mask2<R, N, E>(a, vs, j, b0, b1, combine);
    if constexpr (MODE == COEF_PHASE) {
#pragma unroll
        for (int q = 0; q < E; ++q) v[q] = cmul(v[q], __ldg(a.coef + j + T * q));
    }
}

// TMA: 0 direct loads; 1 bulk prefetch of the next segment into a dedicated staging buffer per
// group, issued as soon as the current segment has been read out of it (a whole block of compute
// to land); 2 bulk prefetch into the (then idle) exchange buffer, issued after the last exchange
// read of the current item (no extra shared memory, but only the inverse's last pass and the store
// to land).
// (Mode 1, a dedicated staging buffer, and mode 3, an L2-only bulk prefetch, measured slower or
// equal in round 1 and were removed: profiles/r01_sweep.md.)
// TWK: 0 factored twiddle table read from global (L1); 1 full table staged in shared memory;
//      2 factored table staged in shared memory; 3 full table held in registers (two-pass plans);
//      4 full table staged in shared memory in the compact (pass, i, k) layout (Plan::tw_coff).
// IO_: 0 complex buffers; 1 / 2 real buffers (see OlsArgs::xr); 3 = complex buffers plus the
// parity dump of the mask every item applies (OlsArgs::gdump; a separate instantiation, so the
// production kernels carry no dump code).
template <class R, int N, int E, int MODE, int GROUPS, int TMA, int TWK, int MINB, int IO_ = 0>
__global__ void __launch_bounds__(GROUPS * Plan<N, E>::T, minb_for(GROUPS * Plan<N, E>::T, MINB)) ols_fused(OlsArgs<R> a) {
    constexpr bool DUMP = IO_ == 3;
    constexpr int IO = DUMP ? 0 : IO_;
    static_assert(TMA >= 0 && TMA <= 2, "prefetch modes: 0 direct loads, 1 staging buffer, 2 exchange-buffer staging");
    static_assert(IO != 2 || TMA != 1, "block pairs stage in the exchange buffer");
    static_assert(IO != 1 || TMA == 0, "one-real-block I/O uses direct loads");
    using C = cx_t<R>;
    constexpr bool TWF = TWK == 1 || TWK == 3 || TWK == 4;
    using PL = Plan<N, E, TWF>;
    constexpr int T = PL::T;
    constexpr uint32_t SEG_BYTES = N * sizeof(C);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* xbuf = reinterpret_cast<C*>(smem_raw);
    C* stg = xbuf + GROUPS * padded<R, E>(N);   // TMA == 1: one N-element staging buffer per group
    C* tws = stg + (TMA == 1 ? GROUPS * N : 0);  // twiddle table staged in shared memory
    static_assert(!(tw_paired<R, N, E, TWF>() && TWK != 0) ||
                      (GROUPS * padded<R, E>(N)) % 2 == 0,
                  "paired twiddle table must be 16-byte aligned in shared memory");
    constexpr bool TW_SMEM = TWK == 1 || TWK == 2 || TWK == 4;  // table staged in shared memory
    constexpr int TW_ENTRIES = TWK == 4 ? PL::TW_COMPACT : PL::TW_PER_THREAD * T;
    uint64_t* bars = reinterpret_cast<uint64_t*>(tws + (TW_SMEM ? TW_ENTRIES : 0));
    // mask table (plans that carry one; 16-byte aligned by shared-memory offset), then V
    R* vs;
    {
        unsigned char* p0 = reinterpret_cast<unsigned char*>(bars + (TMA ? GROUPS : 0));
        R* gt0 = reinterpret_cast<R*>(smem_raw + ((uint32_t(p0 - smem_raw) + 15u) & ~15u));
        vs = gt0 + ((mask_table<R, N>() && MODE != COEF_RAW)
                        ? mask_table_words(N, T, E, a.half_dn, mask_table4<R, N>()) : 0);
    }

    const int tid = threadIdx.x;
    const int g = tid / T;
    const int j = tid - g * T;
    C* buf = xbuf + g * padded<R, E>(N);
    C* stage = TMA == 1 ? stg + g * N : buf;  // TMA == 2: the next segment lands in the idle exchange buffer
    uint64_t* bar = bars + g;

    if constexpr (MODE != COEF_RAW) {
        for (int i = tid; i < a.LV; i += GROUPS * T) vs[i] = a.V[i];
        if constexpr (mask_table<R, N>()) {
            // b-independent mask table in front of V (MaskGen, MASK_TABLE / MASK_TABLE4); LV = span + 1
            const int len = mask_table_len(N, a.half_dn), span = 2 * a.half_dn - 2;
            auto g_of = [&](int i) -> R {  // flat table entry i <-> d = i - OFF
                const int d = i - mask_off<N>();
                return i >= len ? R(0) : (d < 0 ? a.inv_n : ((d <= span && d < a.LV) ? a.V[d] : R(0)));
            };
            if constexpr (mask_table4<R, N>()) {
                R* gt = const_cast<R*>(mask_table_of<R, N, E>(vs, a.half_dn));
                const int rl = mask4_row(N, T, E, a.half_dn);
                for (int i = tid; i < 4 * T * rl; i += GROUPS * T) {
                    const int m = i % rl, sr = i / rl;  // copy s = sr / T, row r = sr % T
                    gt[i] = g_of((sr % T) + T * (m + sr / T));
                }
            } else {
                R* gt = const_cast<R*>(mask_table_of<R, N, E>(vs, a.half_dn));
                for (int i = tid; i < len; i += GROUPS * T) gt[i] = g_of(i);
            }
        }
    }
    if constexpr (TW_SMEM) {
        for (int i = tid; i < TW_ENTRIES; i += GROUPS * T) tws[i] = a.tw[i];
    }
    const C* twsrc = TW_SMEM ? static_cast<const C*>(tws) : a.tw;
    if constexpr (TMA) {
        if (j == 0) mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    // TWK = 3: the thread's whole inter-pass table lives in registers for the kernel's lifetime
    // (two-pass plans: one twiddled pass per transform), so no block re-reads it from shared memory
    constexpr bool TWREG = TWK == 3;
    static_assert(!TWREG || (PL::P == 2 && PL::TW_PER_THREAD <= 32), "register-resident table: two-pass plans");
    using TWU = typename std::conditional<TWREG, TwRegs<C, PL::TW_PER_THREAD>,
                                          typename std::conditional<TWK == 4, TwCompact<C>, const C*>::type>::type;
    TWU twu;
    if constexpr (TWREG) {
#pragma unroll
        for (int k = 0; k < PL::TW_PER_THREAD; ++k) twu.r[k] = twsrc[k * T + j];
    } else if constexpr (TWK == 4) {
        twu.p = twsrc;
    } else {
        twu = twsrc;
    }
    // Programmatic dependent launch: everything above touches only read-only tables and shared
    // memory, so it overlaps the previous launch's tail; global x / y / schedule accesses start
    // after the previous grid has completed and flushed. The next launch may start its own
    // prologue as soon as this grid's CTAs leave the SMs.
    grid_dep_wait();
    grid_dep_launch_dependents();

    // Work item w = channel * nblk + (block - blk_begin), advanced by `stride`. The element
    // offsets of the item's segment in x / y and of its schedule entry are carried incrementally
    // (64-bit adds only; no per-item multiply or divide).
    // Each warp walks ONE contiguous run of work items (consecutive blocks of a channel), its
    // GPW = 32 / T groups taking consecutive items side by side: the (N - M)-sample halo of a
    // block is the tail of a segment the same warp fetched one step earlier (an L2 hit), and the
    // groups sharing a warp still load adjacent segments. (Grid-stride order had neighbouring
    // blocks fetched by different warps at the same moment: ncu c3 read 9.40 GB vs 8.59.)
    constexpr int GPW = T >= 32 ? 1 : 32 / T;
    static_assert(GROUPS % GPW == 0, "whole warps per CTA");
    const int stride = GPW;
    // Balanced contiguous split: CTA c takes total/grid (+1) consecutive items and its warps split
    // them q or q + 1 each, so every SM gets the same work to within one item even when there are
    // only a few items per warp (c2: 9.2), and the warps of one CTA still walk adjacent memory.
    // a.units (host, small launches): only that many warps per CTA take items, so that every round
    // of items is equally full (c1: 18.45 items per SM on 16 one-block groups = 2 rounds, run as
    // 10 + 9 instead of 16 + 3). Every warp runs exactly its own item count.
    const int upc_all = GROUPS / GPW;  // warps (or multi-warp groups) per CTA
    const int upc = (a.units > 0 && a.units < upc_all) ? a.units : upc_all;
    const int nct = int(gridDim.x), cid = int(blockIdx.x), ul = g / GPW;
    const int qc = a.total / nct, rc = a.total % nct;
    const int cbase = cid * qc + min(cid, rc);
    const int ccnt = qc + (cid < rc ? 1 : 0);
    const int qu = ccnt / upc, ru = ccnt % upc;
    const int wbase = cbase + ul * qu + min(ul, ru);
    int w = wbase + g % GPW;
    const int cnt_u = ul < upc ? qu + (ul < ru ? 1 : 0) : 0;
    const int w_end = wbase + cnt_u;
    const int iters = (cnt_u + GPW - 1) / GPW;
    int bl = w % a.nblk;
    const int ch0 = w / a.nblk;
    int ch = ch0;  // (virtual) channel of the current item
    const int dq = stride / a.nblk;
    const int dr = stride - dq * a.nblk;
    const int64_t Mi = a.M;
    constexpr int BF = IO == 2 ? 2 : 1;  // real blocks per work item
    const int64_t Ms = BF * Mi;           // segment stride between consecutive work items
    int64_t seg0 = (a.blk_begin + bl) * Ms - (N - Mi);  // global sample index of segment position 0
    int64_t xo = ch0 * a.x_cs - a.x_first + seg0;       // x element offset of position 0
    int64_t yo = ch0 * a.y_cs - a.y_first + seg0;       // y element offset of output time seg0
    int64_t bo = ch0 * a.b_cs + BF * (a.blk_begin + bl);  // schedule entry of this (first) block
    const int64_t dseg = dr * Ms, dseg_wrap = -int64_t(a.nblk) * Ms;
    const int64_t dx = dq * a.x_cs + dseg, dx_wrap = a.x_cs + dseg_wrap;
    const int64_t dy = dq * a.y_cs + dseg, dy_wrap = a.y_cs + dseg_wrap;
    const int64_t db = dq * a.b_cs + BF * dr, db_wrap = a.b_cs - BF * int64_t(a.nblk);
    // LEAN (complex and one-real-block I/O): only (w, bl, ch) are carried from item to item; the
    // 64-bit offsets are formed from them where they are used (a few integer multiply-adds per
    // block) instead of living in ~16 registers across both transforms together with their eight
    // 64-bit increments (the N = 1024 fp32 kernel, at its 168-register budget, no longer spills).
    // Measured (profiles/r02_sweep.md, "Lean loop state"): c3 +0.3 %, c4 +1 %, the other plans
    // -0.2 .. -2.6 % (N = 8192), so only the fp32 N = 1024 / 4096 plans use it (masks over log2 N).
#ifndef FCVBW_LEAN_F32
#define FCVBW_LEAN_F32 ((1 << 10) | (1 << 12))
#endif
#ifndef FCVBW_LEAN_F64
#define FCVBW_LEAN_F64 0
#endif
    constexpr bool LEAN = (((sizeof(R) == 4 ? (long long)(FCVBW_LEAN_F32) : (long long)(FCVBW_LEAN_F64)) >> ilog2(N)) & 1) &&
                          IO != 2;
    // BLATE (fp32 N = 1024): ncu of the register-starved kernel showed 5 % of all stall samples on
    // the forward transform's first butterfly, waiting to overwrite the address registers of the
    // schedule load issued just before it, and 4.6 % on a spill reload; with the load (and its
    // 64-bit address arithmetic) after the stores the kernel has no spills: c3 0.865 -> 0.891, c2
    // 0.695 -> 0.720. The other plans lose 0.4-1.7 % with it (profiles/r02_sweep.md).
#ifndef FCVBW_BLATE_F32
#define FCVBW_BLATE_F32 (1 << 10)
#endif
    constexpr bool BLATE = sizeof(R) == 4 && ((((long long)(FCVBW_BLATE_F32)) >> ilog2(N)) & 1) && IO != 2;
    auto seg_of = [&](int bl_) -> int64_t { return (a.blk_begin + bl_) * Ms - (N - Mi); };
    auto xo_of = [&](int ch_, int64_t sg) -> int64_t { return ch_ * a.x_cs - a.x_first + sg; };
    auto yo_of = [&](int ch_, int64_t sg) -> int64_t { return ch_ * a.y_cs - a.y_first + sg; };
    auto bo_of = [&](int ch_, int bl_) -> int64_t { return ch_ * a.b_cs + BF * (a.blk_begin + bl_); };

    // RPF (direct-load plans with few elements per thread: fp32 N = 64 / 128 / 256, fp64 N = 64): the
    // NEXT item's segment is loaded into a second register set while the current block computes.
    // Per-instruction stall samples of the direct-load kernels showed 39 % (fp32 N = 256) of all
    // samples on the first butterfly, waiting for the segment just requested. c5 fp32 64 / 128 /
    // 256: 0.74 / 0.80 / 0.835 -> 0.80 / 0.84 / 0.91; fp64 N = 64: 0.86 -> 0.92-0.95. Plans whose
    // second register set spills (fp32 N = 512, fp64 N >= 128) lose 25 % with it.
#ifndef FCVBW_RPF_F32
#define FCVBW_RPF_F32 ((1 << 6) | (1 << 7) | (1 << 8))
#endif
#ifndef FCVBW_RPF_F64
#define FCVBW_RPF_F64 (1 << 6)
#endif
    constexpr bool RPF = (((sizeof(R) == 4 ? (long long)(FCVBW_RPF_F32) : (long long)(FCVBW_RPF_F64)) >> ilog2(N)) & 1) &&
                         IO == 0 && TMA == 0 && !LEAN;
    C vn[RPF ? E : 1];
    auto load_seg = [&](C (&dst)[RPF ? E : 1], bool act, int64_t sg, int64_t xoff) {
        if constexpr (RPF) {
            if (act && sg >= 0 && sg + N <= a.S) {
                const C* src = a.x + xoff + j;
#pragma unroll
                for (int q = 0; q < E; ++q) dst[q] = src[T * q];
            } else {
                const C* xp = a.x + (xoff - sg);
#pragma unroll
                for (int q = 0; q < E; ++q) {
                    const int64_t i = sg + j + T * q;
                    dst[q] = (act && i >= 0 && i < a.S) ? xp[i] : czero(C{});
                }
            }
        }
    };
    if constexpr (RPF) load_seg(vn, w < w_end, seg0, xo);

    uint32_t phase = 0;
    bool staged = false;
    // IO = 2: the union of the pair's two real segments, [seg0, seg0 + M + N), in one bulk copy
    const uint32_t PAIR_BYTES = uint32_t(N + a.M) * uint32_t(sizeof(R));
    auto pair_stageable = [&](int64_t sg, int64_t xoff) {
        return sg >= 0 && sg + Mi + N <= a.S && (PAIR_BYTES & 15u) == 0 &&
               (reinterpret_cast<uintptr_t>(a.xr + xoff) & 15u) == 0;
    };
    // Bulk-copy issue and wait. The copy instruction takes warp-uniform operands, so when several
    // groups share a warp (T < 32) lane 0 issues every group's copy from shuffled arguments and the
    // whole warp waits on every group's barrier in uniform control flow (per-group issue from
    // divergent lanes serialised and left the warp diverged: 1.8x slower, profiles/r02_sweep.md).
    auto issue_copy = [&](bool st, const void* src, uint32_t bytes, bool fence) {
        if constexpr (GPW == 1) {
            if (st && j == 0) {
                if (fence) fence_proxy_async_smem();
                mbar_arrive_expect_tx(bar, bytes);
                bulk_g2s(stage, src, bytes, bar);
            }
        } else {
            const int lane = int(threadIdx.x) & 31;
            const int gw = g - g % GPW;  // first group of this warp (g % GPW == lane / T)
#pragma unroll
            for (int k = 0; k < GPW; ++k) {
                const int sk = __shfl_sync(0xffffffffu, int(st), k * T);
                const unsigned long long pk_ =
                    __shfl_sync(0xffffffffu, static_cast<unsigned long long>(reinterpret_cast<uintptr_t>(src)), k * T);
                if (lane == 0 && sk) {
                    C* dst = TMA == 1 ? stg + (gw + k) * N : xbuf + (gw + k) * padded<R, E>(N);
                    if (fence) fence_proxy_async_smem();
                    mbar_arrive_expect_tx(bars + gw + k, bytes);
                    bulk_g2s(dst, reinterpret_cast<const void*>(static_cast<uintptr_t>(pk_)), bytes, bars + gw + k);
                }
            }
        }
    };
    auto wait_copy = [&](bool st) {
        if constexpr (GPW == 1) {
            if (st) {
                mbar_wait(bar, phase);
                phase ^= 1u;
            }
        } else {
            const int gw = g - g % GPW;
#pragma unroll
            for (int k = 0; k < GPW; ++k) {
                const int sk = __shfl_sync(0xffffffffu, int(st), k * T);
                const uint32_t ph = __shfl_sync(0xffffffffu, phase, k * T);
                if (sk) mbar_wait(bars + gw + k, ph);
            }
            if (st) phase ^= 1u;
        }
    };
    if constexpr (TMA && IO == 0) {
        staged = w < w_end && bl >= a.tma_lo && bl <= a.tma_hi;
        issue_copy(staged, a.x + xo, SEG_BYTES, false);
    } else if constexpr (TMA && IO == 2) {
        staged = w < w_end && pair_stageable(seg0, xo);
        issue_copy(staged, a.xr + xo, PAIR_BYTES, false);
    }

    int b_nx = a.b_const;  // b of the next item (IO 0 / 1 / 3)
    if constexpr (MODE != COEF_RAW && IO != 2) {
        if (a.bsched && w < w_end) b_nx = __ldg(a.bsched + bo);
    }
    for (int it = 0; it < iters; ++it) {
        const bool active = (LEAN && GPW == 1) || w < w_end;
        if constexpr (LEAN) seg0 = seg_of(bl);
        const bool full = seg0 + N <= a.S;  // whole segment (and the block's output) inside the stream

        if constexpr (IO == 2) {
            // ---- real stream, block pair (2p, 2p + 1): one complex transform when both blocks use
            // the same b (exact: H is conjugate-symmetric), else two transforms with Im = 0
            const int64_t rb0 = BF * (a.blk_begin + bl);
            const bool has1 = rb0 + 1 < a.nblk_real;
            int b0v = a.b_const, b1v = a.b_const;
            if (a.bsched && active) {
                b0v = __ldg(a.bsched + bo);
                b1v = has1 ? __ldg(a.bsched + bo + 1) : b0v;
            }
            // Paired blocks with DIFFERENT b share the transform too (mixed): with Z = FFT(x0 + j x1)
            // and Zm(k) = conj(Z(N - k)),  Y = Z (H0 + H1)/2 + Zm (H0 - H1)/2  gives
            // IFFT(Y) = y0 + j y1 exactly, because both structured H are conjugate-symmetric
            // (engine.hpp:147-162); Zm comes through the exchange buffer (below).
            const bool pair = a.pair_real && has1;
            bool mixed = pair && b0v != b1v;
            if constexpr (T < 32) mixed = __any_sync(0xffffffffu, mixed);  // warp-uniform __syncwarp sequence
            const int nsub_own = (has1 && !pair) ? 2 : 1;
            // groups sharing a warp (T < 32) run the same number of transforms, so that their
            // __syncwarp() sequences match; a group with one real transform runs a dummy second
            int nsub = nsub_own;
            if constexpr (T < 32) nsub = __reduce_max_sync(0xffffffffu, nsub_own);
            const int64_t cur_seg0 = seg0, cur_xo = xo, cur_yo = yo;
            w += stride;
            bl += dr;
            seg0 += dseg;
            xo += dx;
            yo += dy;
            bo += db;
            ch += dq;
            if (bl >= a.nblk) {
                bl -= a.nblk;
                seg0 += dseg_wrap;
                xo += dx_wrap;
                yo += dy_wrap;
                bo += db_wrap;
                ++ch;
            }
            // the next pair's segments are bulk-copied into the exchange buffer once the last
            // transform of this item has read it for the last time
            auto prefetch_pair = [&]() {
                if constexpr (TMA) {
                    group_sync<T>(g);
                    staged = w < w_end && pair_stageable(seg0, xo);
                    issue_copy(staged, a.xr + xo, PAIR_BYTES, true);
                }
            };
            for (int sub = 0; sub < nsub; ++sub) {
                const bool act = active && sub < nsub_own;  // false: the dummy transform
                const int64_t sg = cur_seg0 + sub * Mi;  // segment start of this transform's Re block
                const bool im_on = pair;
                const R* x0 = a.xr + (cur_xo + sub * Mi) + j;
                const R* x1 = x0 + Mi;  // the next block's segment
                const bool full0 = sg + N <= a.S, full1 = !im_on || sg + Mi + N <= a.S;
                C v[E];
                if constexpr (TMA != 0) {
                    if (sub == 0) wait_copy(staged);
                }
                if (TMA && staged && sub == 0) {
                    // (an unpaired second transform reloads from global: its first exchange has
                    // overwritten the staged pair)
                    const R* s0 = reinterpret_cast<const R*>(stage) + j;
                    if (im_on) {
#pragma unroll
                        for (int q = 0; q < E; ++q) v[q] = cmake<C>(s0[T * q], s0[Mi + T * q]);
                    } else {
#pragma unroll
                        for (int q = 0; q < E; ++q) v[q] = cmake<C>(s0[T * q], R(0));
                    }
                } else if (act && sg >= 0 && full0 && full1) {
#pragma unroll
                    for (int q = 0; q < E; ++q) v[q] = cmake<C>(x0[T * q], im_on ? x1[T * q] : R(0));
                } else {
#pragma unroll
                    for (int q = 0; q < E; ++q) {
                        const int64_t i = sg + j + T * q;
                        const R re = (act && i >= 0 && i < a.S) ? x0[T * q] : R(0);
                        const R im = (act && im_on && i + Mi >= 0 && i + Mi < a.S) ? x1[T * q] : R(0);
                        v[q] = cmake<C>(re, im);
                    }
                }
                fft_q<R, N, E, false, TWF>(v, buf, twu, j, g);
                const bool last_sub = sub == nsub - 1;
                if (mixed) {
                    mixed_pair_multiply<R, N, E, MODE>(v, a, vs, j, b0v, b1v, buf, g);
                    fft_q<R, N, E, true, TWF>(v, buf, twu, j, g, [&]() {
                        if (last_sub) prefetch_pair();
                    });
                } else {
                    multiply_inverse<R, N, E, MODE, TWF>(v, a, vs, j, sub ? b1v : b0v, buf, twu, g, nullptr, [&]() {
                        if (last_sub) prefetch_pair();
                    });
                }
                if (act) {
                    R* y0 = a.yr + (cur_yo + sub * Mi);  // output time sg <-> y0[0]
                    R* y1 = y0 + Mi;
                    if constexpr (MODE == COEF_SHIFT_Q) {
                        // delay N/8, M = 3N/4: registers q in [E/8, 7E/8) hold the kept positions
                        // n = N/8 + j + T q (compile-time offsets from one base pointer)
                        R* yb0 = y0 + (N / 8 + j);
                        R* yb1 = yb0 + Mi;
                        const bool f1 = sg + Mi + N <= a.S;
                        if (full0 && im_on && f1) {
#pragma unroll
                            for (int q = E / 8; q < 7 * E / 8; ++q) {
                                yb0[T * q] = v[q].x;
                                yb1[T * q] = v[q].y;
                            }
                        } else if (full0 && !im_on) {
#pragma unroll
                            for (int q = E / 8; q < 7 * E / 8; ++q) yb0[T * q] = v[q].x;
                        } else {
                            const int64_t t0 = sg + N / 8 + j;
#pragma unroll
                            for (int q = E / 8; q < 7 * E / 8; ++q) {
                                if (t0 + T * q < a.S) yb0[T * q] = v[q].x;
                                if (im_on && t0 + T * q + Mi < a.S) yb1[T * q] = v[q].y;
                            }
                        }
                    } else {
                        const int sh = MODE == COEF_SHIFT ? a.shift : 0;
#pragma unroll
                        for (int q = 0; q < E; ++q) {
                            const int n = (j + T * q + sh) & (N - 1);
                            if (n >= N - a.M) {
                                const int64_t t = sg + n;
                                if (full0 || t < a.S) y0[n] = v[q].x;
                                if (im_on && (t + Mi < a.S)) y1[n] = v[q].y;
                            }
                        }
                    }
                }
            }
        } else {
            // ---- framing (engine.hpp:141-143): zero-primed history, zero-padded tail
            C v[E];
            if constexpr (TMA != 0) wait_copy(staged);
            if (TMA && staged) {
                const C* src = stage + j;
#pragma unroll
                for (int q = 0; q < E; ++q) v[q] = src[T * q];
            } else if constexpr (RPF) {
#pragma unroll
                for (int q = 0; q < E; ++q) v[q] = vn[q];
            } else if constexpr (IO == 0) {
                if constexpr (LEAN) xo = xo_of(ch, seg0);
                if (active && seg0 >= 0 && full) {
                    const C* src = a.x + xo + j;
#pragma unroll
                    for (int q = 0; q < E; ++q) v[q] = src[T * q];
                } else {
                    const C* xp = a.x + (xo - seg0);
#pragma unroll
                    for (int q = 0; q < E; ++q) {
                        const int64_t i = seg0 + j + T * q;
                        v[q] = (active && i >= 0 && i < a.S) ? xp[i] : czero(C{});
                    }
                }
            } else {
                // one real block, zero imaginary part
                if constexpr (LEAN) xo = xo_of(ch, seg0);
                const R* x0 = a.xr + xo + j;
                if (active && seg0 >= 0 && full) {
#pragma unroll
                    for (int q = 0; q < E; ++q) v[q] = cmake<C>(x0[T * q], R(0));
                } else {
#pragma unroll
                    for (int q = 0; q < E; ++q) {
                        const int64_t i = seg0 + j + T * q;
                        v[q] = (active && i >= 0 && i < a.S) ? cmake<C>(x0[T * q], R(0)) : czero(C{});
                    }
                }
            }
            const int b = b_nx;  // loaded one item ahead (its latency hides behind the previous block)
            int64_t cur_seg0 = seg0, cur_yo = yo;
            int cur_bl = bl, cur_ch = ch;
            if constexpr (LEAN) {
                // opaque copies: the store offsets are re-formed from them after the transforms
                // instead of being kept live (common-subexpression elimination would keep them)
                asm volatile("" : "+r"(cur_bl), "+r"(cur_ch));
            }

            // next work item; its segment is prefetched by TMA while this block computes
            w += stride;
            bl += dr;
            ch += dq;
            if constexpr (!LEAN) {
                seg0 += dseg;
                xo += dx;
                yo += dy;
                bo += db;
            }
            if (bl >= a.nblk) {
                bl -= a.nblk;
                ++ch;
                if constexpr (!LEAN) {
                    seg0 += dseg_wrap;
                    xo += dx_wrap;
                    yo += dy_wrap;
                    bo += db_wrap;
                }
            }
            // a next item exists (one group per warp: iters is the exact item count)
            const bool more = (LEAN && GPW == 1) ? it + 1 < iters : w < w_end;
            if constexpr (RPF) load_seg(vn, more, seg0, xo);  // next item's segment, in flight during this block
            auto prefetch_next = [&]() {
                group_sync<T>(g);  // every lane has consumed the buffer
                staged = more && bl >= a.tma_lo && bl <= a.tma_hi;
                issue_copy(staged, a.x + (LEAN ? xo_of(ch, seg_of(bl)) : xo), SEG_BYTES, true);
            };

            if constexpr (MODE != COEF_RAW && !BLATE) {
                if (a.bsched && more) b_nx = __ldg(a.bsched + (LEAN ? bo_of(ch, bl) : bo));
            }
            if constexpr (TMA == 1) prefetch_next();  // the staging buffer is free again

            // ---- forward DFT (fft.hpp:55-59 / 95-108)
            fft_q<R, N, E, false, TWF>(v, buf, twu, j, g);

            // ---- spectral multiply with on-the-fly coefficients (engine.hpp:147-165), then the
            // inverse DFT (fft.hpp:80-88), 1/N folded into the coefficients
            // parity dump of the mask this item applies (null in production: one uniform branch; the
            // row pointer is formed here, after the forward transform, so it is never live across it)
            R* const gd = (DUMP && active) ? a.gdump + int64_t(w - stride) * N : nullptr;
            if constexpr (TMA == 2)
                multiply_inverse<R, N, E, MODE, TWF>(v, a, vs, j, b, buf, twu, g, gd, prefetch_next);
            else
                multiply_inverse<R, N, E, MODE, TWF>(v, a, vs, j, b, buf, twu, g, gd);

            // ---- discard N - M and store (engine.hpp:171; flush truncation engine.hpp:113)
            if (active) {
                if constexpr (LEAN) {
                    cur_seg0 = seg_of(cur_bl);
                    cur_yo = yo_of(cur_ch, cur_seg0);
                }
                // base pointers + compile-time offsets (no per-store address arithmetic)
                auto store_at = [&](auto& yb0, int off, const C& val) {
                    if constexpr (IO == 0)
                        yb0[off] = val;
                    else
                        yb0[off] = val.x;  // real part only
                };
                using YP = typename std::conditional<IO == 0, C*, R*>::type;
                if constexpr (MODE == COEF_SHIFT_Q) {
                    // L - 1 = N/4: delay N/8 = T E/8, so only registers q in [E/8, 7E/8) land in the
                    // kept range [N - M, N); the others are never computed to completion (dead code)
                    YP yb0 = (IO == 0 ? (YP)(void*)a.y : (YP)(void*)a.yr) + (cur_yo + N / 8 + j);
                    if (full) {
#pragma unroll
                        for (int q = E / 8; q < 7 * E / 8; ++q) store_at(yb0, T * q, v[q]);
                    } else {
                        const int64_t t0 = cur_seg0 + N / 8 + j;
#pragma unroll
                        for (int q = E / 8; q < 7 * E / 8; ++q)
                            if (t0 + T * q < a.S) store_at(yb0, T * q, v[q]);
                    }
                } else {
                    YP yp0 = (IO == 0 ? (YP)(void*)a.y : (YP)(void*)a.yr) + (cur_yo - cur_seg0);
                    const int sh = (MODE == COEF_SHIFT) ? a.shift : 0;
#pragma unroll
                    for (int q = 0; q < E; ++q) {
                        const int n = (j + T * q + sh) & (N - 1);
                        const int64_t t = cur_seg0 + n;
                        if (n >= N - a.M && (full || t < a.S)) {
                            YP p0 = yp0 + t;
                            store_at(p0, 0, v[q]);
                        }
                    }
                }
            }
            // BLATE: the next item's schedule entry is requested here, after the stores, where the
            // transform's registers are free, instead of before the forward transform
            if constexpr (MODE != COEF_RAW && BLATE) {
                if (a.bsched && more) b_nx = __ldg(a.bsched + (LEAN ? bo_of(ch, bl) : bo));
            }
            }
    }
}

// Parity dump of the per-(block, bin) coefficients: same region rule as the fused kernel, the
// magnitude placed as magnitude_samples does (spectrum.hpp:170-187) and H = magnitude * phase in
// the order of assemble_dft_coefficients (spectrum.hpp:234), all in fp64.
static __global__ void coeff_dump_kernel(int N, const int* __restrict__ b, int n_b, int half_dn,
                                  const double* __restrict__ V, const double2* __restrict__ phase,
                                  int8_t* region, int16_t* vidx, double2* H) {
    const int64_t total = int64_t(n_b) * N;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int bi = int(e / N), k = int(e % N);
        const int k1 = b[bi] - half_dn + 1;
        const int span = 2 * half_dn - 2;
        const int f = k < N - k ? k : N - k;
        const int reg = bin_region_of(f, k1, span);
        if (region) region[e] = int8_t(reg);
        if (vidx) vidx[e] = int16_t(reg == 1 ? f - k1 : -1);
        if (H) {
            const double mag = reg == 0 ? 1.0 : (reg == 1 ? V[f - k1] : 0.0);
            const double2 ph = phase[k];
            H[e] = make_double2(mag * ph.x, mag * ph.y);
        }
    }
}

}  // namespace fcvbw_gpu
