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
// there is no bit reversal anywhere. Groups are persistent: each loops over (channel, block)
// work items in grid-stride order, so resident groups always work on a contiguous window of
// blocks and the (N-M)-sample halo re-read of the next block is served by L2.
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

#include "cplx.cuh"
#include "dft.cuh"

namespace fcvbw_gpu {

enum CoefMode : int { COEF_SHIFT = 0, COEF_PHASE = 1, COEF_RAW = 2 };

template <class R>
struct OlsArgs {
    const cx_t<R>* x;  // x[ch * x_cs + (i - x_first)] holds input sample i of channel ch
    cx_t<R>* y;        // y[ch * y_cs + (i - y_first)] receives output sample i
    int64_t x_first, y_first, x_cs, y_cs;
    int64_t S;                    // samples per channel (global stream length)
    int64_t blk_begin, nblk;      // global block range [blk_begin, blk_begin + nblk)
    int64_t total;                // channels * nblk work items
    const int* bsched;            // b per (channel, global block), or null -> b_const
    int64_t b_cs;                 // channel stride of bsched (0: one schedule for all channels)
    int b_const;
    int M, half_dn, LV, shift;    // shift = (L-1)/2 for COEF_SHIFT
    const R* V;                   // LV profile values, pre-scaled by 1/N
    const cx_t<R>* coef;          // COEF_PHASE: phase table; COEF_RAW: table / N
    const cx_t<R>* tw;            // per-thread twiddle table (plan_twiddles layout)
    R inv_n;
};

// ------------------------------------------------------------------ radix plan
__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n / 2); }

template <int N, int E>
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
    // twiddle entries (per thread) before pass p: sum over earlier passes q >= 1 of (E/r_q)(r_q - 1)
    __host__ __device__ static constexpr int tw_off(int p) {
        return p <= 1 ? 0 : tw_off(p - 1) + (E / radix(p - 1)) * (radix(p - 1) - 1);
    }
    static constexpr int TW_PER_THREAD = tw_off(P);
};

// Shared-memory padding: one element per 32 (fp32) / 16 (fp64) keeps both the strided Stockham
// writes and the q-layout reads at the minimum wavefront count.
template <class R>
__device__ __forceinline__ int padi(int a) {
    return a + (a >> (sizeof(R) == 4 ? 5 : 4));
}
template <class R>
__host__ __device__ constexpr int padded(int n) {
    return n + (n >> (sizeof(R) == 4 ? 5 : 4));
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

// ------------------------------------------------------------------ Stockham passes
template <class R, int N, int E, bool INV, int p>
struct Pass {
    using C = cx_t<R>;
    using PL = Plan<N, E>;
    static constexpr int T = PL::T;

    // pass p-1 results (registers, q-layout) -> shared memory in Stockham output order
    __device__ __forceinline__ static void write_prev(C (&v)[E], C* buf, int j) {
        constexpr int r = PL::radix(p - 1);
        constexpr int ns = PL::ns(p - 1);
#pragma unroll
        for (int m = 0; m < E / r; ++m) {
            const int jp = j + m * T;
            const int idxd = (jp / ns) * ns * r + (jp % ns);
#pragma unroll
            for (int i = 0; i < r; ++i) buf[padi<R>(idxd + i * ns)] = v[m + i * (E / r)];
        }
    }

    __device__ __forceinline__ static void run(C (&v)[E], C* buf, const C* __restrict__ tw, int j, int g) {
        if constexpr (p < PL::P) {
            constexpr int r = PL::radix(p);
            group_sync<T>(g);  // previous readers of buf are done
            write_prev(v, buf, j);
            group_sync<T>(g);
#pragma unroll
            for (int q = 0; q < E; ++q) v[q] = buf[padi<R>(j + T * q)];
            // twiddles W_{ns r}^{i k}, k = (j + mT) mod ns, from the per-thread table
            const C* twp = tw + PL::tw_off(p) * T + j;
#pragma unroll
            for (int m = 0; m < E / r; ++m) {
                C t[r];
                t[0] = v[m];
#pragma unroll
                for (int i = 1; i < r; ++i) {
                    const C w = __ldg(twp + (m * (r - 1) + (i - 1)) * T);
                    t[i] = INV ? cmulc(v[m + i * (E / r)], w) : cmul(v[m + i * (E / r)], w);
                }
                dft<r, INV>(t);
#pragma unroll
                for (int i = 0; i < r; ++i) v[m + i * (E / r)] = t[i];
            }
            Pass<R, N, E, INV, p + 1>::run(v, buf, tw, j, g);
        }
    }
};

template <class R, int N, int E, bool INV>
__device__ __forceinline__ void fft_q(cx_t<R> (&v)[E], cx_t<R>* buf, const cx_t<R>* __restrict__ tw, int j,
                                      int g) {
    dft<E, INV>(v);  // pass 0: ns = 1, no twiddles
    Pass<R, N, E, INV, 1>::run(v, buf, tw, j, g);
}

// ------------------------------------------------------------------ the fused kernel
template <class R, int N, int E, int MODE, int GROUPS>
__global__ void __launch_bounds__(GROUPS * Plan<N, E>::T) ols_fused(OlsArgs<R> a) {
    using C = cx_t<R>;
    using PL = Plan<N, E>;
    constexpr int T = PL::T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* xbuf = reinterpret_cast<C*>(smem_raw);
    R* vs = reinterpret_cast<R*>(smem_raw + sizeof(C) * GROUPS * padded<R>(N));

    const int tid = threadIdx.x;
    const int g = tid / T;
    const int j = tid - g * T;
    C* buf = xbuf + g * padded<R>(N);

    if constexpr (MODE != COEF_RAW) {
        for (int i = tid; i < a.LV; i += GROUPS * T) vs[i] = a.V[i];
        __syncthreads();
    }

    for (int64_t base = int64_t(blockIdx.x) * GROUPS; base < a.total; base += int64_t(gridDim.x) * GROUPS) {
        const int64_t w = base + g;
        const bool active = w < a.total;
        const int64_t ch = active ? w / a.nblk : 0;
        const int64_t blk = a.blk_begin + (active ? w - ch * a.nblk : 0);
        const int64_t seg0 = blk * a.M - (N - a.M);  // global index of segment position 0
        const C* xp = a.x + ch * a.x_cs - a.x_first;

        // ---- framing (engine.hpp:141-143): zero-primed history, zero-padded tail
        C v[E];
        if (active && seg0 >= 0 && seg0 + N <= a.S) {
            const C* src = xp + seg0 + j;
#pragma unroll
            for (int q = 0; q < E; ++q) v[q] = src[T * q];
        } else {
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int64_t i = seg0 + j + T * q;
                v[q] = (active && i >= 0 && i < a.S) ? xp[i] : czero(C{});
            }
        }

        // ---- forward DFT (fft.hpp:55-59 / 95-108)
        fft_q<R, N, E, false>(v, buf, a.tw, j, g);

        // ---- spectral multiply (engine.hpp:147-165)
        if constexpr (MODE == COEF_RAW) {
#pragma unroll
            for (int q = 0; q < E; ++q) v[q] = cmul(v[q], __ldg(a.coef + j + T * q));
        } else {
            const int b = a.bsched ? __ldg(a.bsched + ch * a.b_cs + blk) : a.b_const;
            const int k1 = b - a.half_dn + 1;
            const int span = 2 * a.half_dn - 2;  // k2 - k1
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int f = (q < E / 2) ? (j + T * q) : (N - j - T * q);  // min(k, N - k)
                const int region = bin_region_of(f, k1, span);
                R gk = region == 0 ? a.inv_n : R(0);
                if (region == 1) gk = vs[f - k1];
                v[q] = cscale(v[q], gk);
                if constexpr (MODE == COEF_PHASE) v[q] = cmul(v[q], __ldg(a.coef + j + T * q));
            }
        }

        // ---- inverse DFT (fft.hpp:80-88), 1/N already folded in
        fft_q<R, N, E, true>(v, buf, a.tw, j, g);

        // ---- discard N - M and store (engine.hpp:171; flush truncation engine.hpp:113)
        if (active) {
            C* yp = a.y + ch * a.y_cs - a.y_first;
            const int64_t out0 = blk * a.M - (N - a.M);  // output time of position 0
            const int sh = (MODE == COEF_SHIFT) ? a.shift : 0;
            const bool full = (blk + 1) * a.M <= a.S;
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int n = (j + T * q + sh) & (N - 1);
                const int64_t t = out0 + n;
                if (n >= N - a.M && (full || t < a.S)) yp[t] = v[q];
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
