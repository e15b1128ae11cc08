// Design-side verification on the GPU: the dense-grid worst-case
// error of a design over every band centre b, output phase n and grid frequency omega — the
// reference's `verify()` (proj/include/fcvbw/design.hpp:601-673), whose inner loop is the
// O(num_b * K * M * N) sum `response_from_row` (proj/include/fcvbw/ptvir.hpp:355-361).
//
// Algebraic restructuring (exact in real arithmetic): every PTVIR row is a circular shift of one
// base row, d_n(q) = base((q + s_n) mod N) with s_n = (step (n - (M - 1))) mod N
// (ptvir_from_base, ptvir.hpp:147-160). With F = sum_p base(p) e^{-j w p} and the prefix sums
// P_s = sum_{p < s} base(p) e^{-j w p},
//     sum_q d_n(q) e^{-j w q} = e^{j w s} (F - P_s) + e^{j w (s - N)} P_s,
// so all M rows at one omega cost one length-N prefix sum plus O(1) per row:
// O(num_b * K * (N + M)) instead of O(num_b * K * M * N). Everything is fp64.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fcvbw_gpu.h"
#include "grid.h"

namespace verify_impl {

using fcvbw_grid::build_grid;
using fcvbw_grid::Grid;
using fcvbw_grid::kPi;

// base_response_idft (ptvir.hpp:100-115) of assemble_dft_coefficients(bins, V, b)
// (spectrum.hpp:221-242) for every b: base[b][q] = Re(sum_k mag(k) phase(k) root(q k)) / N.
__global__ void base_kernel(int N, int dn, int blo, int num_b, const double* __restrict__ V,
                            const double2* __restrict__ phase, const double2* __restrict__ roots, double* base,
                            int* bad) {
    const int bi = blockIdx.y;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (bi >= num_b || q >= N) return;
    const int b = blo + bi;
    const int k1 = b - dn / 2 + 1, k2 = b + dn / 2 - 1;
    double re = 0.0, im = 0.0;
    for (int k = 0; k < N; ++k) {
        const int f = k < N - k ? k : N - k;
        const double mag = f < k1 ? 1.0 : (f <= k2 ? V[f - k1] : 0.0);
        const double2 h = make_double2(mag * phase[k].x, mag * phase[k].y);
        const double2 r = roots[int((int64_t(q) * k) % N)];
        re += h.x * r.x - h.y * r.y;
        im += h.x * r.y + h.y * r.x;
    }
    if (fabs(im) > 1e-12 * N) atomicExch(bad, 1);
    base[size_t(bi) * N + q] = re / N;
}

// fill_phasors (ptvir.hpp:346-352): ph[g][p] = e^{-j omega_g p}, p in [0, N] (one extra entry).
__global__ void phasor_kernel(int N, int kb, const double* __restrict__ omega, double2* ph) {
    const int64_t total = int64_t(kb) * (N + 1);
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t gi = e / (N + 1);
        const int p = int(e - gi * (N + 1));
        double s, c;
        sincos(-omega[gi] * double(p), &s, &c);
        ph[e] = make_double2(c, s);
    }
}

__device__ __forceinline__ double2 cm(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cj(double2 a) { return make_double2(a.x, -a.y); }

__device__ __forceinline__ void amax(unsigned long long* p, double v) {  // v >= 0: bit order = value order
    atomicMax(p, static_cast<unsigned long long>(__double_as_longlong(v)));
}

struct SweepArgs {
    int N, M, L, dn, blo, num_b, step, kb, g0;  // kb omegas of this batch starting at global index g0
    int64_t kk;                                // total grid size K'
    const double* base;                        // [num_b][N]
    const double2* ph;                         // [kb][N + 1]
    const double* omega;                       // [K'] (global)
    const int8_t* region;                      // [num_b][K']
    unsigned long long* per_bn;                // [num_b][M] max |E| (double bits)
    unsigned long long* pass_stop;             // [2]
    // optional argmax pass for one b: smallest (gi, n) whose error equals target
    int arg_b;
    unsigned long long target;
    unsigned long long* arg_out;  // min over (gi * M + n)
};

// One CTA per (b, omega chunk); one warp per omega at a time. Lanes own contiguous runs of p;
// a warp scan turns run sums into prefix sums, then each lane walks its run evaluating the rows
// whose shift s_n falls in it.
template <bool ARG>
__global__ void __launch_bounds__(256) sweep_kernel(SweepArgs a) {
    extern __shared__ unsigned long long rowmax[];  // [M]
    const int bi = ARG ? a.arg_b : blockIdx.x;  // b fastest: co-resident CTAs share one omega chunk in L2
    const int b = a.blo + bi;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    if (!ARG)
        for (int n = threadIdx.x; n < a.M; n += blockDim.x) rowmax[n] = 0ull;
    __syncthreads();
    const int N = a.N, M = a.M;
    const int run = (N + 31) / 32;
    const int p0 = min(N, lane * run), p1 = min(N, p0 + run);
    const double* base = a.base + size_t(bi) * N;
    const double b_omega = b * 2.0 * kPi / N;
    const double delta = a.dn * 2.0 * kPi / N;
    const double gd = (a.L - 1) / 2.0 + (M - 1);
    double pass_max = 0.0, stop_max = 0.0;
    const int chunk = (a.kb + gridDim.y - 1) / gridDim.y;
    const int c0 = ARG ? 0 : blockIdx.y * chunk, c1 = ARG ? a.kb : min(a.kb, c0 + chunk);
    for (int lg = c0 + (ARG ? blockIdx.x * nwarps + warp : warp); lg < c1; lg += ARG ? gridDim.x * nwarps : nwarps) {
        const int64_t gi = a.g0 + lg;
        const int reg = a.region[size_t(bi) * a.kk + gi];
        if (reg == 2) continue;
        const double omega = a.omega[gi];
        const double2* ph = a.ph + size_t(lg) * (N + 1);
        // desired_response (ptvir.hpp:368-381)
        double2 desired = make_double2(0.0, 0.0);
        if (omega <= b_omega - delta / 2.0 + 1e-12) {
            double s, c;
            sincos(-omega * gd, &s, &c);
            desired = make_double2(c, s);
        }
        // run sum -> exclusive warp scan -> prefix at the run start; F = total
        double2 acc = make_double2(0.0, 0.0);
        for (int p = p0; p < p1; ++p) {
            const double2 t = ph[p];
            acc.x += base[p] * t.x;
            acc.y += base[p] * t.y;
        }
        double2 incl = acc;
        for (int o = 1; o < 32; o <<= 1) {
            const double ux = __shfl_up_sync(0xffffffffu, incl.x, o), uy = __shfl_up_sync(0xffffffffu, incl.y, o);
            if (lane >= o) {
                incl.x += ux;
                incl.y += uy;
            }
        }
        const double2 F = make_double2(__shfl_sync(0xffffffffu, incl.x, 31), __shfl_sync(0xffffffffu, incl.y, 31));
        double2 P = make_double2(incl.x - acc.x, incl.y - acc.y);
        const double2 phN = ph[N];
        for (int s = p0; s < p1; ++s) {
            // the row whose shift is s: s = (step (n - (M - 1))) mod N
            const int n = (a.step > 0 ? s + M - 1 : M - 1 - s) & (N - 1);  // N is a power of two
            if (n < M) {
                const double2 es = cj(ph[s]);        // e^{+j w s}
                const double2 esn = cm(es, phN);     // e^{+j w (s - N)}
                const double2 FmP = make_double2(F.x - P.x, F.y - P.y);
                const double2 sum = make_double2(es.x * FmP.x - es.y * FmP.y + esn.x * P.x - esn.y * P.y,
                                                 es.x * FmP.y + es.y * FmP.x + esn.x * P.y + esn.y * P.x);
                const double2 hn = cm(ph[n], sum);   // prefactor e^{-j w n}
                const double err = hypot(hn.x - desired.x, hn.y - desired.y);
                if (ARG) {
                    if (static_cast<unsigned long long>(__double_as_longlong(err)) == a.target)
                        atomicMin(a.arg_out, static_cast<unsigned long long>(gi * M + n));
                } else {
                    amax(&rowmax[n], err);
                    if (reg == 0)
                        pass_max = fmax(pass_max, err);
                    else
                        stop_max = fmax(stop_max, err);
                }
            }
            P.x += base[s] * ph[s].x;
            P.y += base[s] * ph[s].y;
        }
    }
    if (ARG) return;
    amax(&a.pass_stop[0], pass_max);
    amax(&a.pass_stop[1], stop_max);
    __syncthreads();
    for (int n = threadIdx.x; n < M; n += blockDim.x) atomicMax(&a.per_bn[size_t(bi) * M + n], rowmax[n]);
}

struct Failure {
    int code;
    std::string msg;
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Failure{FCVBW_GPU_ERROR, std::string(what) + ": " + cudaGetErrorString(e)};
}

template <class T>
struct Dev {
    T* p = nullptr;
    explicit Dev(size_t n) { ck(cudaMalloc(&p, sizeof(T) * std::max<size_t>(1, n)), "cudaMalloc"); }
    ~Dev() { cudaFree(p); }
};

}  // namespace verify_impl

namespace fcvbw_gpu_detail {
void set_last_error(const std::string& m);
}

using namespace verify_impl;

extern "C" int fcvbw_gpu_verify(const fcvbw_gpu_design* d, int dense_points, double delta_e, int window_offset,
                                int step, int device, double* per_b_max, double* per_n_max,
                                fcvbw_gpu_verification* report) {
    try {
        if (!d || !report) throw Failure{FCVBW_GPU_VALIDATION, "verify: null argument"};
        const int N = d->fft_length, L = d->filter_length, M = d->block_length, dn = d->transition_width_bins;
        const int blo = d->b_low, bhi = d->b_high, num_b = bhi - blo + 1;
        // BinSpec::validate (spectrum.hpp:63-76) and verify's preconditions (design.hpp:603-604)
        if (N < 8 || (N & (N - 1)) || L < 1 || L > N || M != N - L + 1 || dn < 2 || dn % 2 ||
            !(dn / 2 <= blo && blo <= bhi && bhi <= N / 2 - dn / 2 - 1))
            throw Failure{FCVBW_GPU_VALIDATION, "BinSpec: invalid geometry"};
        if (d->profile_length != dn - 1 || !d->profile)
            throw Failure{FCVBW_GPU_VALIDATION, "verify: profile length must be delta_N - 1"};
        if (dense_points < 4 * d->grid_points)
            throw Failure{FCVBW_GPU_VALIDATION, "verify: dense grid must have at least 4x the design points"};
        if (dense_points < 2 * N) throw Failure{FCVBW_GPU_VALIDATION, "FrequencyGrid: need K >= 2N grid points"};
        if (step != 1 && step != -1) throw Failure{FCVBW_GPU_VALIDATION, "verify: shift step must be +-1"};
        if (window_offset != 1 - M)
            throw Failure{FCVBW_GPU_VALIDATION, "verify: only the overlap-save window offset 1 - M is supported"};
        ck(cudaSetDevice(device), "cudaSetDevice");

        Grid grid = build_grid(N, dn, blo, bhi, dense_points);
        const int64_t kk = int64_t(grid.omega.size());
        // tables: phase_table (spectrum.hpp:208-219) and unit roots (ptvir.hpp:70-77), host fp64
        std::vector<double2> phase(N), roots(N);
        const int64_t order = L - 1;
        for (int k = 0; k <= N / 2; ++k) {
            const int64_t folded = (int64_t(k) * order) % (2 * int64_t(N));
            const double ang = -kPi * static_cast<double>(folded) / N;
            phase[k] = make_double2(std::cos(ang), std::sin(ang));
        }
        for (int k = N / 2 + 1; k < N; ++k) phase[k] = make_double2(phase[N - k].x, -phase[N - k].y);
        for (int m = 0; m < N; ++m) {
            const double ang = 2.0 * kPi * m / N;
            roots[m] = make_double2(std::cos(ang), std::sin(ang));
        }
        Dev<double> dV(dn - 1), dbase(size_t(num_b) * N), domega(kk);
        Dev<double2> dphase(N), droots(N);
        Dev<int8_t> dregion(size_t(num_b) * kk);
        Dev<int> dbad(1);
        Dev<unsigned long long> dper(size_t(num_b) * M), dps(2), darg(1);
        ck(cudaMemcpy(dV.p, d->profile, sizeof(double) * (dn - 1), cudaMemcpyHostToDevice), "H2D V");
        ck(cudaMemcpy(dphase.p, phase.data(), sizeof(double2) * N, cudaMemcpyHostToDevice), "H2D phase");
        ck(cudaMemcpy(droots.p, roots.data(), sizeof(double2) * N, cudaMemcpyHostToDevice), "H2D roots");
        ck(cudaMemcpy(domega.p, grid.omega.data(), sizeof(double) * kk, cudaMemcpyHostToDevice), "H2D omega");
        ck(cudaMemcpy(dregion.p, grid.region.data(), size_t(num_b) * kk, cudaMemcpyHostToDevice), "H2D region");
        ck(cudaMemset(dbad.p, 0, sizeof(int)), "memset");
        ck(cudaMemset(dper.p, 0, sizeof(unsigned long long) * size_t(num_b) * M), "memset");
        ck(cudaMemset(dps.p, 0, 2 * sizeof(unsigned long long)), "memset");

        base_kernel<<<dim3((N + 127) / 128, num_b), 128>>>(N, dn, blo, num_b, dV.p, dphase.p, droots.p, dbase.p,
                                                           dbad.p);
        ck(cudaGetLastError(), "base kernel");
        int bad = 0;
        ck(cudaMemcpy(&bad, dbad.p, sizeof(int), cudaMemcpyDeviceToHost), "D2H bad");
        if (bad) throw Failure{FCVBW_GPU_VALIDATION, "base_response_idft: table is not conjugate-symmetric"};

        // omega batches so that the phasor table stays below ~2 GiB
        const int64_t per_omega = int64_t(N + 1) * int64_t(sizeof(double2));
        const int kb_max = int(std::max<int64_t>(1, std::min<int64_t>(kk, (int64_t(2) << 30) / per_omega)));
        Dev<double2> dph(size_t(kb_max) * (N + 1));
        const size_t smem = sizeof(unsigned long long) * M;
        if (smem > 48 * 1024)
            ck(cudaFuncSetAttribute(sweep_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)),
               "smem attr");
        SweepArgs sa{};
        sa.N = N;
        sa.M = M;
        sa.L = L;
        sa.dn = dn;
        sa.blo = blo;
        sa.num_b = num_b;
        sa.step = step;
        sa.kk = kk;
        sa.base = dbase.p;
        sa.ph = dph.p;
        sa.omega = domega.p;
        sa.region = dregion.p;
        sa.per_bn = dper.p;
        sa.pass_stop = dps.p;
        for (int64_t g0 = 0; g0 < kk; g0 += kb_max) {
            const int kb = int(std::min<int64_t>(kb_max, kk - g0));
            phasor_kernel<<<592, 256>>>(N, kb, domega.p + g0, dph.p);
            ck(cudaGetLastError(), "phasor kernel");
            sa.kb = kb;
            sa.g0 = int(g0);
            // omega chunks: each chunk's phasor slab (<= 16 MiB) stays L2-resident while the num_b CTAs
            // of that chunk run; enough chunks to fill 148 SMs x 8 CTAs; >= 8 omegas (one per warp)
            const int64_t slab = int64_t(16) << 20;
            int64_t chunks = std::max<int64_t>((int64_t(kb) * per_omega + slab - 1) / slab, (148 * 8 + num_b - 1) / num_b);
            chunks = std::max<int64_t>(1, std::min<int64_t>({chunks, kb / 8, 65535}));
            sweep_kernel<false><<<dim3(num_b, chunks), 256, smem>>>(sa);
            ck(cudaGetLastError(), "sweep kernel");
        }
        ck(cudaDeviceSynchronize(), "sweep sync");

        std::vector<unsigned long long> per(size_t(num_b) * M);
        unsigned long long ps[2];
        ck(cudaMemcpy(per.data(), dper.p, sizeof(unsigned long long) * per.size(), cudaMemcpyDeviceToHost), "D2H");
        ck(cudaMemcpy(ps, dps.p, sizeof(ps), cudaMemcpyDeviceToHost), "D2H");
        auto as_d = [](unsigned long long u) {
            double v;
            std::memcpy(&v, &u, sizeof v);
            return v;
        };
        std::memset(report, 0, sizeof(*report));
        report->dense_points = dense_points;
        report->worst_b = -1;
        report->worst_n = -1;
        std::vector<double> pn(size_t(M), 0.0);
        unsigned long long best = 0;
        for (int bi = 0; bi < num_b; ++bi) {
            unsigned long long mb = 0;
            for (int n = 0; n < M; ++n) {
                const unsigned long long u = per[size_t(bi) * M + n];
                mb = std::max(mb, u);
                pn[n] = std::max(pn[n], as_d(u));
            }
            if (per_b_max) per_b_max[bi] = as_d(mb);
            if (as_d(mb) > report->delta) {  // first strictly larger b wins, as in design.hpp:654-659
                report->delta = as_d(mb);
                report->worst_b = blo + bi;
                best = mb;
            }
        }
        if (per_n_max) std::memcpy(per_n_max, pn.data(), sizeof(double) * M);
        report->passband_max = as_d(ps[0]);
        report->stopband_max = as_d(ps[1]);
        if (report->worst_b >= 0) {
            // argmax pass for the worst b: the first (omega, n) in the reference's loop order
            const unsigned long long init = ~0ull;
            ck(cudaMemcpy(darg.p, &init, sizeof(init), cudaMemcpyHostToDevice), "H2D arg");
            sa.arg_b = report->worst_b - blo;
            sa.target = best;
            sa.arg_out = darg.p;
            for (int64_t g0 = 0; g0 < kk; g0 += kb_max) {
                const int kb = int(std::min<int64_t>(kb_max, kk - g0));
                phasor_kernel<<<592, 256>>>(N, kb, domega.p + g0, dph.p);
                sa.kb = kb;
                sa.g0 = int(g0);
                sweep_kernel<true><<<64, 256>>>(sa);
                ck(cudaGetLastError(), "argmax kernel");
            }
            unsigned long long arg = 0;
            ck(cudaMemcpy(&arg, darg.p, sizeof(arg), cudaMemcpyDeviceToHost), "D2H arg");
            if (arg != init) {
                report->worst_n = int(arg % M);
                report->worst_omega = grid.omega[size_t(arg / M)];
            }
        }
        report->pass = report->delta <= delta_e;
        report->refinement_bound = d->delta / std::cos(kPi / d->facets) + 1e-9;
        report->within_bound = report->delta <= report->refinement_bound;
        fcvbw_gpu_detail::set_last_error("");
        return FCVBW_GPU_OK;
    } catch (const Failure& f) {
        fcvbw_gpu_detail::set_last_error(f.msg);
        return f.code;
    } catch (const std::exception& e) {
        fcvbw_gpu_detail::set_last_error(e.what());
        return FCVBW_GPU_ERROR;
    }
}
