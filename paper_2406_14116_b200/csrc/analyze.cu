// Design analysis on the GPU: the quantities behind the reference's
// `fcvbw analyze` tables (proj/tools/fcvbw_cli.cpp:120-193) and `error_on_grid`
// (proj/include/fcvbw/ptvir.hpp:402-431): for every requested band centre b and grid frequency
// omega, the response H_n(omega) of all M output phases, reduced to max |H_n|, min |H_n| and
// max |E_n| (masked points only), optionally kept per phase; plus the PTVIR table of one b.
//
// Every H_n is evaluated exactly as the reference does (response.cuh: same operation order, no
// FMA, host-libm phasors, glibc's hypot algorithm), so |H_n| and |E_n| are bit-identical to the
// reference's and the CSV tables byte-identical (tests/test_cli_design.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "../../include/fcvbw_gpu.h"
#include "grid.h"
#include "response.cuh"

namespace fcvbw_gpu_detail {
void set_last_error(const std::string& m);
}

namespace analyze_impl {

using namespace fcvbw_grid;
using namespace fcvbw_resp;

struct Failure {
    int code;
    std::string msg;
};
[[noreturn]] void validation(const std::string& m) { throw Failure{FCVBW_GPU_VALIDATION, m}; }
void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Failure{FCVBW_GPU_ERROR, std::string(what) + ": " + cudaGetErrorString(e)};
}

template <class T>
struct Dev {
    T* p = nullptr;
    explicit Dev(size_t n) { ck(cudaMalloc(&p, sizeof(T) * std::max<size_t>(1, n)), "cudaMalloc"); }
    Dev(const Dev&) = delete;
    ~Dev() { cudaFree(p); }
    void put(const T* h, size_t n) { ck(cudaMemcpy(p, h, sizeof(T) * n, cudaMemcpyHostToDevice), "H2D"); }
    void get(T* h, size_t n) const { ck(cudaMemcpy(h, p, sizeof(T) * n, cudaMemcpyDeviceToHost), "D2H"); }
};

struct Geometry {
    int N, L, M, dn, blo, bhi;
    std::vector<double> v;
};

Geometry check(const fcvbw_gpu_design* d) {
    if (!d) validation("analyze: null design");
    Geometry g{d->fft_length, d->filter_length, d->block_length, d->transition_width_bins, d->b_low, d->b_high, {}};
    // BinSpec::validate (spectrum.hpp:63-76) and the profile-length check
    if (g.N < 8 || (g.N & (g.N - 1))) validation("BinSpec: N must be 2^Q with Q >= 3");
    if (g.L < 1 || g.L > g.N || g.M != g.N - g.L + 1 || g.dn < 2 || g.dn % 2 ||
        !(g.dn / 2 <= g.blo && g.blo <= g.bhi && g.bhi <= g.N / 2 - g.dn / 2 - 1))
        validation("BinSpec: invalid geometry");
    if (!d->profile || d->profile_length != g.dn - 1) validation("analyze: profile length must be delta_N - 1");
    g.v.assign(d->profile, d->profile + g.dn - 1);
    return g;
}

// Base rows (base_response_idft of assemble_dft_coefficients) of the given band centres, on the device.
void base_rows(const Geometry& g, const std::vector<int>& bs, double* d_base) {
    const int N = g.N;
    const auto phase = phase_table(N, g.L);
    const auto roots = unit_roots(N);
    std::vector<cd> tabs(bs.size() * size_t(N));
    for (size_t i = 0; i < bs.size(); ++i) assemble_table(N, g.dn, bs[i], g.v.data(), phase, tabs.data() + i * N);
    Dev<double2> dt(tabs.size()), dr(static_cast<size_t>(N));
    dt.put(reinterpret_cast<const double2*>(tabs.data()), tabs.size());
    dr.put(reinterpret_cast<const double2*>(roots.data()), size_t(N));
    Dev<int> bad(1);
    ck(cudaMemset(bad.p, 0, sizeof(int)), "memset");
    base_rows_kernel<<<dim3((N + 127) / 128, unsigned(bs.size())), 128>>>(N, int(bs.size()), dt.p, dr.p, d_base, bad.p);
    ck(cudaGetLastError(), "base_rows_kernel");
    int flag = 0;
    bad.get(&flag, 1);
    if (flag) validation("base_response_idft: table is not conjugate-symmetric");
}

// One CTA per (omega, b): threads over the output phases n; block reduction of max/min |H_n| and
// max |E_n| in shared memory (order-independent reductions).
__global__ void __launch_bounds__(256) analyze_kernel(int N, int M, int step, int kk, int g0, int nb,
                                                      const int* __restrict__ bvals, int blo,
                                                      const double* __restrict__ base /* [nb][N] */,
                                                      const double2* __restrict__ ph, const double2* __restrict__ des_pass,
                                                      const double* __restrict__ omega,
                                                      const int8_t* __restrict__ region /* [num_b][K'] */,
                                                      double delta, double* h_max, double* h_min, double* e_max,
                                                      double* abs_h, double* abs_e) {
    __shared__ double s_hmax[256], s_hmin[256], s_emax[256];
    const int gi = g0 + blockIdx.x, bl = blockIdx.y;
    const int b = bvals[bl];
    const int reg = region[size_t(b - blo) * kk + gi];
    const double2* phg = ph + size_t(gi) * N;
    const double b_omega = b * 2.0 * 3.14159265358979323846 / N;
    double2 d = make_double2(0.0, 0.0);
    if (reg != 2 && omega[gi] <= __dadd_rn(__dsub_rn(b_omega, delta / 2.0), 1e-12)) d = des_pass[gi];
    double hmax = 0.0, hmin = INFINITY, emax = 0.0;
    const size_t cell = size_t(bl) * kk + gi;
    for (int n = threadIdx.x; n < M; n += blockDim.x) {
        const double2 h = row_response(base + size_t(bl) * N, N, step * (n - (M - 1)), phg, phg[n]);
        const double ah = glibc_hypot(h.x, h.y);
        hmax = fmax(hmax, ah);
        hmin = fmin(hmin, ah);
        double ae = NAN;
        if (reg != 2) {
            ae = glibc_hypot(__dsub_rn(h.x, d.x), __dsub_rn(h.y, d.y));
            emax = fmax(emax, ae);
        }
        if (abs_h) abs_h[cell * M + n] = ah;
        if (abs_e) abs_e[cell * M + n] = ae;
    }
    s_hmax[threadIdx.x] = hmax;
    s_hmin[threadIdx.x] = hmin;
    s_emax[threadIdx.x] = emax;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            s_hmax[threadIdx.x] = fmax(s_hmax[threadIdx.x], s_hmax[threadIdx.x + o]);
            s_hmin[threadIdx.x] = fmin(s_hmin[threadIdx.x], s_hmin[threadIdx.x + o]);
            s_emax[threadIdx.x] = fmax(s_emax[threadIdx.x], s_emax[threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (h_max) h_max[cell] = s_hmax[0];
        if (h_min) h_min[cell] = s_hmin[0];
        if (e_max) e_max[cell] = reg != 2 ? s_emax[0] : NAN;
    }
}

}  // namespace analyze_impl

using namespace analyze_impl;

namespace {
int finish_ok() {
    fcvbw_gpu_detail::set_last_error("");
    return FCVBW_GPU_OK;
}
int finish_fail(const Failure& f) {
    fcvbw_gpu_detail::set_last_error(f.msg);
    return f.code;
}
}  // namespace

extern "C" int fcvbw_gpu_frequency_grid(const fcvbw_gpu_design* design, int grid_points, double* omega,
                                        int64_t capacity, int64_t* size) {
    try {
        const Geometry g = check(design);
        if (grid_points < 2 * g.N) validation("FrequencyGrid: need K >= 2N grid points");
        const Grid grid = build_grid(g.N, g.dn, g.blo, g.bhi, grid_points);
        if (size) *size = int64_t(grid.omega.size());
        if (omega) {
            if (capacity < int64_t(grid.omega.size())) validation("frequency_grid: output capacity too small");
            std::memcpy(omega, grid.omega.data(), sizeof(double) * grid.omega.size());
        }
        return finish_ok();
    } catch (const Failure& f) {
        return finish_fail(f);
    } catch (const std::exception& e) {
        return finish_fail(Failure{FCVBW_GPU_ERROR, e.what()});
    }
}

extern "C" int fcvbw_gpu_ptvir(const fcvbw_gpu_design* design, int b, int step, int device, double* rows) {
    try {
        const Geometry g = check(design);
        if (b < g.blo || b > g.bhi) validation("ptvir: b outside the design range");
        if (step != 1 && step != -1) validation("ptvir: shift step must be +-1");
        if (!rows) validation("ptvir: null output");
        ck(cudaSetDevice(device), "cudaSetDevice");
        Dev<double> d_base(static_cast<size_t>(g.N));
        base_rows(g, {b}, d_base.p);
        std::vector<double> base(size_t(g.N));
        d_base.get(base.data(), base.size());
        // ptvir_from_base (ptvir.hpp:147-160): row n = base((q + step (n - (M - 1))) mod N)
        for (int n = 0; n < g.M; ++n) {
            const int shift = step * (n - (g.M - 1));
            for (int q = 0; q < g.N; ++q) rows[size_t(n) * g.N + q] = base[size_t((q + shift) & (g.N - 1))];
        }
        return finish_ok();
    } catch (const Failure& f) {
        return finish_fail(f);
    } catch (const std::exception& e) {
        return finish_fail(Failure{FCVBW_GPU_ERROR, e.what()});
    }
}

extern "C" int fcvbw_gpu_analyze(const fcvbw_gpu_design* design, int grid_points, const int32_t* b_list, int nb,
                                 int step, int device, double* h_max, double* h_min, double* e_max, double* abs_h,
                                 double* abs_e) {
    try {
        const Geometry g = check(design);
        if (grid_points < 2 * g.N) validation("FrequencyGrid: need K >= 2N grid points");
        if (nb < 1 || !b_list) validation("analyze: empty band-centre list");
        if (step != 1 && step != -1) validation("analyze: shift step must be +-1");
        std::vector<int> bs(b_list, b_list + nb);
        for (int b : bs)
            if (b < g.blo || b > g.bhi) validation("analyze: b_N outside the design range");
        ck(cudaSetDevice(device), "cudaSetDevice");
        const int N = g.N, M = g.M;
        const Grid grid = build_grid(N, g.dn, g.blo, g.bhi, grid_points);
        const size_t kk = grid.omega.size();
        std::vector<cd> ph(kk * size_t(N)), des(kk);
        fill_phasor_table(grid.omega, N, ph.data());
        const double gd = (g.L - 1) / 2.0 + (M - 1);
        for (size_t i = 0; i < kk; ++i) {
            const double ang = -grid.omega[i] * gd;
            des[i] = {std::cos(ang), std::sin(ang)};
        }
        Dev<double2> d_ph(ph.size()), d_des(kk);
        d_ph.put(reinterpret_cast<const double2*>(ph.data()), ph.size());
        d_des.put(reinterpret_cast<const double2*>(des.data()), kk);
        Dev<double> d_omega(kk);
        d_omega.put(grid.omega.data(), kk);
        Dev<int8_t> d_region(grid.region.size());
        d_region.put(grid.region.data(), grid.region.size());
        const double delta = g.dn * 2.0 * kPi / N;

        // band centres in batches: the per-phase outputs of a batch stay below ~1 GiB on the device
        const bool per_phase = abs_h || abs_e;
        const size_t per_b = kk * (per_phase ? size_t(M) : 1);
        const int batch = int(std::max<size_t>(1, std::min<size_t>(size_t(nb), (size_t(1) << 27) / per_b)));
        Dev<double> d_base(static_cast<size_t>(batch) * N);
        Dev<int> d_b(static_cast<size_t>(batch));
        Dev<double> d_hmax(size_t(batch) * kk), d_hmin(size_t(batch) * kk), d_emax(size_t(batch) * kk);
        Dev<double> d_ah(per_phase && abs_h ? size_t(batch) * kk * M : 1);
        Dev<double> d_ae(per_phase && abs_e ? size_t(batch) * kk * M : 1);
        for (int b0 = 0; b0 < nb; b0 += batch) {
            const int n_here = std::min(batch, nb - b0);
            std::vector<int> part(bs.begin() + b0, bs.begin() + b0 + n_here);
            base_rows(g, part, d_base.p);
            d_b.put(part.data(), part.size());
            for (size_t g0 = 0; g0 < kk; g0 += 65535) {
                const unsigned gx = unsigned(std::min<size_t>(65535, kk - g0));
                analyze_kernel<<<dim3(gx, n_here), 256>>>(N, M, step, int(kk), int(g0), n_here, d_b.p, g.blo,
                                                          d_base.p, d_ph.p, d_des.p, d_omega.p, d_region.p, delta,
                                                          d_hmax.p, d_hmin.p, d_emax.p, abs_h ? d_ah.p : nullptr,
                                                          abs_e ? d_ae.p : nullptr);
                ck(cudaGetLastError(), "analyze_kernel");
            }
            const size_t cells = size_t(n_here) * kk, off = size_t(b0) * kk;
            if (h_max) d_hmax.get(h_max + off, cells);
            if (h_min) d_hmin.get(h_min + off, cells);
            if (e_max) d_emax.get(e_max + off, cells);
            if (abs_h) d_ah.get(abs_h + off * M, cells * M);
            if (abs_e) d_ae.get(abs_e + off * M, cells * M);
        }
        return finish_ok();
    } catch (const Failure& f) {
        return finish_fail(f);
    } catch (const std::exception& e) {
        return finish_fail(Failure{FCVBW_GPU_ERROR, e.what()});
    }
}
