// Host-side design tables shared by verify.cu and design.cu. Host libm (glibc) computes every
// trigonometric value, as the reference does, so that device sums built from these tables can
// reproduce the reference's results bit for bit.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

namespace fcvbw_grid {

constexpr double kPi = 3.14159265358979323846;

struct cd {  // complex double with the layout of CUDA's double2
    double x, y;
};

// FrequencyGrid::build (ptvir.hpp:309-343): K uniform points on [0, pi] plus both band edges of
// every b; region per b: 0 passband (omega <= pass edge), 1 stopband (>= stop edge), 2 excluded.
struct Grid {
    std::vector<double> omega;
    std::vector<int8_t> region;  // [num_b][K']
};

inline Grid build_grid(int n, int dn, int blo, int bhi, int k_points) {
    Grid g;
    g.omega.reserve(size_t(k_points) + 2 * size_t(bhi - blo + 1));
    for (int i = 0; i < k_points; ++i) g.omega.push_back(kPi * i / (k_points - 1));
    const int half = dn / 2;
    auto omega_of_bin = [&](int b) { return b * 2.0 * kPi / n; };
    for (int b = blo; b <= bhi; ++b) {
        for (int edge : {b - half, b + half}) {
            const double w = omega_of_bin(edge);
            auto it = std::lower_bound(g.omega.begin(), g.omega.end(), w);
            if (it == g.omega.end() || *it != w) g.omega.insert(it, w);
        }
    }
    const size_t kk = g.omega.size();
    g.region.resize(size_t(bhi - blo + 1) * kk);
    for (int b = blo; b <= bhi; ++b) {
        const double pass_edge = omega_of_bin(b - half), stop_edge = omega_of_bin(b + half);
        int8_t* r = g.region.data() + size_t(b - blo) * kk;
        for (size_t i = 0; i < kk; ++i)
            r[i] = g.omega[i] <= pass_edge ? 0 : (g.omega[i] >= stop_edge ? 1 : 2);
    }
    return g;
}

// phase_table (spectrum.hpp:208-219)
inline std::vector<cd> phase_table(int n, int l) {
    std::vector<cd> t(static_cast<size_t>(n));
    const int64_t order = l - 1;
    for (int k = 0; k <= n / 2; ++k) {
        const int64_t folded = (int64_t(k) * order) % (2 * int64_t(n));
        const double ang = -kPi * static_cast<double>(folded) / n;
        t[k] = {std::cos(ang), std::sin(ang)};
    }
    for (int k = n / 2 + 1; k < n; ++k) t[k] = {t[n - k].x, -t[n - k].y};
    return t;
}

// detail::unit_roots (ptvir.hpp:70-77)
inline std::vector<cd> unit_roots(int n) {
    std::vector<cd> r(static_cast<size_t>(n));
    for (int m = 0; m < n; ++m) {
        const double ang = 2.0 * kPi * m / n;
        r[m] = {std::cos(ang), std::sin(ang)};
    }
    return r;
}

// magnitude_samples (spectrum.hpp:170-187) x phase_table (assemble_dft_coefficients, :221-242):
// out[k] = mag(k) * phase[k] for band centre b and profile v (delta_N - 1 values).
inline void assemble_table(int n, int dn, int b, const double* v, const std::vector<cd>& phase, cd* out) {
    const int k1 = b - dn / 2 + 1, k2 = b + dn / 2 - 1;
    std::vector<double> mag(static_cast<size_t>(n), 0.0);
    mag[0] = 1.0;
    for (int k = 1; k < k1; ++k) mag[k] = mag[n - k] = 1.0;
    for (int r = 0; r <= k2 - k1; ++r) mag[k1 + r] = mag[n - (k1 + r)] = v[r];
    for (int k = 0; k < n; ++k) out[k] = {mag[k] * phase[k].x, mag[k] * phase[k].y};
}

// fill_phasors (ptvir.hpp:346-352) for every grid point: out[g * n + q] = e^{-j omega_g q}.
// Host threads; the values are glibc's, like the reference's.
inline void fill_phasor_table(const std::vector<double>& omega, int n, cd* out) {
    const size_t kk = omega.size();
    unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) {
        th.emplace_back([&, t] {
            for (size_t g = t; g < kk; g += nt) {
                cd* row = out + g * size_t(n);
                for (int q = 0; q < n; ++q) {
                    const double ang = -omega[g] * static_cast<double>(q);
                    row[q] = {std::cos(ang), std::sin(ang)};
                }
            }
        });
    }
    for (auto& x : th) x.join();
}

}  // namespace fcvbw_grid
