// fcvbw_gpu.hpp — header-only C++ adapter over the C-ABI (include/fcvbw_gpu.h).
//
// `fcvbw::gpu::OlsEngineGpu` mirrors the reference `fcvbw::OlsEngine<Radix2Fft<double>>`
// (proj/include/fcvbw/engine.hpp:28-192) method for method — block_length, fft_length, current_b,
// blocks_processed, reset, set_bandwidth, process_block, feed, flush — with the same real-valued
// `std::span<const double>` signatures and the same exception taxonomy
// (proj/include/fcvbw/errors.hpp:7-29), so reference-style callers and the reference's own
// `BlockProcessor` consumers (measure_ptvir / calibrate_shift_convention,
// proj/include/fcvbw/ptvir.hpp:20-26, 163-294) run unchanged against the GPU engine.
//
// Real streams are carried as complex128 with zero imaginary part (the filter is conjugate-
// symmetric, so the imaginary output is zero up to rounding and is dropped, exactly like the
// reference inverse keeps only the real part, fft.hpp:68-78). The complex entry points
// (process_block_complex / feed_complex / flush_complex) expose the native complex path.
#pragma once

#include <complex>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "fcvbw_gpu.h"

namespace fcvbw::gpu {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ValidationError : Error {
    using Error::Error;
};

inline void check(int rc) {
    if (rc == FCVBW_GPU_OK) return;
    const std::string msg = fcvbw_gpu_last_error();
    if (rc == FCVBW_GPU_VALIDATION) throw ValidationError(msg);
    throw Error(msg);
}

// Geometry of a structured engine (mirrors fcvbw::BinSpec, spectrum.hpp:50-77).
struct Bins {
    int fft_length = 0, filter_length = 0, block_length = 0, transition_width_bins = 0, b_low = 0, b_high = 0;
};

class OlsEngineGpu {
  public:
    // OlsEngine(const BinSpec&, TransitionProfile, int initial_b) (engine.hpp:31-45)
    OlsEngineGpu(const Bins& bins, const std::vector<double>& profile, int initial_b, int dtype = FCVBW_GPU_C128,
                 int device = 0, unsigned flags = 0) {
        fcvbw_gpu_config cfg{bins.fft_length, bins.filter_length, bins.block_length, bins.transition_width_bins,
                             bins.b_low,      bins.b_high,        profile.data(),    static_cast<int>(profile.size()),
                             initial_b,       dtype,              device,            flags};
        check(fcvbw_gpu_create(&cfg, &h_));
    }
    // OlsEngine(DftCoefficients, int M) (engine.hpp:47-56)
    OlsEngineGpu(const std::vector<std::complex<double>>& table, int block_length, int dtype = FCVBW_GPU_C128,
                 int device = 0) {
        check(fcvbw_gpu_create_raw(static_cast<int>(table.size()), block_length,
                                   reinterpret_cast<const double*>(table.data()), dtype, device, &h_));
    }
    OlsEngineGpu(const OlsEngineGpu&) = delete;
    OlsEngineGpu& operator=(const OlsEngineGpu&) = delete;
    OlsEngineGpu(OlsEngineGpu&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
    ~OlsEngineGpu() { fcvbw_gpu_destroy(h_); }

    int block_length() const { return fcvbw_gpu_block_length(h_); }
    int fft_length() const { return fcvbw_gpu_fft_length(h_); }
    int current_b() const { return fcvbw_gpu_current_b(h_); }
    std::int64_t blocks_processed() const { return fcvbw_gpu_blocks_processed(h_); }
    fcvbw_gpu_engine* handle() const { return h_; }

    void reset() { check(fcvbw_gpu_reset(h_)); }
    void set_bandwidth(int b) { check(fcvbw_gpu_set_bandwidth(h_, b)); }

    std::vector<double> process_block(std::span<const double> input) {
        auto x = to_complex(input);
        std::vector<std::complex<double>> y(x.size());
        check(fcvbw_gpu_process_block(h_, x.data(), static_cast<std::int64_t>(x.size()), y.data()));
        return real_part(y);
    }
    std::vector<double> feed(std::span<const double> samples) { return real_part(feed_complex(to_complex(samples))); }
    std::vector<double> flush() { return real_part(flush_complex()); }

    std::vector<std::complex<double>> process_block_complex(std::span<const std::complex<double>> x) {
        std::vector<std::complex<double>> y(x.size());
        check(fcvbw_gpu_process_block(h_, x.data(), static_cast<std::int64_t>(x.size()), y.data()));
        return y;
    }
    std::vector<std::complex<double>> feed_complex(std::span<const std::complex<double>> x) {
        const std::int64_t m = block_length();
        std::vector<std::complex<double>> y(static_cast<std::size_t>((static_cast<std::int64_t>(x.size()) / m + 2) * m));
        std::int64_t n = 0;
        check(fcvbw_gpu_feed(h_, x.empty() ? nullptr : x.data(), static_cast<std::int64_t>(x.size()), y.data(),
                             static_cast<std::int64_t>(y.size()), &n));
        y.resize(static_cast<std::size_t>(n));
        return y;
    }
    std::vector<std::complex<double>> flush_complex() {
        std::vector<std::complex<double>> y(static_cast<std::size_t>(block_length()));
        std::int64_t n = 0;
        check(fcvbw_gpu_flush(h_, y.data(), static_cast<std::int64_t>(y.size()), &n));
        y.resize(static_cast<std::size_t>(n));
        return y;
    }

  private:
    static std::vector<std::complex<double>> to_complex(std::span<const double> x) {
        std::vector<std::complex<double>> c(x.size());
        for (std::size_t i = 0; i < x.size(); ++i) c[i] = {x[i], 0.0};
        return c;
    }
    static std::vector<double> real_part(const std::vector<std::complex<double>>& y) {
        std::vector<double> r(y.size());
        for (std::size_t i = 0; i < y.size(); ++i) r[i] = y[i].real();
        return r;
    }
    fcvbw_gpu_engine* h_ = nullptr;
};

}  // namespace fcvbw::gpu
