// fcvbw_gpu.hpp — header-only C++ adapter over the C-ABI (include/fcvbw_gpu.h).
//
// `fcvbw::gpu::OlsEngineGpu` mirrors the reference `fcvbw::OlsEngine<Radix2Fft<double>>`
// (proj/include/fcvbw/engine.hpp:28-192) method for method — block_length, fft_length, current_b,
// blocks_processed, reset, set_bandwidth, process_block, feed, flush(PadMode) — with the same
// real-valued `std::span<const double>` signatures, and `fcvbw::gpu::new_engine` mirrors the factory
// `new_engine(const DesignResult&, int)` (proj/include/fcvbw/design.hpp:579-582). A reference
// caller swaps the engine type and nothing else, and the reference's own
// `BlockProcessor` consumers (measure_ptvir / calibrate_shift_convention,
// proj/include/fcvbw/ptvir.hpp:20-26, 163-294) run unchanged against the GPU engine.
//
// Errors: when the reference headers are on the include path (`<fcvbw/errors.hpp>`), the adapter
// throws the reference's own `fcvbw::ValidationError` / `fcvbw::Error`
// (proj/include/fcvbw/errors.hpp:7-29), so a caller's existing handlers — e.g. `fcvbw run` mapping
// ValidationError to exit 2, proj/tools/fcvbw_cli.cpp:346-355 — keep working. Without them the
// adapter defines look-alike types in fcvbw::gpu.
//
// Real streams go through the real-valued streaming entry points (fcvbw_gpu_feed_real ...): real
// samples cross PCIe (half the bytes of complex128) and each block is one transform with a zero
// imaginary part, so outputs are invariant to how the caller batches its input
// (test_oracle_engine.cpp:268-288). The complex entry points (process_block_complex /
// feed_complex / flush_complex) expose the native complex path. The adapter is fp64 (the
// reference's only precision): engines are FCVBW_GPU_C128.
#pragma once

#include <complex>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "fcvbw_gpu.h"

#if __has_include(<fcvbw/errors.hpp>)
#include <fcvbw/errors.hpp>
#define FCVBW_GPU_REFERENCE_ERRORS 1
#endif
#if __has_include(<fcvbw/design.hpp>) && __has_include(<fcvbw/engine.hpp>)
#include <fcvbw/design.hpp>
#include <fcvbw/engine.hpp>
#define FCVBW_GPU_REFERENCE_TYPES 1
#endif

namespace fcvbw::gpu {

#ifdef FCVBW_GPU_REFERENCE_ERRORS
using Error = fcvbw::Error;
using ValidationError = fcvbw::ValidationError;
#else
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ValidationError : Error {
    using Error::Error;
};
#endif

#ifdef FCVBW_GPU_REFERENCE_TYPES
using PadMode = fcvbw::PadMode;
#else
enum class PadMode { zero };  // engine.hpp:13
#endif

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
    OlsEngineGpu(const Bins& bins, const std::vector<double>& profile, int initial_b, int device = 0,
                 unsigned flags = 0) {
        fcvbw_gpu_config cfg{bins.fft_length, bins.filter_length, bins.block_length, bins.transition_width_bins,
                             bins.b_low,      bins.b_high,        profile.data(),    static_cast<int>(profile.size()),
                             initial_b,       FCVBW_GPU_C128,     device,            flags};
        check(fcvbw_gpu_create(&cfg, &h_));
    }
#ifdef FCVBW_GPU_REFERENCE_TYPES
    // the reference's own argument types
    OlsEngineGpu(const fcvbw::BinSpec& bins, fcvbw::TransitionProfile profile, int initial_b, int device = 0)
        : OlsEngineGpu(Bins{bins.fft_length, bins.filter_length, bins.block_length, bins.transition_width_bins,
                            bins.b_low, bins.b_high},
                       profile.values, initial_b, device) {}
#endif
    // OlsEngine(DftCoefficients, int M) (engine.hpp:47-56)
    OlsEngineGpu(const std::vector<std::complex<double>>& table, int block_length, int device = 0) {
        check(fcvbw_gpu_create_raw(static_cast<int>(table.size()), block_length,
                                   reinterpret_cast<const double*>(table.data()), FCVBW_GPU_C128, device, &h_));
    }
    OlsEngineGpu(const OlsEngineGpu&) = delete;
    OlsEngineGpu& operator=(const OlsEngineGpu&) = delete;
    OlsEngineGpu(OlsEngineGpu&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
    OlsEngineGpu& operator=(OlsEngineGpu&& o) noexcept {
        if (this != &o) {
            fcvbw_gpu_destroy(h_);
            h_ = o.h_;
            o.h_ = nullptr;
        }
        return *this;
    }
    ~OlsEngineGpu() { fcvbw_gpu_destroy(h_); }

    int block_length() const { return fcvbw_gpu_block_length(h_); }
    int fft_length() const { return fcvbw_gpu_fft_length(h_); }
    int current_b() const { return fcvbw_gpu_current_b(h_); }
    std::int64_t blocks_processed() const { return fcvbw_gpu_blocks_processed(h_); }
    fcvbw_gpu_engine* handle() const { return h_; }
    fcvbw_gpu_ops op_counts() const {
        fcvbw_gpu_ops o{};
        check(fcvbw_gpu_op_counts(h_, &o));
        return o;
    }

    void reset() { check(fcvbw_gpu_reset(h_)); }
    void set_bandwidth(int b) { check(fcvbw_gpu_set_bandwidth(h_, b)); }

    // real-valued streaming (engine.hpp:82-115)
    std::vector<double> process_block(std::span<const double> input) {
        std::vector<double> y(input.size());
        check(fcvbw_gpu_process_block_real(h_, input.data(), static_cast<std::int64_t>(input.size()), y.data()));
        return y;
    }
    std::vector<double> feed(std::span<const double> samples) {
        std::vector<double> y(out_capacity(samples.size()));
        std::int64_t n = 0;
        check(fcvbw_gpu_feed_real(h_, samples.empty() ? nullptr : samples.data(),
                                  static_cast<std::int64_t>(samples.size()), y.data(),
                                  static_cast<std::int64_t>(y.size()), &n));
        y.resize(static_cast<std::size_t>(n));
        return y;
    }
    std::vector<double> flush(PadMode = PadMode::zero) {
        std::vector<double> y(static_cast<std::size_t>(block_length()));
        std::int64_t n = 0;
        check(fcvbw_gpu_flush_real(h_, y.data(), static_cast<std::int64_t>(y.size()), &n));
        y.resize(static_cast<std::size_t>(n));
        return y;
    }

    // native complex streaming
    std::vector<std::complex<double>> process_block_complex(std::span<const std::complex<double>> x) {
        std::vector<std::complex<double>> y(x.size());
        check(fcvbw_gpu_process_block(h_, x.data(), static_cast<std::int64_t>(x.size()), y.data()));
        return y;
    }
    std::vector<std::complex<double>> feed_complex(std::span<const std::complex<double>> x) {
        std::vector<std::complex<double>> y(out_capacity(x.size()));
        std::int64_t n = 0;
        check(fcvbw_gpu_feed(h_, x.empty() ? nullptr : x.data(), static_cast<std::int64_t>(x.size()), y.data(),
                             static_cast<std::int64_t>(y.size()), &n));
        y.resize(static_cast<std::size_t>(n));
        return y;
    }
    std::vector<std::complex<double>> flush_complex(PadMode = PadMode::zero) {
        std::vector<std::complex<double>> y(static_cast<std::size_t>(block_length()));
        std::int64_t n = 0;
        check(fcvbw_gpu_flush(h_, y.data(), static_cast<std::int64_t>(y.size()), &n));
        y.resize(static_cast<std::size_t>(n));
        return y;
    }

  private:
    // every block the pending samples plus `n` new ones can complete
    std::size_t out_capacity(std::size_t n) const {
        const std::size_t m = static_cast<std::size_t>(block_length());
        return (n / m + 2) * m;
    }
    fcvbw_gpu_engine* h_ = nullptr;
};

#ifdef FCVBW_GPU_REFERENCE_TYPES
// new_engine(const DesignResult&, int) (design.hpp:579-582): `fcvbw::new_engine(result, b0)` becomes
// `fcvbw::gpu::new_engine(result, b0)`.
inline OlsEngineGpu new_engine(const fcvbw::DesignResult& result, int initial_b, int device = 0) {
    return OlsEngineGpu(result.bins, result.profile, initial_b, device);
}
#endif

}  // namespace fcvbw::gpu
