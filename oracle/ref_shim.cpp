// TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// C-ABI shim over the UNMODIFIED reference headers (`/root/reference/proj/include/fcvbw/*.hpp`),
// compiled in place by `oracle/Makefile` into `oracle/_ref/libfcvbw_ref.so`. No reference
// source is copied into this repository: this file only #includes the headers and exposes the
// reference's own functions under plain C names so that tests, golden-vector generation and the
// bench's `cpu_baseline` / `--impl reference` leg can call them from Python (ctypes).
//
// Reference interfaces wrapped here (file:line relative to /root/reference):
//   OlsEngine                       proj/include/fcvbw/engine.hpp:28-192
//   Radix2Fft                       proj/include/fcvbw/fft.hpp:32-115
//   phase_table                     proj/include/fcvbw/spectrum.hpp:208-219
//   magnitude_samples / bin_region  proj/include/fcvbw/spectrum.hpp:170-202
//   assemble_dft_coefficients       proj/include/fcvbw/spectrum.hpp:221-242
//   BinSpec::validate               proj/include/fcvbw/spectrum.hpp:63-76
//   NaiveBlockFilter / naive_block_filter / direct_fir_convolution
//                                   proj/include/fcvbw/oracle.hpp:36-134
//   SeededRng                       proj/include/fcvbw/ops.hpp:62-86
//   design / DesignOptions          proj/include/fcvbw/design.hpp:452-577
//   verify / calibrated_shift_rule  proj/include/fcvbw/design.hpp:476-484,584-673
//   solve_minimax / design          proj/include/fcvbw/design.hpp:276-446,486-577
//   cmd_run block loop (restated)   proj/tools/fcvbw_cli.cpp:95-113
//
// Complex streams: the reference engine is real-input only (engine.hpp:82,92). Because every
// structured H(k) is conjugate-symmetric, the complex OLS output equals engine(Re x) + j
// engine(Im x) exactly; `ref_ols_complex` runs those two real engines.

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "fcvbw/design.hpp"
#include "fcvbw/engine.hpp"
#include "fcvbw/oracle.hpp"
#include "fcvbw/spectrum.hpp"

using namespace fcvbw;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const ValidationError*>(&e)) return 2;
    return 1;
}

BinSpec make_bins(int n, int l, int dn, int blo, int bhi) {
    BinSpec b;
    b.fft_length = n;
    b.filter_length = l;
    b.block_length = n - l + 1;
    b.transition_width_bins = dn;
    b.b_low = blo;
    b.b_high = bhi;
    return b;
}

// Runs one real stream through a fresh reference engine over global blocks [b0, b1), writing
// outputs of those blocks into y (indexed by absolute time). Blocks are fed exactly as the
// reference CLI does (proj/tools/fcvbw_cli.cpp:100-113): set_bandwidth before the named block,
// process_block for full blocks, feed+flush for the partial tail. The engine is primed by
// re-running the `prime` preceding blocks (their output discarded), which is exact because a
// block depends only on its N-sample segment (engine.hpp:139-172).
// x[i - x_off] holds input time i and y[i - y_off] receives output time i.
void run_real_range(const BinSpec& bins, const TransitionProfile& prof, const double* x,
                    std::int64_t x_off, std::int64_t s, const int* bsched, int b_default,
                    std::int64_t b0, std::int64_t b1, double* y, std::int64_t y_off) {
    const int m = bins.block_length;
    const int n = bins.fft_length;
    const std::int64_t prime_blocks = (n - m + m - 1) / m;
    const std::int64_t start = std::max<std::int64_t>(0, b0 - prime_blocks);
    OlsEngine<> eng(bins, prof, bsched ? bsched[start] : b_default);
    for (std::int64_t blk = start; blk < b1; ++blk) {
        if (bsched) eng.set_bandwidth(bsched[blk]);
        const std::int64_t pos = blk * m;
        const std::int64_t take = std::min<std::int64_t>(m, s - pos);
        std::vector<double> out;
        if (take == m) {
            out = eng.process_block(
                std::span<const double>(x + (pos - x_off), static_cast<std::size_t>(m)));
        } else {
            eng.feed(std::span<const double>(x + (pos - x_off), static_cast<std::size_t>(take)));
            out = eng.flush();
        }
        if (blk >= b0) std::copy(out.begin(), out.end(), y + (pos - y_off));
    }
}

template <class Fn>
void parallel_ranges(std::int64_t nblocks, int threads, Fn&& fn) {
    if (threads <= 1 || nblocks <= 1) {
        fn(0, nblocks);
        return;
    }
    threads = static_cast<int>(std::min<std::int64_t>(threads, nblocks));
    std::vector<std::thread> pool;
    std::vector<std::exception_ptr> errs(static_cast<std::size_t>(threads));
    const std::int64_t chunk = (nblocks + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        const std::int64_t lo = t * chunk, hi = std::min(nblocks, lo + chunk);
        if (lo >= hi) break;
        pool.emplace_back([&, t, lo, hi] {
            try {
                fn(lo, hi);
            } catch (...) {
                errs[t] = std::current_exception();
            }
        });
    }
    for (auto& th : pool) th.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// BinSpec::validate + profile-length check (spectrum.hpp:63-76, engine.hpp:39-41).
int ref_validate(int n, int l, int m, int dn, int blo, int bhi, int lv) {
    try {
        BinSpec b = make_bins(n, l, dn, blo, bhi);
        b.block_length = m;
        b.validate();
        if (lv != b.profile_length())
            throw ValidationError("engine: profile length must be delta_N - 1");
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Whole real stream through the structured engine. `bsched` (nullable) holds one b per block.
int ref_ols_real(int n, int l, int dn, int blo, int bhi, const double* v, const double* x,
                 std::int64_t s, const int* bsched, int b0, double* y, int threads) {
    try {
        BinSpec bins = make_bins(n, l, dn, blo, bhi);
        TransitionProfile prof{std::vector<double>(v, v + bins.profile_length())};
        const std::int64_t nb = (s + bins.block_length - 1) / bins.block_length;
        parallel_ranges(nb, threads, [&](std::int64_t lo, std::int64_t hi) {
            run_real_range(bins, prof, x, 0, s, bsched, b0, lo, hi, y, 0);
        });
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Multichannel complex streams, interleaved (re, im) doubles, layout [channels][s]; `bsched`
// is [channels][nblocks] when b_channel_stride == nblocks, or one shared schedule when 0.
// Parallel over (channel, component, block range).
int ref_ols_complex(int n, int l, int dn, int blo, int bhi, const double* v, const double* x,
                    std::int64_t s, int channels, const int* bsched,
                    std::int64_t b_channel_stride, int b0, double* y, int threads) {
    try {
        BinSpec bins = make_bins(n, l, dn, blo, bhi);
        bins.validate();
        TransitionProfile prof{std::vector<double>(v, v + bins.profile_length())};
        const std::int64_t nb = (s + bins.block_length - 1) / bins.block_length;
        const std::int64_t streams = 2LL * channels;
        // split every (channel, component) stream into ranges so that all threads stay busy
        const std::int64_t ranges_per_stream =
            std::max<std::int64_t>(1, std::min<std::int64_t>(nb, (threads + streams - 1) / streams));
        const std::int64_t per = (nb + ranges_per_stream - 1) / ranges_per_stream;
        const std::int64_t units = streams * ranges_per_stream;
        const std::int64_t m = bins.block_length;
        const std::int64_t prime_blocks = (bins.fft_length - m + m - 1) / m;
        parallel_ranges(units, threads, [&](std::int64_t lo, std::int64_t hi) {
            std::vector<double> xr, yr;
            for (std::int64_t u = lo; u < hi; ++u) {
                const std::int64_t st = u / ranges_per_stream, r = u % ranges_per_stream;
                const std::int64_t ch = st / 2, comp = st % 2;
                const std::int64_t rb0 = r * per, rb1 = std::min(nb, rb0 + per);
                if (rb0 >= rb1) continue;
                // de-interleave only the window this range reads (primer blocks included)
                const std::int64_t w0 = std::max<std::int64_t>(0, rb0 - prime_blocks) * m;
                const std::int64_t w1 = std::min<std::int64_t>(s, rb1 * m);
                const std::int64_t t0 = rb0 * m;
                const double* xc = x + 2 * ch * s;
                xr.resize(static_cast<std::size_t>(w1 - w0));
                yr.resize(static_cast<std::size_t>(w1 - t0));
                for (std::int64_t i = w0; i < w1; ++i) xr[i - w0] = xc[2 * i + comp];
                const int* bs = bsched ? bsched + ch * b_channel_stride : nullptr;
                run_real_range(bins, prof, xr.data(), w0, s, bs, b0, rb0, rb1, yr.data(), t0);
                double* yc = y + 2 * ch * s;
                for (std::int64_t i = t0; i < w1; ++i) yc[2 * i + comp] = yr[i - t0];
            }
        });
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Raw-table engine (engine.hpp:47-56, 163-165) over a real stream with feed + flush.
int ref_ols_raw_real(int n, int m, const double* table, const double* x, std::int64_t s,
                     double* y) {
    try {
        DftCoefficients c;
        c.table.resize(static_cast<std::size_t>(n));
        for (int k = 0; k < n; ++k) c.table[k] = {table[2 * k], table[2 * k + 1]};
        OlsEngine<> eng(c, m);
        auto out = eng.feed(std::span<const double>(x, static_cast<std::size_t>(s)));
        auto tail = eng.flush();
        out.insert(out.end(), tail.begin(), tail.end());
        std::copy(out.begin(), out.end(), y);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// naive_block_filter (oracle.hpp:105-121): O(N^2) per block, independent of the FFT.
int ref_naive_block_filter(int n, int m, const double* table, const double* x, std::int64_t s,
                           double* y) {
    try {
        DftCoefficients c;
        c.table.resize(static_cast<std::size_t>(n));
        for (int k = 0; k < n; ++k) c.table[k] = {table[2 * k], table[2 * k + 1]};
        auto out = naive_block_filter(c, std::span<const double>(x, static_cast<std::size_t>(s)), m);
        std::copy(out.begin(), out.end(), y);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// direct_fir_convolution (oracle.hpp:124-134).
int ref_direct_fir(const double* taps, int nt, const double* x, std::int64_t s, double* y) {
    try {
        auto out = direct_fir_convolution(std::span<const double>(taps, static_cast<std::size_t>(nt)),
                                          std::span<const double>(x, static_cast<std::size_t>(s)));
        std::copy(out.begin(), out.end(), y);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// phase_table (spectrum.hpp:208-219) as 2N interleaved doubles.
int ref_phase_table(int n, int l, double* out) {
    try {
        auto t = phase_table(n, l);
        for (int k = 0; k < n; ++k) {
            out[2 * k] = t[k].real();
            out[2 * k + 1] = t[k].imag();
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// magnitude_samples + bin_region + assemble_dft_coefficients (spectrum.hpp:170-242) for one b.
// region: 0 passband, 1 transition, 2 stopband (BinRegion order).
int ref_coefficients(int n, int l, int dn, int blo, int bhi, const double* v, int b,
                     double* mag, int* region, double* table) {
    try {
        BinSpec bins = make_bins(n, l, dn, blo, bhi);
        bins.validate();
        TransitionProfile prof{std::vector<double>(v, v + bins.profile_length())};
        auto mg = magnitude_samples(bins, prof, b);
        auto c = assemble_dft_coefficients(bins, prof, b);
        for (int k = 0; k < n; ++k) {
            if (mag) mag[k] = mg[k];
            if (region) region[k] = static_cast<int>(bin_region(bins, b, k));
            if (table) {
                table[2 * k] = c.table[k].real();
                table[2 * k + 1] = c.table[k].imag();
            }
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// SeededRng (ops.hpp:62-86): `count` draws of uniform(lo, hi) or uniform_int(lo, hi).
void ref_rng_uniform(std::uint64_t seed, double lo, double hi, double* out, std::int64_t count) {
    SeededRng rng(seed);
    for (std::int64_t i = 0; i < count; ++i) out[i] = rng.uniform(lo, hi);
}
void ref_rng_uniform_int(std::uint64_t seed, int lo, int hi, int* out, std::int64_t count) {
    SeededRng rng(seed);
    for (std::int64_t i = 0; i < count; ++i) out[i] = rng.uniform_int(lo, hi);
}

// design() with fixed (N, L) (design.hpp:486-528 with both overrides): produces the shared
// transition-band table V used by the BASELINE config artifacts.
int ref_design(int n, int l, int dn, int blo, int bhi, int grid_k, double* v_out,
               double* delta_out) {
    try {
        FilterSpec spec;
        spec.transition_width = dn * 2.0 * kPi / n;
        spec.ripple_pass = 0.01;
        spec.ripple_stop = 0.01;
        spec.max_error = 0.5;
        spec.band_center_low = blo * 2.0 * kPi / n;
        spec.band_center_high = bhi * 2.0 * kPi / n;
        DesignOptions opt;
        opt.fft_length_override = n;
        opt.filter_length_override = l;
        opt.grid_points = grid_k;
        DesignResult r = design(spec, opt);
        for (int i = 0; i < r.profile.length(); ++i) v_out[i] = r.profile.values[i];
        *delta_out = r.delta;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// verify() (design.hpp:601-673) on a DesignResult assembled from its fields, with the reference's
// own calibrated shift rule. Output layout as orc_verify (oracle/fcvbw_oracle.c).
int ref_verify(int n, int l, int dn, int blo, int bhi, const double* v, double design_delta,
               int grid_points, int facets, int dense, double delta_e, double* per_b,
               double* per_n, double* out_d, int* out_i) {
    try {
        DesignResult r;
        r.bins = make_bins(n, l, dn, blo, bhi);
        r.bins.validate();
        r.profile.values.assign(v, v + (dn - 1));
        r.delta = design_delta;
        r.grid_points = grid_points;
        r.facets = facets;
        VerificationReport rep = verify(r, dense, delta_e);
        if (per_b)
            for (int b = blo; b <= bhi; ++b) per_b[b - blo] = rep.per_b_max.at(b);
        if (per_n) std::copy(rep.per_n_max.begin(), rep.per_n_max.end(), per_n);
        out_d[0] = rep.delta;
        out_d[1] = rep.passband_max;
        out_d[2] = rep.stopband_max;
        out_d[3] = rep.worst_omega;
        out_d[4] = rep.refinement_bound;
        out_i[0] = rep.dense_points;
        out_i[1] = rep.worst_b;
        out_i[2] = rep.worst_n;
        out_i[3] = rep.pass;
        out_i[4] = rep.within_bound;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// calibrated_shift_rule (design.hpp:476-484): the (window_offset, step) verify() uses.
int ref_shift_rule(int n, int l, int dn, int blo, int bhi, int* window_offset, int* step) {
    try {
        BinSpec bins = make_bins(n, l, dn, blo, bhi);
        bins.validate();
        ShiftRule rule = calibrated_shift_rule(bins);
        *window_offset = rule.window_offset;
        *step = rule.step;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// solve_minimax (design.hpp:276-446) for one BinSpec with the calibrated shift rule, as design()
// evaluates one candidate order. out_d = {delta, lp_delta}; out_i = {rounds, lp_iterations,
// active triples}.
int ref_solve_minimax(int n, int l, int dn, int blo, int bhi, int grid_k, int facets, double exchange_tol,
                      int max_rounds, int seed_stride, double* v_out, double* out_d, std::int64_t* out_i) {
    try {
        BinSpec bins = make_bins(n, l, dn, blo, bhi);
        bins.validate();
        DesignProblem problem{bins, FrequencyGrid::build(bins, grid_k), facets, exchange_tol, max_rounds,
                              seed_stride};
        SolveOutcome o = solve_minimax(problem, calibrated_shift_rule(bins));
        for (int i = 0; i < o.profile.length(); ++i) v_out[i] = o.profile.values[i];
        out_d[0] = o.delta;
        out_d[1] = o.lp_delta;
        out_i[0] = o.rounds;
        out_i[1] = o.lp_iterations;
        out_i[2] = static_cast<std::int64_t>(o.system.size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// design(spec, options) (design.hpp:486-577) with the order loop. spec_d = {transition_width,
// ripple_pass, ripple_stop, max_error, band_center_low, band_center_high}; opt_i = {fft_length_override,
// filter_length_override, grid_points, facets, max_rounds, seed_stride}; opt_d = {exchange_tol, margin}.
// geo_out = {N, L, M, delta_N, b_low, b_high, iterations, exchange_rounds}; v_out capacity vcap.
int ref_design_full(const double* spec_d, const int* opt_i, const double* opt_d, int* geo_out, double* v_out,
                    int vcap, double* delta_out) {
    try {
        FilterSpec spec;
        spec.transition_width = spec_d[0];
        spec.ripple_pass = spec_d[1];
        spec.ripple_stop = spec_d[2];
        spec.max_error = spec_d[3];
        spec.band_center_low = spec_d[4];
        spec.band_center_high = spec_d[5];
        DesignOptions opt;
        opt.fft_length_override = opt_i[0];
        opt.filter_length_override = opt_i[1];
        opt.grid_points = opt_i[2];
        opt.facets = opt_i[3];
        opt.max_rounds = opt_i[4];
        opt.seed_stride = opt_i[5];
        opt.exchange_tol = opt_d[0];
        opt.margin = opt_d[1];
        DesignResult r = design(spec, opt);
        geo_out[0] = r.bins.fft_length;
        geo_out[1] = r.bins.filter_length;
        geo_out[2] = r.bins.block_length;
        geo_out[3] = r.bins.transition_width_bins;
        geo_out[4] = r.bins.b_low;
        geo_out[5] = r.bins.b_high;
        geo_out[6] = r.iterations;
        geo_out[7] = r.exchange_rounds;
        if (r.profile.length() > vcap) throw Error("ref_design_full: profile capacity");
        for (int i = 0; i < r.profile.length(); ++i) v_out[i] = r.profile.values[i];
        *delta_out = r.delta;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
