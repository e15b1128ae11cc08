// GPU adapter parity checks written the way the reference writes its own engine tests
// (proj/tests/test_oracle_engine.cpp), but with fcvbw::gpu::OlsEngineGpu (the C-ABI adapter) in
// place of the reference OlsEngine, and the UNMODIFIED reference headers (engine, oracle, ptvir)
// as the checker. Built by __graft_entry__.build() where /root/reference exists (the binary
// travels to the GPU box); run by tests/test_gpu_cpp.py. Prints one PASS/FAIL line per check.
#include <cmath>
#include <cstdio>
#include <functional>
#include <span>
#include <string>
#include <vector>

#include "fcvbw/engine.hpp"
#include "fcvbw/oracle.hpp"
#include "fcvbw/ptvir.hpp"
#include "fcvbw/spectrum.hpp"
#include "fcvbw_gpu.hpp"

using namespace fcvbw;

static int failures = 0;
static void check(bool ok, const std::string& what) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok) ++failures;
}

static BinSpec narrowband_bins() {
    FilterSpec spec{0.25 * kPi, 0.001, 0.001, 0.001, 0.75 * kPi, 0.8594 * kPi};
    return validate_and_discretize(spec, 128, 33);
}
static gpu::Bins to_gpu(const BinSpec& b) {
    return {b.fft_length, b.filter_length, b.block_length, b.transition_width_bins, b.b_low, b.b_high};
}
static TransitionProfile random_profile(const BinSpec& bins, std::uint64_t seed) {
    SeededRng rng(seed);
    TransitionProfile p;
    p.values.resize(static_cast<std::size_t>(bins.profile_length()));
    for (auto& v : p.values) v = rng.uniform(0.0, 1.0);
    return p;
}
static std::vector<double> random_stream(std::size_t len, std::uint64_t seed) {
    SeededRng rng(seed);
    std::vector<double> x(len);
    for (auto& v : x) v = rng.uniform(-1.0, 1.0);
    return x;
}
static double max_abs_diff(std::span<const double> a, std::span<const double> b) {
    if (a.size() != b.size()) return INFINITY;
    double w = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) w = std::max(w, std::abs(a[i] - b[i]));
    return w;
}

// the GPU adapter satisfies the reference's BlockProcessor concept (ptvir.hpp:20-26)
static_assert(BlockProcessor<gpu::OlsEngineGpu>);

int main() {
    const BinSpec bins = narrowband_bins();
    {  // engine.hpp vs GPU on random blocks (test_oracle_engine.cpp:113-123)
        auto prof = random_profile(bins, 51);
        OlsEngine<> ref(bins, prof, 48);
        gpu::OlsEngineGpu g(to_gpu(bins), prof.values, 48);
        auto x = random_stream(96 * 10, 52);
        double worst = 0;
        for (int blk = 0; blk < 10; ++blk) {
            std::span<const double> c(x.data() + blk * 96, 96);
            worst = std::max(worst, max_abs_diff(ref.process_block(c), g.process_block(c)));
        }
        check(worst <= 1e-12, "process_block matches reference OlsEngine (max " + std::to_string(worst) + ")");
    }
    {  // retune at block 10 vs retuned naive oracle (test_oracle_engine.cpp:183-197)
        auto prof = random_profile(bins, 58);
        gpu::OlsEngineGpu g(to_gpu(bins), prof.values, 48);
        NaiveBlockFilter oracle(assemble_dft_coefficients(bins, prof, 48), 96);
        auto x = random_stream(96 * 24, 59);
        double worst = 0;
        for (int blk = 0; blk < 24; ++blk) {
            if (blk == 10) {
                g.set_bandwidth(55);
                oracle.set_table(assemble_dft_coefficients(bins, prof, 55));
            }
            std::span<const double> c(x.data() + blk * 96, 96);
            worst = std::max(worst, max_abs_diff(g.process_block(c), oracle.process_block(c)));
        }
        check(worst <= 1e-9, "bandwidth switching vs naive oracle");
    }
    {  // exceptions mirror the reference taxonomy
        gpu::OlsEngineGpu g(to_gpu(bins), random_profile(bins, 62).values, 48);
        bool threw = false;
        try { g.set_bandwidth(56); } catch (const gpu::ValidationError&) { threw = true; }
        check(threw, "set_bandwidth out of range -> ValidationError");
        threw = false;
        std::vector<double> wrong(95, 0.0);
        try { g.process_block(wrong); } catch (const gpu::ValidationError&) { threw = true; }
        check(threw, "block length enforced -> ValidationError");
    }
    {  // feed/flush, batching bit-identity (test_oracle_engine.cpp:242-288)
        auto prof = random_profile(bins, 67);
        auto x = random_stream(96 * 5 + 17, 68);
        gpu::OlsEngineGpu one(to_gpu(bins), prof.values, 53), drip(to_gpu(bins), prof.values, 53);
        auto y1 = one.feed(x);
        auto t1 = one.flush();
        y1.insert(y1.end(), t1.begin(), t1.end());
        std::vector<double> y2;
        for (std::size_t i = 0; i < x.size(); i += 7) {
            auto o = drip.feed(std::span<const double>(x.data() + i, std::min<std::size_t>(7, x.size() - i)));
            y2.insert(y2.end(), o.begin(), o.end());
        }
        auto t2 = drip.flush();
        y2.insert(y2.end(), t2.begin(), t2.end());
        check(y1 == y2, "output independent of caller batching (bit-identical)");
        OlsEngine<> ref(bins, prof, 53);
        auto yr = ref.feed(x);
        auto tr = ref.flush();
        yr.insert(yr.end(), tr.begin(), tr.end());
        check(max_abs_diff(y1, yr) <= 1e-12, "feed+flush matches reference OlsEngine");
        check(one.flush().empty(), "second flush is empty");
    }
    {  // classical OLS = direct FIR through the raw-table GPU engine (test_oracle_engine.cpp:290-307)
        Radix2Fft<double> fft(128);
        SeededRng rng(69);
        double worst = 0;
        for (int trial = 0; trial < 5; ++trial) {
            std::vector<double> h(33);
            for (auto& v : h) v = rng.uniform(-1.0, 1.0);
            std::vector<double> padded(128, 0.0);
            std::copy(h.begin(), h.end(), padded.begin());
            std::vector<std::complex<double>> table(128);
            fft.forward(std::span<const double>(padded), std::span<std::complex<double>>(table));
            gpu::OlsEngineGpu g(table, 96);
            auto x = random_stream(96 * 4 + 31, 70 + trial);
            auto y = g.feed(x);
            auto t = g.flush();
            y.insert(y.end(), t.begin(), t.end());
            worst = std::max(worst, max_abs_diff(y, direct_fir_convolution(h, x)));
        }
        check(worst <= 1e-9, "classical overlap-save equals direct convolution");
    }
    {  // P10: the reference's measure_ptvir probes the GPU engine directly (test_oracle_engine.cpp:403-417)
        auto prof = random_profile(bins, 75);
        const int b = 48;
        auto coeffs = assemble_dft_coefficients(bins, prof, b);
        gpu::OlsEngineGpu g(to_gpu(bins), prof.values, b);
        NaiveBlockFilter oracle_proc(coeffs, 96);
        ShiftRule rule = default_shift_rule(96);
        PtvirSet via_gpu = measure_ptvir(g, rule, b);
        PtvirSet via_oracle = measure_ptvir(oracle_proc, rule, b);
        double worst = 0.0;
        for (std::size_t i = 0; i < via_gpu.d.size(); ++i)
            worst = std::max(worst, std::abs(via_gpu.d[i] - via_oracle.d[i]));
        check(worst <= 1e-9, "measure_ptvir through the GPU adapter equals the naive oracle's");
        ShiftRule cal = calibrate_shift_convention(g, coeffs);
        check(cal.window_offset == rule.window_offset && cal.step == rule.step,
              "calibrate_shift_convention on the GPU engine finds the OLS rule");
    }
    {  // three-way: GPU engine, naive oracle, LPTV convolution (test_oracle_engine.cpp:309-331)
        auto prof = random_profile(bins, 71);
        const int b = 52;
        auto coeffs = assemble_dft_coefficients(bins, prof, b);
        auto x = random_stream(96 * 12 + 5, 72);
        gpu::OlsEngineGpu g(to_gpu(bins), prof.values, b);
        auto y = g.feed(x);
        auto t = g.flush();
        y.insert(y.end(), t.begin(), t.end());
        auto yn = naive_block_filter(coeffs, x, 96);
        NaiveBlockFilter probe(coeffs, 96);
        ShiftRule rule = default_shift_rule(96);
        auto yl = lptv_convolution(measure_ptvir(probe, rule, b), x, rule.window_offset);
        check(max_abs_diff(y, yn) <= 1e-9 && max_abs_diff(y, yl) <= 1e-9, "three-way agreement GPU/naive/LPTV");
    }
    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
