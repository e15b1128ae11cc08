// Drop-in check of the C++ adapter: the block loop of the reference's `fcvbw run`
// (proj/tools/fcvbw_cli.cpp:76-113) and its exception-to-exit-code mapping (:338-355), restated
// with ONLY the engine factory changed — `fcvbw::new_engine` (design.hpp:579-582) for the reference
// and `fcvbw::gpu::new_engine` for the GPU. The GPU run must:
//   * return exit 2 when the schedule requests a b outside the design range, or the initial b is out
//     of range (the adapter throws the reference's own fcvbw::ValidationError);
//   * write the same f64le bytes as the in-process GPU engine fed the whole stream (bitwise), and
//     agree with the reference CLI loop within 1e-12;
//   * tally exactly the reference's variable multiplications (2 L_V per block, none per retune).
// Prints one PASS/FAIL line per check; run by tests/test_cpp_boundary.py on the GPU.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <iostream>
#include <span>
#include <string>
#include <vector>

#include "fcvbw/design.hpp"
#include "fcvbw/engine.hpp"
#include "fcvbw/errors.hpp"
#include "fcvbw/ops.hpp"
#include "fcvbw/spectrum.hpp"
#include "fcvbw_gpu.hpp"

namespace {

int failures = 0;
void check(bool ok, const std::string& what) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok) ++failures;
}

struct ScheduleEntry {
    std::int64_t block;
    int b;
    std::size_t line;
};

constexpr int kExitUsage = 2;  // fcvbw_cli.cpp:16-17

// fcvbw_cli.cpp:76-113 with the engine factory as the only parameter. (Reading the artifact and the
// signal and load_schedule's own range check are outside the loop; the schedule here is passed
// unchecked so that the ENGINE's set_bandwidth raises the ValidationError.)
template <class NewEngine>
int cmd_run(const fcvbw::DesignResult& result, const std::vector<double>& input,
            const std::vector<ScheduleEntry>& schedule, int initial_b, std::vector<double>& output_out,
            NewEngine new_engine) {
    const int b0 = initial_b >= 0 ? initial_b : result.bins.b_low;

    auto engine = new_engine(result, b0);
    const int m = result.bins.block_length;
    const std::int64_t total_blocks =
        static_cast<std::int64_t>((input.size() + m - 1) / static_cast<std::size_t>(m));
    for (const auto& ev : schedule) {
        if (ev.block >= total_blocks)
            throw fcvbw::ValidationError("schedule:" + std::to_string(ev.line) + ": block index " +
                                         std::to_string(ev.block) + " beyond the input stream (" +
                                         std::to_string(total_blocks) + " blocks)");
    }

    std::vector<double> output;
    output.reserve(input.size());
    std::size_t pos = 0;
    std::int64_t block = 0;
    std::size_t next_event = 0;
    while (pos < input.size()) {
        while (next_event < schedule.size() && schedule[next_event].block == block) {
            engine.set_bandwidth(schedule[next_event].b);
            ++next_event;
        }
        const std::size_t take = std::min<std::size_t>(input.size() - pos, static_cast<std::size_t>(m));
        std::span<const double> chunk(input.data() + pos, take);
        std::vector<double> y = take == static_cast<std::size_t>(m) ? engine.process_block(chunk)
                                                                     : (engine.feed(chunk), engine.flush());
        output.insert(output.end(), y.begin(), y.end());
        pos += take;
        ++block;
    }
    output_out = output;
    return 0;
}

// fcvbw_cli.cpp:338-355: the CLI's exception-to-exit-code mapping
template <class F>
int cli_main(F&& body) {
    try {
        return body();
    } catch (const fcvbw::NonConvergenceError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 3;
    } catch (const fcvbw::ValidationError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitUsage;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}

fcvbw::DesignResult narrowband_design() {
    fcvbw::FilterSpec spec{0.25 * fcvbw::kPi, 0.001, 0.001, 0.001, 0.75 * fcvbw::kPi, 0.8594 * fcvbw::kPi};
    fcvbw::DesignResult r;
    r.bins = fcvbw::validate_and_discretize(spec, 128, 33);
    fcvbw::SeededRng rng(3);
    r.profile.values.resize(static_cast<std::size_t>(r.bins.profile_length()));
    for (auto& v : r.profile.values) v = rng.uniform(0.0, 1.0);
    return r;
}

std::vector<double> stream(std::size_t len, std::uint64_t seed) {
    fcvbw::SeededRng rng(seed);
    std::vector<double> x(len);
    for (auto& v : x) v = rng.uniform(-1.0, 1.0);
    return x;
}

}  // namespace

int main() {
    const fcvbw::DesignResult res = narrowband_design();
    const int m = res.bins.block_length;
    const auto x = stream(static_cast<std::size_t>(m) * 20 + 13, 7);
    const std::vector<ScheduleEntry> sched{{0, 48, 1}, {5, 55, 2}, {11, 50, 3}};
    auto ref_factory = [](const fcvbw::DesignResult& r, int b) { return fcvbw::new_engine(r, b); };
    auto gpu_factory = [](const fcvbw::DesignResult& r, int b) { return fcvbw::gpu::new_engine(r, b); };

    std::vector<double> y_ref, y_gpu;
    const int rc_ref = cli_main([&] { return cmd_run(res, x, sched, 48, y_ref, ref_factory); });
    const int rc_gpu = cli_main([&] { return cmd_run(res, x, sched, 48, y_gpu, gpu_factory); });
    check(rc_ref == 0 && rc_gpu == 0, "cmd_run exits 0 with the reference and the GPU engine");
    check(y_gpu.size() == x.size(), "GPU run emits one output per input sample");
    double worst = 0.0;
    for (std::size_t i = 0; i < y_ref.size() && i < y_gpu.size(); ++i)
        worst = std::max(worst, std::abs(y_ref[i] - y_gpu[i]));
    check(y_ref.size() == y_gpu.size() && worst <= 1e-12,
          "GPU cmd_run matches the reference cmd_run (max " + std::to_string(worst) + ")");

    {  // f64le bytes equal to the in-process GPU engine fed the whole stream with the same schedule
        auto eng = fcvbw::gpu::new_engine(res, 48);
        std::vector<double> y;
        for (std::int64_t blk = 0; blk * m < static_cast<std::int64_t>(x.size()); ++blk) {
            for (const auto& ev : sched)
                if (ev.block == blk) eng.set_bandwidth(ev.b);
            const std::size_t lo = static_cast<std::size_t>(blk * m);
            const std::size_t n = std::min<std::size_t>(x.size() - lo, static_cast<std::size_t>(m));
            auto o = eng.feed(std::span<const double>(x.data() + lo, n));
            y.insert(y.end(), o.begin(), o.end());
        }
        auto t = eng.flush(fcvbw::PadMode::zero);
        y.insert(y.end(), t.begin(), t.end());
        check(y.size() == y_gpu.size() && std::memcmp(y.data(), y_gpu.data(), y.size() * sizeof(double)) == 0,
              "f64le output bitwise equal to the in-process GPU engine (test_cli.cpp:134-150)");
    }

    {  // out-of-range schedule entry -> the engine throws fcvbw::ValidationError -> exit 2
        const std::vector<ScheduleEntry> bad{{0, 48, 1}, {3, res.bins.b_high + 1, 2}};
        std::vector<double> y;
        const int rc = cli_main([&] { return cmd_run(res, x, bad, 48, y, gpu_factory); });
        const int rc_r = cli_main([&] { return cmd_run(res, x, bad, 48, y, ref_factory); });
        check(rc == kExitUsage && rc_r == kExitUsage,
              "out-of-range schedule -> exit 2 (GPU " + std::to_string(rc) + ", reference " + std::to_string(rc_r) +
                  ") (test_cli.cpp:152-163)");
        const int rc0 = cli_main([&] { return cmd_run(res, x, {}, res.bins.b_low - 1, y, gpu_factory); });
        check(rc0 == kExitUsage, "out-of-range initial b -> exit 2");
        const std::vector<ScheduleEntry> late{{100000, 48, 1}};
        const int rc1 = cli_main([&] { return cmd_run(res, x, late, 48, y, gpu_factory); });
        check(rc1 == kExitUsage, "schedule beyond the stream -> exit 2");
    }

    {  // AC8: variable multiplications 2 L_V per block, zero flops per retune
       // (test_oracle_engine.cpp:216-240, ops.hpp:15-30)
        auto eng = fcvbw::gpu::new_engine(res, 51);
        fcvbw::OlsEngine<> ref(res.bins, res.profile, 51);
        std::vector<double> block(static_cast<std::size_t>(m), 0.5);
        eng.process_block(block);
        ref.process_block(block);
        const auto g0 = eng.op_counts();
        fcvbw::op_counters().reset();
        for (int i = 0; i < 5; ++i) {
            eng.process_block(block);
            ref.process_block(block);
        }
        const auto g1 = eng.op_counts();
        const std::uint64_t lv = static_cast<std::uint64_t>(res.bins.profile_length());
        check(g1.variable_mul - g0.variable_mul == fcvbw::op_counters().variable_mul &&
                  fcvbw::op_counters().variable_mul == 5u * 2u * lv,
              "variable multiplications = reference OpCounters = 2 L_V per block (" +
                  std::to_string(g1.variable_mul - g0.variable_mul) + ")");
        const fcvbw::OpCounters before = fcvbw::op_counters();
        eng.set_bandwidth(55);
        eng.set_bandwidth(48);
        ref.set_bandwidth(55);
        ref.set_bandwidth(48);
        const auto g2 = eng.op_counts();
        check(fcvbw::op_counters() == before && g2.variable_mul == g1.variable_mul && g2.retune_flops == 0,
              "retuning performs no floating-point arithmetic");
    }

    {  // construction-time self-check (check_provider, engine.hpp:126-137): a corrupted twiddle fails
        bool threw = false;
        try {
            fcvbw::gpu::OlsEngineGpu g(
                fcvbw::gpu::Bins{res.bins.fft_length, res.bins.filter_length, res.bins.block_length,
                                 res.bins.transition_width_bins, res.bins.b_low, res.bins.b_high},
                res.profile.values, 48, 0, FCVBW_GPU_TEST_CORRUPT_TWIDDLES);
        } catch (const fcvbw::ValidationError& e) {
            threw = std::string(e.what()).find("round-trip") != std::string::npos;
        }
        check(threw, "corrupted twiddle table fails the round-trip self-check -> ValidationError");
    }

    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
