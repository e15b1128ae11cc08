// TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// The reference's `design` and `analyze` CLI verbs (proj/tools/fcvbw_cli.cpp:44-70 cmd_design,
// :120-193 cmd_analyze) re-expressed as C functions over the UNMODIFIED reference headers, because
// the CLI itself cannot be built here (it needs CLI11, fcvbw_cli.cpp:10). Only the argument
// parsing is absent; every computation and every file writer is the reference's own
// (parse_spec_file, design, verify, save_artifact, verification_to_json, load_artifact,
// FrequencyGrid, ptvir_from_base, response_from_row, desired_response, write_ptvir_csv,
// format_double). Built by oracle/Makefile into oracle/_ref/libfcvbw_ref_cli.so with the
// nlohmann/json header the reference's io.hpp includes. Used by tests/golden/make_cli_golden.py.

#include <cstdint>
#include <fstream>
#include <iostream>
#include <limits>
#include <string>
#include <vector>

#include "fcvbw/design.hpp"
#include "fcvbw/io.hpp"
#include "fcvbw/ptvir.hpp"

namespace {
thread_local std::string g_err;
constexpr int kUsage = 2, kNoConverge = 3;  // fcvbw_cli.cpp:16-17
}  // namespace

extern "C" {

const char* ref_cli_last_error(void) { return g_err.c_str(); }

// cmd_design: spec file -> design() -> verify() on the dense grid -> artifact + report JSON.
// Returns the CLI exit code (0 meets max_error, 1 not met / other error, 2 validation, 3 no
// convergence), fcvbw_cli.cpp:44-70,338-355.
int ref_cli_design(const char* spec_path, const char* artifact_path, const char* report_path, int dense_k) {
    try {
        fcvbw::SpecFile file = fcvbw::parse_spec_file(spec_path);
        fcvbw::DesignResult result = fcvbw::design(file.spec, file.options);
        const int k = dense_k > 0 ? dense_k : 4 * file.options.grid_points;
        fcvbw::VerificationReport report = fcvbw::verify(result, k, file.spec.max_error);
        result.verification = report.delta;
        fcvbw::save_artifact(artifact_path, result);
        std::ofstream out(report_path);
        if (!out) throw fcvbw::Error(std::string("cannot write ") + report_path);
        out << fcvbw::verification_to_json(report).dump(2) << '\n';
        return result.delta <= file.spec.max_error ? 0 : 1;
    } catch (const fcvbw::NonConvergenceError& e) {
        g_err = e.what();
        return kNoConverge;
    } catch (const fcvbw::ValidationError& e) {
        g_err = e.what();
        return kUsage;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// cmd_analyze: profile CSV, response CSV (per b and grid point: max/min |H_n| over n, max |E_n| on
// masked points), one PTVIR table per b, optional per-phase long CSV. b < 0 means "all".
int ref_cli_analyze(const char* artifact_path, int grid_k, int b_single, const char* prefix_c, int per_phase) {
    try {
        const std::string prefix = prefix_c;
        fcvbw::DesignResult result = fcvbw::load_artifact(artifact_path);
        const fcvbw::BinSpec& bins = result.bins;
        fcvbw::FrequencyGrid grid = fcvbw::FrequencyGrid::build(bins, grid_k);
        const fcvbw::ShiftRule rule = fcvbw::calibrated_shift_rule(bins);
        std::vector<int> bs;
        if (b_single < 0) {
            for (int b = bins.b_low; b <= bins.b_high; ++b) bs.push_back(b);
        } else {
            if (!bins.contains_b(b_single)) throw fcvbw::ValidationError("analyze: b_N outside the design range");
            bs.push_back(b_single);
        }
        {
            std::ofstream pf(prefix + "_profile.csv");
            pf << "r,V\n";
            for (int r = 0; r < result.profile.length(); ++r)
                pf << r << ',' << fcvbw::format_double(result.profile.values[r]) << '\n';
        }
        std::ofstream resp(prefix + "_response.csv");
        resp << "b_N,omega_over_pi,region,abs_Hn_max,abs_Hn_min,abs_En_max\n";
        std::ofstream phases;
        if (per_phase) {
            phases.open(prefix + "_phases.csv");
            phases << "b_N,n,omega_over_pi,abs_Hn,abs_En\n";
        }
        const int m = bins.block_length;
        std::vector<std::complex<double>> ph(static_cast<std::size_t>(bins.fft_length));
        for (int b : bs) {
            const auto coeffs = fcvbw::assemble_dft_coefficients(bins, result.profile, b);
            const fcvbw::PtvirSet rows = fcvbw::ptvir_from_base(fcvbw::base_response_idft(coeffs), m, rule, b);
            {
                std::ofstream pt(prefix + "_ptvir_" + std::to_string(b) + ".csv");
                fcvbw::write_ptvir_csv(pt, rows);
            }
            const auto region = grid.region(b);
            const double b_omega = bins.omega_of_bin(b);
            for (std::size_t gi = 0; gi < grid.omega.size(); ++gi) {
                const double w = grid.omega[gi];
                fcvbw::fill_phasors(w, ph);
                const bool masked = region[gi] != 2;
                const std::complex<double> want =
                    masked ? fcvbw::desired_response(w, b_omega, bins.delta(), bins.filter_length, m)
                           : std::complex<double>{};
                double hmax = 0.0, hmin = std::numeric_limits<double>::infinity(), emax = 0.0;
                for (int n = 0; n < m; ++n) {
                    const std::complex<double> h = fcvbw::response_from_row(rows.row(n), ph, ph[n]);
                    hmax = std::max(hmax, std::abs(h));
                    hmin = std::min(hmin, std::abs(h));
                    if (masked) emax = std::max(emax, std::abs(h - want));
                    if (per_phase) {
                        phases << b << ',' << n << ',' << fcvbw::format_double(w / fcvbw::kPi) << ','
                               << fcvbw::format_double(std::abs(h)) << ',';
                        if (masked) phases << fcvbw::format_double(std::abs(h - want));
                        phases << '\n';
                    }
                }
                const char* name = region[gi] == 0 ? "pass" : region[gi] == 1 ? "stop" : "transition";
                resp << b << ',' << fcvbw::format_double(w / fcvbw::kPi) << ',' << name << ','
                     << fcvbw::format_double(hmax) << ',' << fcvbw::format_double(hmin) << ',';
                if (masked) resp << fcvbw::format_double(emax);
                resp << '\n';
            }
        }
        return 0;
    } catch (const fcvbw::ValidationError& e) {
        g_err = e.what();
        return kUsage;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

}  // extern "C"
