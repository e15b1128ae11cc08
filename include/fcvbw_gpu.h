/* fcvbw_gpu.h — C-ABI of the B200-native overlap-save variable-bandwidth (VBW) filter.
 *
 * Drop-in boundary for the hot path of the reference `fcvbw` library (arXiv 2406.14116),
 * i.e. `OlsEngine<Radix2Fft<double>>` (proj/include/fcvbw/engine.hpp:28-192) and the block loop
 * of `fcvbw run` that drives it (proj/tools/fcvbw_cli.cpp:72-118). Paths are relative to the
 * reference root. All entry points are `extern "C"`, take plain pointers and sizes, and return a
 * status code mirroring the reference's error taxonomy and CLI exit codes
 * (proj/include/fcvbw/errors.hpp:7-29, proj/tools/fcvbw_cli.cpp:16-17,338-355):
 *
 *   FCVBW_GPU_OK          0   success
 *   FCVBW_GPU_ERROR       1   fcvbw::Error / any CUDA failure
 *   FCVBW_GPU_VALIDATION  2   fcvbw::ValidationError (documented precondition violated)
 *
 * The message of the most recent failure on the calling thread is returned by
 * fcvbw_gpu_last_error().
 *
 * Data layout: complex samples, interleaved (re, im); FCVBW_GPU_C64 = 2 x float32 per sample,
 * FCVBW_GPU_C128 = 2 x float64 per sample. Multichannel buffers are [channels][S] with an
 * explicit channel stride. Device pointers are CUDA device addresses on the engine's device.
 *
 * Threading (proj/include/fcvbw/engine.hpp:26-29; SPEC.md "independent engines may run in
 * parallel"): one handle is one stream, bound to one device, not re-entrant. Different handles
 * may be used concurrently from different host threads.
 */
#ifndef FCVBW_GPU_H
#define FCVBW_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FCVBW_GPU_OK 0
#define FCVBW_GPU_ERROR 1
#define FCVBW_GPU_VALIDATION 2
#define FCVBW_GPU_NONCONVERGENCE 3 /* fcvbw::NonConvergenceError (design side only) */
#define FCVBW_GPU_LP_ERROR 4       /* fcvbw::LpError (design side only) */

/* sample type of an engine */
#define FCVBW_GPU_C64 0  /* complex float32 */
#define FCVBW_GPU_C128 1 /* complex float64 */

/* fcvbw_gpu_config.flags */
#define FCVBW_GPU_FORCE_PHASE_MULTIPLY 1u /* multiply by phase_table even when L is odd */
#define FCVBW_GPU_TEST_CORRUPT_TWIDDLES 0x100u /* fault injection: corrupt one twiddle before the
                                                  construction self-check (tests only) */

/* fcvbw_gpu_run*() flags */
#define FCVBW_GPU_RUN_TRUSTED_SCHEDULE 1u /* skip the (synchronising) range check of a device b schedule */
#define FCVBW_GPU_RUN_PAIRED_SCHEDULES 2u /* run_real: rows 2i and 2i+1 of the schedule are identical */
#define FCVBW_GPU_RUN_ONE_BLOCK_PER_TRANSFORM 4u /* run_real: every real block in its own transform
                                                    (Im = 0; comparison runs and tests) */

typedef struct fcvbw_gpu_engine fcvbw_gpu_engine;

/* Structured engine configuration = BinSpec + TransitionProfile + initial b
 * (proj/include/fcvbw/spectrum.hpp:50-85; the field names follow the design artifact,
 * proj/include/fcvbw/io.hpp:34-47). */
typedef struct {
    int fft_length;            /* N = 2^Q, Q >= 3               (BinSpec::fft_length)          */
    int filter_length;         /* L, 1 <= L <= N                (BinSpec::filter_length)       */
    int block_length;          /* M = N - L + 1                 (BinSpec::block_length)        */
    int transition_width_bins; /* delta_N, even, >= 2           (BinSpec::transition_width_bins) */
    int b_low;                 /* delta_N/2 <= b_low <= b_high <= N/2 - delta_N/2 - 1          */
    int b_high;
    const double* profile;     /* V(r), profile_length = delta_N - 1 values (host memory)      */
    int profile_length;
    int initial_b;             /* OlsEngine(bins, profile, initial_b), engine.hpp:31           */
    int dtype;                 /* FCVBW_GPU_C64 | FCVBW_GPU_C128                               */
    int device;                /* CUDA device ordinal                                          */
    unsigned flags;            /* FCVBW_GPU_FORCE_PHASE_MULTIPLY                                */
} fcvbw_gpu_config;

/* ---------------------------------------------------------------- lifetime */

/* Replaces OlsEngine(const BinSpec&, TransitionProfile, int initial_b)
 * (engine.hpp:31-45) and new_engine(const DesignResult&, int) (design.hpp:579-582).
 * Validates exactly like BinSpec::validate (spectrum.hpp:63-76), the profile-length check
 * (engine.hpp:40-41) and set_bandwidth (engine.hpp:72-75). Then runs the construction-time
 * self-check, the GPU form of check_provider (engine.hpp:44,126-137): the seeded uniform(-1, 1)
 * vector (SeededRng(0x7ab1e5eed), N samples) goes through the engine's FFT plan and twiddle tables
 * with an all-pass table and must return within 1e-12 per sample (fp64; 1e-5 for FCVBW_GPU_C64),
 * else status 2 ("transform provider failed the round-trip check"). create_raw does the same
 * (engine.hpp:55). */
int fcvbw_gpu_create(const fcvbw_gpu_config* cfg, fcvbw_gpu_engine** out);

/* Replaces OlsEngine(DftCoefficients coeffs, int block_length) (engine.hpp:47-56): the classical
 * overlap-save filter with an arbitrary N-entry table (interleaved re/im doubles, host memory).
 * Requires N a power of two in [2, 8192] (Radix2Fft ctor, fft.hpp:35-38) and 1 <= M <= N
 * (engine.hpp:53). */
int fcvbw_gpu_create_raw(int fft_length, int block_length, const double* table, int dtype,
                         int device, fcvbw_gpu_engine** out);

void fcvbw_gpu_destroy(fcvbw_gpu_engine* h);

/* ---------------------------------------------------------------- accessors (engine.hpp:58-61) */
int fcvbw_gpu_block_length(const fcvbw_gpu_engine* h);
int fcvbw_gpu_fft_length(const fcvbw_gpu_engine* h);
int fcvbw_gpu_current_b(const fcvbw_gpu_engine* h);
int64_t fcvbw_gpu_blocks_processed(const fcvbw_gpu_engine* h);
int fcvbw_gpu_dtype(const fcvbw_gpu_engine* h);

/* ---------------------------------------------------------------- bandwidth (engine.hpp:70-80)
 * Index update only; takes effect at the next block boundary. Status 2 if b is outside
 * [b_low, b_high] or the engine is a raw-table engine. */
int fcvbw_gpu_set_bandwidth(fcvbw_gpu_engine* h, int b);

/* ---------------------------------------------------------------- streaming API
 * Host buffers, one channel, same semantics as the reference (bit-identical regardless of how
 * the caller batches its input, proj/tests/test_oracle_engine.cpp:268-288).
 *   reset          engine.hpp:63-67   zero history, drop pending input, blocks_processed = 0
 *   process_block  engine.hpp:82-88   exactly M samples in, M out; status 2 if n != M or input
 *                                     is pending
 *   feed           engine.hpp:92-103  any n; emits M samples per completed block
 *   flush          engine.hpp:107-115 zero-pads the pending partial block, emits only the
 *                                     samples that correspond to real input times
 * Outputs go to y_host (capacity y_cap samples); *n_out receives the number written. */
int fcvbw_gpu_reset(fcvbw_gpu_engine* h);
int fcvbw_gpu_process_block(fcvbw_gpu_engine* h, const void* x_host, int64_t n, void* y_host);
int fcvbw_gpu_feed(fcvbw_gpu_engine* h, const void* x_host, int64_t n, void* y_host, int64_t y_cap,
                   int64_t* n_out);
int fcvbw_gpu_flush(fcvbw_gpu_engine* h, void* y_host, int64_t y_cap, int64_t* n_out);

/* Real-valued streaming: the reference's own signatures (std::span<const double> in,
 * std::vector<double> out: engine.hpp:82,92,107) on REAL host samples of the engine's real type
 * (double for FCVBW_GPU_C128, float for FCVBW_GPU_C64). Structured engines carry consecutive real
 * blocks as the real and imaginary parts of one complex transform (exact: H is conjugate-
 * symmetric), so a real stream moves and transforms half the data of the complex entry points.
 * Semantics and statuses as feed / process_block / flush. An engine streams either real or
 * complex samples between resets (status 2 when a call mixes them). */
int fcvbw_gpu_feed_real(fcvbw_gpu_engine* h, const void* x_host, int64_t n, void* y_host, int64_t y_cap,
                        int64_t* n_out);
int fcvbw_gpu_process_block_real(fcvbw_gpu_engine* h, const void* x_host, int64_t n, void* y_host);
int fcvbw_gpu_flush_real(fcvbw_gpu_engine* h, void* y_host, int64_t y_cap, int64_t* n_out);

/* ---------------------------------------------------------------- instrumentation
 * The reference's OpCounters (ops.hpp:15-30) as analytic tallies of this engine's work since
 * creation, over every entry point: variable_mul = data-dependent real multiplications by the
 * transition profile V, 2 L_V per real block (exactly the reference's count, engine.hpp:150-153;
 * test_oracle_engine.cpp:229-240) and 4 L_V per complex block (two real streams); retune_flops =
 * floating-point operations spent by set_bandwidth, always 0 (test_oracle_engine.cpp:216-227). */
typedef struct fcvbw_gpu_ops {
    uint64_t variable_mul;
    uint64_t retune_flops;
    int64_t real_blocks;    /* real blocks processed (real entry points) */
    int64_t complex_blocks; /* complex blocks processed */
} fcvbw_gpu_ops;
int fcvbw_gpu_op_counts(const fcvbw_gpu_engine* h, fcvbw_gpu_ops* out);

/* ---------------------------------------------------------------- batched whole-stream run
 * Replaces the `fcvbw run` block loop (fcvbw_cli.cpp:95-113) over `channels` independent
 * streams of S samples each, in ONE fused kernel launch on `stream` (a cudaStream_t, 0 = legacy
 * default stream), asynchronous with respect to the host:
 *   - block m of channel c uses b = b_sched[c * b_channel_stride + m] (one entry per block, the
 *     schedule event applied before that block, fcvbw_cli.cpp:101-104); b_channel_stride = 0
 *     shares one schedule; b_sched = NULL uses current_b for every block;
 *   - the first block's history is zero (engine.hpp:119), the tail block is zero-padded and the
 *     output truncated to S samples (feed + flush, engine.hpp:107-115).
 * x_dev / y_dev: [channels][S] device buffers (channel stride S samples). The streaming state of
 * the handle is not touched. Unless FCVBW_GPU_RUN_TRUSTED_SCHEDULE is set, a device schedule is
 * range-checked first (a small kernel plus a synchronising 4-byte read) and status 2 is returned
 * if any b lies outside [b_low, b_high] (engine.hpp:72-75). */
int fcvbw_gpu_run(fcvbw_gpu_engine* h, const void* x_dev, int64_t S, int channels,
                  const int32_t* b_sched_dev, int64_t b_channel_stride, void* y_dev, void* stream,
                  unsigned flags);

/* Sharding primitive: global blocks [blk_begin, blk_end) of every channel. Input sample i of
 * channel c is read from x_dev[c * x_channel_stride + (i - x_first)] for
 * i in [max(0, blk_begin*M - (N - M)), min(S, blk_end*M)) (the (N - M)-sample halo included);
 * output sample i goes to y_dev[c * y_channel_stride + (i - y_first)] for
 * i in [blk_begin*M, min(S, blk_end*M)). The b schedule is indexed by GLOBAL block number.
 * Output is bit-identical to the corresponding slice of fcvbw_gpu_run. */
int fcvbw_gpu_run_range(fcvbw_gpu_engine* h, const void* x_dev, int64_t x_first,
                        int64_t x_channel_stride, int64_t S, int channels,
                        const int32_t* b_sched_dev, int64_t b_channel_stride, void* y_dev,
                        int64_t y_first, int64_t y_channel_stride, int64_t blk_begin,
                        int64_t blk_end, void* stream, unsigned flags);

/* Real-input fast path (the reference's native signature is real: engine.hpp:82,92). x_dev / y_dev
 * are REAL [channels][S] device buffers of the engine's real type (float for FCVBW_GPU_C64, double
 * for FCVBW_GPU_C128). For a structured engine, blocks 2p and 2p+1 of each channel are carried as
 * the real and imaginary parts of ONE complex transform — exact, because every structured H(k) is
 * conjugate-symmetric — so a real stream costs half the transforms of a complex one; when the two
 * blocks use different b the spectrum is combined as Z (H0 + H1)/2 + conj(Z(N-k)) (H0 - H1)/2
 * (one extra shared-memory exchange, no second transform). FCVBW_GPU_RUN_ONE_BLOCK_PER_TRANSFORM
 * runs every real block as its own transform with a zero imaginary part instead. Raw-table
 * engines (possibly asymmetric tables: the reference keeps Re(IFFT), fft.hpp:68-78) always run
 * one real block per transform. Same launch / validation semantics as fcvbw_gpu_run
 * (FCVBW_GPU_RUN_PAIRED_SCHEDULES is accepted and ignored). */
int fcvbw_gpu_run_real(fcvbw_gpu_engine* h, const void* x_dev, int64_t S, int channels,
                       const int32_t* b_sched_dev, int64_t b_channel_stride, void* y_dev, void* stream,
                       unsigned flags);

/* Host-memory whole-stream run (what `fcvbw run` does with its in-memory signal): the same
 * semantics as fcvbw_gpu_run, with host->device copies, the fused kernel and device->host copies
 * pipelined over block chunks on several CUDA streams. Pinned (page-locked) host buffers give
 * full PCIe bandwidth. The schedule is host memory and is range-checked on the host (status 2).
 * Synchronous: returns when y_host is complete. */
int fcvbw_gpu_run_host(fcvbw_gpu_engine* h, const void* x_host, int64_t S, int channels,
                       const int32_t* b_sched_host, int64_t b_channel_stride, void* y_host);

/* Host-memory real-input run: fcvbw_gpu_run_real semantics on REAL host buffers [channels][S]
 * (float / double per the engine dtype), pipelined like fcvbw_gpu_run_host. This is the
 * reference's own call shape (`fcvbw run` on a real signal) at half the PCIe bytes and half the
 * transforms of carrying the signal as complex. Synchronous. */
int fcvbw_gpu_run_real_host(fcvbw_gpu_engine* h, const void* x_host, int64_t S, int channels,
                            const int32_t* b_sched_host, int64_t b_channel_stride, void* y_host);

/* ---------------------------------------------------------------- parity / introspection
 * Per-(block, bin) coefficient masks produced by the kernel's own coefficient generator for the
 * n_b band centres in b_host, written row-major [n_b][N] to host memory (any output may be NULL):
 *   region[k]  0 passband, 1 transition, 2 stopband             (bin_region, spectrum.hpp:194-202)
 *   v_index[k] r in [0, delta_N - 2] on transition bins, else -1 (magnitude_samples, :170-192)
 *   H[2k..2k+1] magnitude[k] * phase[k] in fp64              (assemble_dft_coefficients, :221-242)
 * Structured engines only (status 2 otherwise, or if a b is outside [b_low, b_high]). */
int fcvbw_gpu_coeff_dump(fcvbw_gpu_engine* h, const int32_t* b_host, int n_b, int8_t* region,
                         int16_t* v_index, double* H);

/* The mask the PRODUCTION kernel applies: n_b blocks, block m using b_host[m], run through the same
 * fused-kernel instantiation as fcvbw_gpu_run with its dump pointer set; g_out[m * N + k] receives
 * the real factor g(k)/N that multiplies bin k (1/N in the passband, V[f - k1]/N on transition
 * bins, 0 in the stopband; f = min(k, N - k)), in the engine's precision, widened exactly to
 * double. Equals magnitude_samples(bins, V, b)[k] / N (spectrum.hpp:170-192) rounded to the engine
 * type, bit for bit. Structured engines only. */
int fcvbw_gpu_mask_dump(fcvbw_gpu_engine* h, const int32_t* b_host, int n_b, double* g_out);

/* ---------------------------------------------------------------- synthetic workload
 * Bench / test utility (no reference counterpart): fills [channels][S] complex samples (channel
 * stride ch_stride samples) of dtype on the current device with the seeded unit-variance complex
 * Gaussian of paper_2406_14116_b200/workload.py: channel c uses seed seed_base + ch_first + c,
 * sample index start + i. Asynchronous on `stream`. */
int fcvbw_gpu_fill_gaussian(void* x_dev, int dtype, int64_t S, int channels, int64_t ch_stride,
                            uint64_t seed_base, int64_t ch_first, int64_t start, void* stream);

/* ---------------------------------------------------------------- design verification
 * Dense-grid worst-case error of a design, on the GPU: the reference's
 * `verify(const DesignResult&, int dense_points, double delta_e)` (proj/include/fcvbw/design.hpp:
 * 601-673; report fields :584-597). `fcvbw_gpu_design` carries the DesignResult fields verify reads
 * (design.hpp:463-472: bins, profile, delta, grid_points, facets). The PTVIR shift rule is passed
 * explicitly as (window_offset, step) — the rule `calibrated_shift_rule` measures for the
 * overlap-save engine is (1 - M, +1) (ptvir.hpp:52-56); other offsets are rejected (status 2),
 * step must be +-1. Outputs: per_b_max[b - b_low] (may be NULL; the reference's per_b_max map),
 * per_n_max[M] (may be NULL), and the scalar report. fp64 throughout. */
typedef struct fcvbw_gpu_design {
    int32_t fft_length, filter_length, block_length, transition_width_bins, b_low, b_high;
    const double* profile; /* V, delta_N - 1 values, host memory */
    int32_t profile_length;
    double delta;        /* achieved design-grid error (DesignResult::delta) */
    int32_t grid_points; /* K of the design grid */
    int32_t facets;      /* P of the SOCP linearisation */
} fcvbw_gpu_design;

typedef struct fcvbw_gpu_verification {
    double delta; /* dense-grid worst case over all (n, b) */
    double passband_max, stopband_max;
    int32_t dense_points, worst_b, worst_n;
    double worst_omega;
    int32_t pass;
    double refinement_bound; /* delta_design * sec(pi/P) + 1e-9 */
    int32_t within_bound;
} fcvbw_gpu_verification;

int fcvbw_gpu_verify(const fcvbw_gpu_design* design, int dense_points, double delta_e, int window_offset,
                     int step, int device, double* per_b_max, double* per_n_max,
                     fcvbw_gpu_verification* report);

/* Same contract, evaluated the reference's way (one length-N sum per (b, n, omega) in the
 * reference's operation order, glibc's hypot): every report field bit-identical to the reference's
 * verify(). O(num_b K M N) instead of fcvbw_gpu_verify's O(num_b K (N + M)). */
int fcvbw_gpu_verify_exact(const fcvbw_gpu_design* design, int dense_points, double delta_e, int window_offset,
                           int step, int device, double* per_b_max, double* per_n_max,
                           fcvbw_gpu_verification* report);

/* ---------------------------------------------------------------- shift-rule calibration
 * `calibrated_shift_rule(bins)` (proj/include/fcvbw/design.hpp:476-484) with this library's
 * overlap-save engine as the probed BlockProcessor: impulse probes of every input phase (one
 * batched launch), then `calibrate_shift_convention` (ptvir.hpp:225-294) — support windows,
 * measure_ptvir's energy and superposition checks, per-row circular-shift fit (on the device).
 * Writes the ShiftRule (window_offset, step) the design / verify / analyze entry points take.
 * Uses the geometry fields of `design` only. Status 1 if the measurements fit no affine rule. */
int fcvbw_gpu_calibrate_shift(const fcvbw_gpu_design* design, int device, int* window_offset, int* step);

/* ---------------------------------------------------------------- minimax design
 * The reference's cutting-plane exchange `solve_minimax(const DesignProblem&, const ShiftRule&)`
 * (proj/include/fcvbw/design.hpp:276-446) for one BinSpec — what `design()` runs per candidate
 * order (design.hpp:486-577; the order loop itself is host-side, paper_2406_14116_b200/design.py).
 * Constraint assembly and the dense true-error sweep run on the GPU; the LP
 * (ChebyshevLpSolver, lp.hpp:32-208) on the host. `geometry` supplies the BinSpec (its profile,
 * delta, grid_points and facets fields are ignored); options mirror DesignOptions
 * (design.hpp:452-461). The designed profile (delta_N - 1 values) is written to v_out.
 * Status: 2 validation, 3 NonConvergenceError, 4 LpError, 1 other. */
typedef struct fcvbw_gpu_solve_options {
    int32_t grid_points; /* K (>= 2N) */
    int32_t facets;      /* P (even, >= 8) */
    double exchange_tol;
    int32_t max_rounds;
    int32_t seed_stride;
} fcvbw_gpu_solve_options;

typedef struct fcvbw_gpu_solve_result {
    double delta;    /* true worst case over the design grid (SolveOutcome::delta) */
    double lp_delta; /* optimum of the final polyhedral LP */
    int32_t rounds;
    int64_t lp_iterations;
    int64_t active_triples;
    int64_t lp_rows;
    int64_t grid_size; /* K' = K plus inserted band edges */
    double seconds_tables, seconds_assembly, seconds_lp, seconds_sweep; /* host wall time per phase */
} fcvbw_gpu_solve_result;

int fcvbw_gpu_solve_minimax(const fcvbw_gpu_design* geometry, const fcvbw_gpu_solve_options* options, int step,
                            int device, double* v_out, fcvbw_gpu_solve_result* result);

/* ---------------------------------------------------------------- design analysis
 * The data behind `fcvbw analyze` (proj/tools/fcvbw_cli.cpp:120-193), `error_on_grid`
 * (proj/include/fcvbw/ptvir.hpp:402-431) and `ptvir_from_base` (ptvir.hpp:147-160) for a design
 * (bins + profile in `design`; delta / grid_points / facets unused). `step` is the PTVIR shift step
 * (+1 for the overlap-save engine, see fcvbw_gpu_verify).
 *
 * fcvbw_gpu_frequency_grid: FrequencyGrid::build (ptvir.hpp:309-343) — *size = K'; omega (capacity
 *   entries, may be NULL) receives the sorted grid.
 * fcvbw_gpu_ptvir: the M x N PTVIR table of band centre b, row-major (write_ptvir_csv layout,
 *   io.hpp:251-260).
 * fcvbw_gpu_analyze: for each b in b_list (nb entries) and each grid point g, over the M phases:
 *   h_max / h_min = max / min |H_n(omega_g)|, e_max = max |H_n - H_desired| (NaN on excluded
 *   transition-band points); layout [nb][K']. abs_h / abs_e (may be NULL) receive the per-phase
 *   values [nb][K'][M] (abs_e NaN when excluded). */
int fcvbw_gpu_frequency_grid(const fcvbw_gpu_design* design, int grid_points, double* omega, int64_t capacity,
                             int64_t* size);
int fcvbw_gpu_ptvir(const fcvbw_gpu_design* design, int b, int step, int device, double* rows);
int fcvbw_gpu_analyze(const fcvbw_gpu_design* design, int grid_points, const int32_t* b_list, int nb, int step,
                      int device, double* h_max, double* h_min, double* e_max, double* abs_h, double* abs_e);

/* Number of fused-kernel launches issued by this handle since creation (bench bookkeeping). */
int64_t fcvbw_gpu_kernel_launches(const fcvbw_gpu_engine* h);

/* Message for the last failure on the calling thread ("" if none). */
const char* fcvbw_gpu_last_error(void);

/* Library version string. */
const char* fcvbw_gpu_version(void);

#ifdef __cplusplus
}
#endif

#endif /* FCVBW_GPU_H */
