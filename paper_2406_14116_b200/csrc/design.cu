// GPU-assisted minimax design of the transition-band profile V:
// the reference's cutting-plane exchange `solve_minimax` (proj/include/fcvbw/design.hpp:276-446)
// with its two O(N)-per-point inner kernels moved to the B200:
//   * constraint assembly `append_constraints` (design.hpp:121-153): one length-N response sum
//     per (active triple, affine table), and the PTVIR base rows `band_tables` (:105-116);
//   * the dense true-error sweep `sweep_true_error` (design.hpp:203-269): one length-N response
//     sum per (b, n, omega) — O(num_b K M N) per exchange round.
// The LP (`ChebyshevLpSolver`, proj/include/fcvbw/lp.hpp:32-208) and the exchange bookkeeping stay on
// the host, restated below.
//
// Bit-compatibility: the device evaluates every response in the reference's summation order with
// explicit round-to-nearest multiplies and adds (no FMA contraction), from phasor / root / phase
// tables computed by host libm exactly as the reference computes them (grid.h). The affine
// constraint data c, a (and therefore every LP solve) are bit-identical to the reference's, and the
// sweep's |E| uses a restatement of glibc's hypot (response.cuh), so the sweep maxima, thresholds
// and the reported delta are too. tests/test_design.py compares V, delta, rounds and LP iteration
// counts with the reference's.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <chrono>
#include <functional>
#include <thread>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <string>
#include <tuple>
#include <unordered_set>
#include <vector>

#include "../../include/fcvbw_gpu.h"
#include "grid.h"
#include "response.cuh"

namespace fcvbw_gpu_detail {
void set_last_error(const std::string& m);
}

namespace design_impl {

using namespace fcvbw_grid;
using namespace fcvbw_resp;

struct Failure {
    int code;
    std::string msg;
};
[[noreturn]] void validation(const std::string& m) { throw Failure{FCVBW_GPU_VALIDATION, m}; }
[[noreturn]] void nonconvergence(const std::string& m) { throw Failure{FCVBW_GPU_NONCONVERGENCE, m}; }
[[noreturn]] void lp_error(const std::string& m) { throw Failure{FCVBW_GPU_LP_ERROR, m}; }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Failure{FCVBW_GPU_ERROR, std::string(what) + ": " + cudaGetErrorString(e)};
}

template <class T>
struct Dev {
    T* p = nullptr;
    size_t n = 0;
    Dev() = default;
    explicit Dev(size_t count) { resize(count); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    ~Dev() { cudaFree(p); }
    void resize(size_t count) {
        if (count <= n && p) return;
        cudaFree(p);
        p = nullptr;
        n = std::max<size_t>(1, count);
        ck(cudaMalloc(&p, sizeof(T) * n), "cudaMalloc");
    }
    void put(const T* h, size_t count) { ck(cudaMemcpy(p, h, sizeof(T) * count, cudaMemcpyHostToDevice), "H2D"); }
    void get(T* h, size_t count) const { ck(cudaMemcpy(h, p, sizeof(T) * count, cudaMemcpyDeviceToHost), "D2H"); }
};

// ------------------------------------------------------------------------------------ device
// cmul_x, base_rows_kernel, row_response: response.cuh

struct TripleDev {
    int n, bi, gi, pad;
};

// append_constraints (design.hpp:121-153): one warp per triple, lane j = affine table j of the
// triple's band (j = 0: F, j = 1..lv: G_{j-1}); c = H_F - desired, a_r = H_{G_r}.
__global__ void assemble_kernel(int N, int M, int lv, int step, int ntr, const TripleDev* __restrict__ tr,
                                const double* __restrict__ band_base /* [num_b][lv + 1][N] */,
                                const double2* __restrict__ ph /* [K'][N] */, const double2* __restrict__ des_pass,
                                const double* __restrict__ omega, int blo, double delta, double2* c, double2* a) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= ntr) return;
    const TripleDev t = tr[warp];
    const int shift = step * (t.n - (M - 1));
    const double2* phg = ph + size_t(t.gi) * N;
    const double2 pre = phg[t.n];
    for (int j = lane; j <= lv; j += 32) {
        const double2 h = row_response(band_base + (size_t(t.bi) * (lv + 1) + j) * N, N, shift, phg, pre);
        if (j == 0) {
            // desired_response (ptvir.hpp:368-381): passband iff omega <= b_omega - delta/2 + 1e-12
            const double b_omega = (blo + t.bi) * 2.0 * kPi / N;
            const double w = omega[t.gi];
            double2 d = make_double2(0.0, 0.0);
            if (w <= __dadd_rn(__dsub_rn(b_omega, delta / 2.0), 1e-12)) d = des_pass[t.gi];
            c[warp] = make_double2(__dsub_rn(h.x, d.x), __dsub_rn(h.y, d.y));
        } else {
            a[size_t(warp) * lv + (j - 1)] = h;
        }
    }
}

struct Hit {
    double err;
    int bi, n, gi, pad;
};

// sweep_true_error (design.hpp:203-269), evaluation half: |E| for every (b in batch, omega, n);
// -1 marks excluded points. Points above `thr` are appended to `hits` (order irrelevant: the host
// sorts them by a total key).
__global__ void sweep_eval_kernel(int N, int M, int step, int kk, int g0, int bi0, const double* __restrict__ base /* [nb][N] */,
                                  const double2* __restrict__ ph, const double2* __restrict__ des_pass,
                                  const double* __restrict__ omega, const int8_t* __restrict__ region /* [num_b][K'] */,
                                  int blo, double delta, double thr, double* err_out /* [nb][K'][M] */,
                                  Hit* hits, unsigned long long* nhits, unsigned long long cap) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    const int gi = g0 + blockIdx.y;
    const int bl = blockIdx.z, bi = bi0 + bl;
    if (n >= M) return;
    double* out = err_out + (size_t(bl) * kk + gi) * M + n;
    const int reg = region[size_t(bi) * kk + gi];
    if (reg == 2) {
        *out = -1.0;
        return;
    }
    const double2* phg = ph + size_t(gi) * N;
    const double2 h = row_response(base + size_t(bl) * N, N, step * (n - (M - 1)), phg, phg[n]);
    const double b_omega = (blo + bi) * 2.0 * kPi / N;
    double2 d = make_double2(0.0, 0.0);
    if (omega[gi] <= __dadd_rn(__dsub_rn(b_omega, delta / 2.0), 1e-12)) d = des_pass[gi];
    const double err = glibc_hypot(__dsub_rn(h.x, d.x), __dsub_rn(h.y, d.y));
    *out = err;
    if (err > thr) {
        const unsigned long long slot = atomicAdd(nhits, 1ull);
        if (slot < cap) hits[slot] = Hit{err, bi, n, gi, 0};
    }
}

// sweep_true_error, reduction half: per (b, n) the first grid index attaining the maximum
// (strict >, omega ascending, starting from max_abs = -1), as SweepCell (design.hpp:184-187).
// With `region` non-null also the passband / stopband maxima per (b, n) (verify, design.hpp:637-641).
__global__ void sweep_reduce_kernel(int M, int kk, int nb, int bi0, const double* __restrict__ err,
                                    double* cell_max, int* cell_gi, const int8_t* __restrict__ region,
                                    double* cell_pass, double* cell_stop) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    const int bl = blockIdx.y;
    if (n >= M || bl >= nb) return;
    double best = -1.0, pass = 0.0, stop = 0.0;
    int arg = -1;
    const double* e = err + size_t(bl) * kk * M + n;
    const int8_t* reg = region ? region + size_t(bi0 + bl) * kk : nullptr;
    for (int g = 0; g < kk; ++g) {
        const double v = e[size_t(g) * M];
        if (v >= 0.0 && v > best) {
            best = v;
            arg = g;
        }
        if (reg && v >= 0.0) {
            if (reg[g] == 0)
                pass = fmax(pass, v);
            else
                stop = fmax(stop, v);
        }
    }
    cell_max[size_t(bi0 + bl) * M + n] = best;
    cell_gi[size_t(bi0 + bl) * M + n] = arg;
    if (reg) {
        cell_pass[size_t(bi0 + bl) * M + n] = pass;
        cell_stop[size_t(bi0 + bl) * M + n] = stop;
    }
}

struct Violation {
    double amount;
    int64_t triple;
    int facet, pad;
};

// The violation scan of solve_minimax's lazy row generation (design.hpp:378-393) for every active
// triple: E = c + sum_r v_r a_r (ConstraintSystem::error_at order), skip |E|^2 <= reject, then every
// facet not yet in the LP whose value exceeds delta + 1e-11. Counts the violations with
// amount >= thr (and their maximum); collects them when `out` is non-null.
__global__ void violation_scan_kernel(int64_t ntr, int lv, int facets, const double* __restrict__ v,
                                      const double2* __restrict__ c, const double2* __restrict__ a,
                                      const uint8_t* __restrict__ added, const double* __restrict__ cos_f,
                                      const double* __restrict__ sin_f, double reject, double lim, double lp_delta,
                                      double thr, unsigned long long* count, unsigned long long* max_bits,
                                      Violation* out, unsigned long long cap) {
    const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (t >= ntr) return;
    double2 e = c[t];
    const double2* at = a + t * lv;
    for (int r = 0; r < lv; ++r) {
        const double2 ar = at[r];
        e.x = __dadd_rn(e.x, __dmul_rn(v[r], ar.x));
        e.y = __dadd_rn(e.y, __dmul_rn(v[r], ar.y));
    }
    if (__dadd_rn(__dmul_rn(e.x, e.x), __dmul_rn(e.y, e.y)) <= reject) return;
    const uint8_t* ad = added + t * facets;
    for (int p = 0; p < facets; ++p) {
        if (ad[p]) continue;
        const double value = __dsub_rn(__dmul_rn(cos_f[p], e.x), __dmul_rn(sin_f[p], e.y));
        if (value > lim) {
            const double amount = __dsub_rn(value, lp_delta);
            if (amount >= thr) {
                atomicMax(max_bits, static_cast<unsigned long long>(__double_as_longlong(amount)));
                const unsigned long long slot = atomicAdd(count, 1ull);
                if (out && slot < cap) out[slot] = Violation{amount, t, p, 0};
            }
        }
    }
}

__global__ void mark_added_kernel(int n, const int64_t* __restrict__ idx, uint8_t* added) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) added[idx[i]] = 1;
}

// ------------------------------------------------------------------------------------ host
// SeededRng (proj/include/fcvbw/ops.hpp:62-86)
struct Rng {
    uint64_t s;
    explicit Rng(uint64_t seed) : s(seed ? seed : 0x9e3779b97f4a7c15ULL) {}
    uint64_t next() {
        uint64_t x = s;
        x ^= x >> 12;
        x ^= x << 25;
        x ^= x >> 27;
        s = x;
        return x * 0x2545F4914F6CDD1DULL;
    }
    double uniform(double lo, double hi) { return lo + (hi - lo) * (static_cast<double>(next() >> 11) * 0x1.0p-53); }
};

struct Triple {
    int n, b, gi;
};

struct Clock {
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    double lap() {
        const auto t = std::chrono::steady_clock::now();
        const double s = std::chrono::duration<double>(t - t0).count();
        t0 = t;
        return s;
    }
};
inline bool by_bng(const Triple& x, const Triple& y) {
    return std::tie(x.b, x.n, x.gi) < std::tie(y.b, y.n, y.gi);
}
inline uint64_t key_of(const Triple& t) {
    return (uint64_t(uint32_t(t.b)) << 44) ^ (uint64_t(uint32_t(t.n)) << 28) ^ uint64_t(uint32_t(t.gi));
}

// ChebyshevLpSolver (lp.hpp:32-208): minimise delta s.t. a.v - gamma delta <= beta, solved on the
// dual by a two-phase revised simplex on a dense (nv+1)^2 basis inverse; Dantzig pricing with a
// Bland fallback after 64 stalled pivots; ties to the lowest index.
struct LpRows {
    int nv = 0;
    std::vector<double> a, gamma, beta;
    int size() const { return int(beta.size()); }
    void push(const double* row, double g, double bt) {
        a.insert(a.end(), row, row + nv);
        gamma.push_back(g);
        beta.push_back(bt);
    }
};

struct LpSolution {
    std::vector<double> v;
    double delta = 0.0;
    int iterations = 0;
};

// Small persistent worker pool for the LP's pricing loop (one short job per simplex iteration).
// Small worker pool for the LP pricing loop. Workers spin briefly after each job (pricing calls
// arrive back to back within one LP solve), then block on a condition variable, so idle workers
// cost no CPU between LP iterations, during the device phases, or after the solve.
class SpinPool {
  public:
    explicit SpinPool(int n) : n_(std::max(1, n)) {
        for (int t = 1; t < n_; ++t) th_.emplace_back([this, t] { loop(t); });
    }
    ~SpinPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_.store(true, std::memory_order_release);
            gen_.fetch_add(1, std::memory_order_acq_rel);
        }
        cv_.notify_all();
        for (auto& x : th_) x.join();
    }
    int size() const { return n_; }
    template <class F>
    void run(F&& f) {  // f(t) for t in [0, n); returns when all are done
        job_ = std::function<void(int)>(std::forward<F>(f));
        done_.store(0, std::memory_order_release);
        {
            std::lock_guard<std::mutex> lk(mu_);
            gen_.fetch_add(1, std::memory_order_acq_rel);
        }
        cv_.notify_all();
        job_(0);
        while (done_.load(std::memory_order_acquire) < n_ - 1) std::this_thread::yield();
    }

  private:
    static constexpr int kSpin = 4096;  // polls before blocking (a few tens of microseconds)
    void loop(int t) {
        unsigned seen = 0;
        for (;;) {
            unsigned g = gen_.load(std::memory_order_acquire);
            for (int i = 0; g == seen && i < kSpin; ++i) {
                std::this_thread::yield();
                g = gen_.load(std::memory_order_acquire);
            }
            if (g == seen) {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_.load(std::memory_order_acquire) != seen; });
                g = gen_.load(std::memory_order_acquire);
            }
            seen = g;
            if (stop_.load(std::memory_order_acquire)) return;
            job_(t);
            done_.fetch_add(1, std::memory_order_acq_rel);
        }
    }
    int n_;
    std::vector<std::thread> th_;
    std::function<void(int)> job_;
    std::atomic<unsigned> gen_{0};
    std::atomic<int> done_{0};
    std::atomic<bool> stop_{false};
    std::mutex mu_;
    std::condition_variable cv_;
};

class ChebyshevLp {
  public:
    explicit ChebyshevLp(int nv) : nv_(nv), m_(nv + 1) {}
    // Pricing over the columns is split into contiguous ranges across `pool` when the LP is large;
    // each range keeps the first minimum (Dantzig) / first candidate (Bland) and the ranges are
    // merged by (reduced cost, index), so the entering column is the sequential loop's.
    void set_pool(SpinPool* pool) { pool_ = pool; }

    LpSolution solve(const LpRows& rows) const {
        const int cols = rows.size();
        if (cols == 0) lp_error("lp: empty constraint set");
        std::vector<int> basis(m_);
        std::vector<double> binv(size_t(m_) * m_, 0.0), xb(m_, 0.0);
        for (int i = 0; i < m_; ++i) {
            basis[i] = cols + i;
            binv[size_t(i) * m_ + i] = 1.0;
        }
        xb[m_ - 1] = 1.0;
        int iterations = 0;
        phase(rows, basis, binv, xb, true, iterations);
        double infeas = 0.0;
        for (int i = 0; i < m_; ++i)
            if (basis[i] >= cols) infeas += xb[i];
        if (infeas > 1e-9) lp_error("lp: dual infeasible (primal unbounded); constraint set too thin");
        phase(rows, basis, binv, xb, false, iterations);

        std::vector<double> y(m_);
        multipliers(rows, basis, binv, false, y);
        LpSolution sol;
        sol.iterations = iterations;
        sol.v.assign(y.begin(), y.begin() + nv_);
        sol.delta = -y[m_ - 1];
        double scale = 1.0 + std::abs(sol.delta);
        for (int r = 0; r < cols; ++r) scale = std::max(scale, std::abs(rows.beta[r]));
        for (int r = 0; r < cols; ++r) {
            double lhs = -rows.gamma[r] * sol.delta;
            const double* ar = rows.a.data() + size_t(r) * nv_;
            for (int j = 0; j < nv_; ++j) lhs += ar[j] * sol.v[j];
            if (lhs > rows.beta[r] + 1e-7 * scale) lp_error("lp: recovered primal violates a constraint");
        }
        return sol;
    }

  private:
    double cost(const LpRows& rows, int col, bool phase1) const {
        const int cols = rows.size();
        if (phase1) return col >= cols ? 1.0 : 0.0;
        return col >= cols ? 0.0 : rows.beta[col];
    }

    void multipliers(const LpRows& rows, const std::vector<int>& basis, const std::vector<double>& binv, bool phase1,
                     std::vector<double>& y) const {
        for (int j = 0; j < m_; ++j) {
            double acc = 0.0;
            for (int i = 0; i < m_; ++i) acc += cost(rows, basis[i], phase1) * binv[size_t(i) * m_ + j];
            y[j] = acc;
        }
    }

    void phase(const LpRows& rows, std::vector<int>& basis, std::vector<double>& binv, std::vector<double>& xb,
               bool phase1, int& iterations) const {
        const int cols = rows.size();
        const long cap = 50000 + 256L * (cols + m_);
        std::vector<double> y(m_), u(m_), column(m_);
        auto objective = [&] {
            double acc = 0.0;
            for (int i = 0; i < m_; ++i) acc += cost(rows, basis[i], phase1) * xb[i];
            return acc;
        };
        double last = objective();
        int stall = 0;
        for (long iter = 0;; ++iter) {
            if (iter > cap) lp_error("lp: iteration cap exceeded");
            ++iterations;
            multipliers(rows, basis, binv, phase1, y);
            const bool bland = stall > 64;
            auto price = [&](int j0, int j1, int& ent, double& best) {
                ent = -1;
                best = -1e-10;
                for (int j = j0; j < j1; ++j) {
                    double rc = cost(rows, j, phase1);
                    const double* aj = rows.a.data() + size_t(j) * nv_;
                    for (int i = 0; i < nv_; ++i) rc -= y[i] * aj[i];
                    rc -= y[m_ - 1] * rows.gamma[j];
                    if (rc < best) {
                        ent = j;
                        if (bland) break;
                        best = rc;
                    }
                }
            };
            int entering = -1;
            if (pool_ && pool_->size() > 1 && cols >= 2048) {
                const int nt = pool_->size();
                std::vector<int> ent(nt);
                std::vector<double> best(nt);
                pool_->run([&](int t) {
                    const int j0 = int(int64_t(cols) * t / nt), j1 = int(int64_t(cols) * (t + 1) / nt);
                    price(j0, j1, ent[t], best[t]);
                });
                double most_negative = -1e-10;
                for (int t = 0; t < nt; ++t) {  // ranges ascending: first hit / strict minimum wins
                    if (ent[t] < 0) continue;
                    if (bland) {
                        entering = ent[t];
                        break;
                    }
                    if (best[t] < most_negative) {
                        most_negative = best[t];
                        entering = ent[t];
                    }
                }
            } else {
                double most_negative;
                price(0, cols, entering, most_negative);
            }
            if (entering < 0) return;
            const double* ae = rows.a.data() + size_t(entering) * nv_;
            for (int i = 0; i < nv_; ++i) column[i] = ae[i];
            column[m_ - 1] = rows.gamma[entering];
            for (int i = 0; i < m_; ++i) {
                double acc = 0.0;
                for (int j = 0; j < m_; ++j) acc += binv[size_t(i) * m_ + j] * column[j];
                u[i] = acc;
            }
            int leaving = -1;
            double best = std::numeric_limits<double>::infinity();
            for (int i = 0; i < m_; ++i) {
                if (u[i] > 1e-11) {
                    const double ratio = xb[i] / u[i];
                    if (ratio < best || (ratio == best && (leaving < 0 || basis[i] < basis[leaving]))) {
                        best = ratio;
                        leaving = i;
                    }
                }
            }
            if (leaving < 0) lp_error("lp: dual unbounded (primal infeasible)");
            const double pivot = u[leaving];
            for (int j = 0; j < m_; ++j) binv[size_t(leaving) * m_ + j] /= pivot;
            xb[leaving] /= pivot;
            for (int i = 0; i < m_; ++i) {
                if (i == leaving || u[i] == 0.0) continue;
                const double f = u[i];
                for (int j = 0; j < m_; ++j) binv[size_t(i) * m_ + j] -= f * binv[size_t(leaving) * m_ + j];
                xb[i] -= f * xb[leaving];
                if (xb[i] < 0.0 && xb[i] > -1e-12) xb[i] = 0.0;
            }
            basis[leaving] = entering;
            const double now = objective();
            if (now < last - 1e-15 * (1.0 + std::abs(last))) {
                stall = 0;
                last = now;
            } else {
                ++stall;
            }
        }
    }

    int nv_, m_;
    SpinPool* pool_ = nullptr;
};

// The design problem on the device: grid, phasors, desired responses and per-band affine bases.
struct Problem {
    int N, L, M, dn, blo, bhi, num_b, lv, step;
    double delta;  // BinSpec::delta()
    Grid grid;
    std::vector<cd> phase, roots;
    Dev<double2> ph, des_pass, d_roots;
    Dev<double> d_omega;
    Dev<int8_t> d_region;
    Dev<double> band_base;  // [num_b][lv + 1][N]
    Dev<double2> tables;    // scratch: coefficient tables
    Dev<double> base;       // scratch: base rows of a profile
    Dev<int> bad;

    double omega_of_bin(int b) const { return b * 2.0 * kPi / N; }

    void assemble_table(const double* v, int b, cd* out) const {
        fcvbw_grid::assemble_table(N, dn, b, v, phase, out);
    }

    void base_rows(int T, const std::vector<cd>& tabs, double* dst) {
        tables.resize(size_t(T) * N);
        tables.put(reinterpret_cast<const double2*>(tabs.data()), size_t(T) * N);
        ck(cudaMemset(bad.p, 0, sizeof(int)), "memset");
        base_rows_kernel<<<dim3((N + 127) / 128, T), 128>>>(N, T, tables.p, d_roots.p, dst, bad.p);
        ck(cudaGetLastError(), "base_rows_kernel");
        int flag = 0;
        bad.get(&flag, 1);
        if (flag) validation("base_response_idft: table is not conjugate-symmetric");
    }

    // band_tables (design.hpp:105-116) for every b: F = assemble(zeros), G_r = phase on k1 + r and N - k1 - r
    void build_band_tables() {
        const size_t per_b = size_t(lv + 1) * N;
        band_base.resize(size_t(num_b) * per_b);
        const int batch = int(std::max<size_t>(1, (size_t(256) << 20) / (per_b * sizeof(cd))));
        std::vector<double> zeros(size_t(lv), 0.0);
        for (int b0 = 0; b0 < num_b; b0 += batch) {
            const int nb = std::min(batch, num_b - b0);
            std::vector<cd> tabs(size_t(nb) * per_b, cd{0.0, 0.0});
            for (int i = 0; i < nb; ++i) {
                const int b = blo + b0 + i;
                cd* t = tabs.data() + size_t(i) * per_b;
                assemble_table(zeros.data(), b, t);
                const int k1 = b - dn / 2 + 1;
                for (int r = 0; r < lv; ++r) {
                    cd* g = t + size_t(r + 1) * N;
                    g[k1 + r] = phase[k1 + r];
                    g[N - (k1 + r)] = phase[N - (k1 + r)];
                }
            }
            base_rows(int(nb * (lv + 1)), tabs, band_base.p + size_t(b0) * per_b);
        }
    }
};

// Device mirror of the constraint system (c, a and the per-(triple, facet) "row added" flags) for
// the violation scan; grows geometrically.
struct DevSystem {
    int lv = 0, facets = 0;
    size_t size = 0, cap = 0;
    double2 *c = nullptr, *a = nullptr;
    uint8_t* added = nullptr;
    ~DevSystem() {
        cudaFree(c);
        cudaFree(a);
        cudaFree(added);
    }
    void reserve(size_t n) {
        if (n <= cap) return;
        const size_t nc = std::max(n, cap * 2);
        double2 *c2, *a2;
        uint8_t* ad2;
        ck(cudaMalloc(&c2, sizeof(double2) * nc), "cudaMalloc c");
        ck(cudaMalloc(&a2, sizeof(double2) * nc * lv), "cudaMalloc a");
        ck(cudaMalloc(&ad2, nc * facets), "cudaMalloc added");
        ck(cudaMemset(ad2, 0, nc * facets), "memset");
        if (size) {
            ck(cudaMemcpy(c2, c, sizeof(double2) * size, cudaMemcpyDeviceToDevice), "D2D");
            ck(cudaMemcpy(a2, a, sizeof(double2) * size * lv, cudaMemcpyDeviceToDevice), "D2D");
            ck(cudaMemcpy(ad2, added, size * facets, cudaMemcpyDeviceToDevice), "D2D");
        }
        cudaFree(c);
        cudaFree(a);
        cudaFree(added);
        c = c2;
        a = a2;
        added = ad2;
        cap = nc;
    }
};

struct System {
    int lv = 0;
    std::vector<Triple> triples;
    std::vector<cd> c, a;  // a: triple-major, lv each
    DevSystem dev;
    size_t size() const { return triples.size(); }
    // ConstraintSystem::error_at (design.hpp:86-91)
    cd error_at(size_t t, const double* v) const {
        cd e = c[t];
        const cd* at = a.data() + t * size_t(lv);
        for (int r = 0; r < lv; ++r) {
            e.x += v[r] * at[r].x;
            e.y += v[r] * at[r].y;
        }
        return e;
    }
};

void append_constraints(Problem& P, System& S, const std::vector<Triple>& fresh) {
    if (fresh.empty()) return;
    std::vector<TripleDev> h(fresh.size());
    for (size_t i = 0; i < fresh.size(); ++i) h[i] = TripleDev{fresh[i].n, fresh[i].b - P.blo, fresh[i].gi, 0};
    Dev<TripleDev> dt(h.size());
    dt.put(h.data(), h.size());
    Dev<double2> dc(h.size()), da(h.size() * size_t(P.lv));
    const int ntr = int(h.size());
    assemble_kernel<<<(ntr + 7) / 8, 256>>>(P.N, P.M, P.lv, P.step, ntr, dt.p, P.band_base.p, P.ph.p, P.des_pass.p,
                                           P.d_omega.p, P.blo, P.delta, dc.p, da.p);
    ck(cudaGetLastError(), "assemble_kernel");
    const size_t c0 = S.c.size(), a0 = S.a.size();
    S.c.resize(c0 + h.size());
    S.a.resize(a0 + h.size() * size_t(P.lv));
    dc.get(reinterpret_cast<double2*>(S.c.data() + c0), h.size());
    da.get(reinterpret_cast<double2*>(S.a.data() + a0), h.size() * size_t(P.lv));
    S.triples.insert(S.triples.end(), fresh.begin(), fresh.end());
    S.dev.reserve(S.triples.size());
    ck(cudaMemcpy(S.dev.c + c0, dc.p, sizeof(double2) * h.size(), cudaMemcpyDeviceToDevice), "D2D c");
    ck(cudaMemcpy(S.dev.a + a0, da.p, sizeof(double2) * h.size() * P.lv, cudaMemcpyDeviceToDevice), "D2D a");
    S.dev.size = S.triples.size();
}

// host response_from_row on a base row (spot checks only)
cd host_row_response(const double* base, int N, int shift, const cd* ph) {
    cd acc{0.0, 0.0};
    for (int q = 0; q < N; ++q) {
        const double d = base[((q + shift) % N + N) % N];
        acc.x += d * ph[q].x;
        acc.y += d * ph[q].y;
    }
    return acc;
}

// verify_constraints (design.hpp:156-190): the affine model must reproduce direct evaluation at
// random profiles on a strided subset of the triples.
void verify_constraints(Problem& P, const System& S, const std::vector<cd>& ph_host, int probes = 10) {
    if (S.size() == 0 || S.lv == 0) return;
    Rng rng(0xaff1e5);
    std::vector<double> v(static_cast<size_t>(S.lv));
    const size_t stride = std::max<size_t>(1, S.size() / 16);
    for (int probe = 0; probe < probes; ++probe) {
        for (auto& x : v) x = rng.uniform(-0.25, 1.25);
        std::vector<int> bs;
        for (size_t t = probe % stride; t < S.size(); t += stride) bs.push_back(S.triples[t].b);
        std::sort(bs.begin(), bs.end());
        bs.erase(std::unique(bs.begin(), bs.end()), bs.end());
        std::vector<cd> tabs(bs.size() * size_t(P.N));
        for (size_t i = 0; i < bs.size(); ++i) P.assemble_table(v.data(), bs[i], tabs.data() + i * P.N);
        P.base.resize(bs.size() * size_t(P.N));
        P.base_rows(int(bs.size()), tabs, P.base.p);
        std::vector<double> rows(bs.size() * size_t(P.N));
        P.base.get(rows.data(), rows.size());
        for (size_t t = probe % stride; t < S.size(); t += stride) {
            const Triple& tr = S.triples[t];
            const size_t bi = size_t(std::lower_bound(bs.begin(), bs.end(), tr.b) - bs.begin());
            const cd* phg = ph_host.data() + size_t(tr.gi) * P.N;
            const int shift = P.step * (tr.n - (P.M - 1));
            const cd acc = host_row_response(rows.data() + bi * P.N, P.N, shift, phg);
            const cd pre = phg[tr.n];
            cd direct{pre.x * acc.x - pre.y * acc.y, pre.x * acc.y + pre.y * acc.x};
            const double w = P.grid.omega[size_t(tr.gi)];
            if (w <= P.omega_of_bin(tr.b) - P.delta / 2.0 + 1e-12) {
                const double gd = (P.L - 1) / 2.0 + (P.M - 1);
                direct.x -= std::cos(-w * gd);
                direct.y -= std::sin(-w * gd);
            }
            const cd aff = S.error_at(t, v.data());
            if (std::hypot(direct.x - aff.x, direct.y - aff.y) > 1e-10)
                throw Failure{FCVBW_GPU_ERROR, "build_constraints: affine model failed verification"};
        }
    }
}

struct ScanBuffers {
    Dev<double> v;
    Dev<unsigned long long> stats;  // count, max bits
    Dev<Violation> list;
};

// Violations of the current LP point with the reference's selection (design.hpp:378-401):
// all (triple, facet) pairs not yet in the LP with facet value > delta + 1e-11, ordered by amount
// desc then (triple, facet) asc, first `take`. Counting passes narrow an amount threshold until at
// most `cap` candidates remain (every pair tied with the take-th is kept), then the host orders them.
std::vector<Violation> top_violations(System& S, ScanBuffers& B, const LpSolution& lp, const double* d_cos,
                                      const double* d_sin, size_t take) {
    const int64_t ntr = int64_t(S.size());
    const int lv = S.lv, facets = S.dev.facets;
    B.v.resize(size_t(lv));
    B.v.put(lp.v.data(), size_t(lv));
    B.stats.resize(2);
    const double reject = (lp.delta + 1e-11) * (lp.delta + 1e-11);
    const double lim = lp.delta + 1e-11;
    B.list.resize(size_t(1) << 20);
    unsigned long long st[2];
    auto pass = [&](double thr, bool collect) {
        ck(cudaMemset(B.stats.p, 0, 2 * sizeof(unsigned long long)), "memset");
        violation_scan_kernel<<<unsigned((ntr + 255) / 256), 256>>>(
            ntr, lv, facets, B.v.p, S.dev.c, S.dev.a, S.dev.added, d_cos, d_sin, reject, lim, lp.delta, thr,
            B.stats.p, B.stats.p + 1, collect ? B.list.p : nullptr, B.list.n);
        ck(cudaGetLastError(), "violation_scan_kernel");
        B.stats.get(st, 2);
        return st[0];
    };
    auto as_double = [](uint64_t u) {
        double d;
        std::memcpy(&d, &u, sizeof d);
        return d;
    };
    unsigned long long count = pass(0.0, true);
    if (count > B.list.n) {
        // bisect the bit pattern of a (positive) amount threshold until take <= count <= capacity
        const unsigned long long cap = B.list.n;
        uint64_t lo = 0, hi = st[1] + 1;  // count(lo) > cap, count(hi) = 0
        uint64_t thr = lo;
        bool found = false;
        while (hi - lo > 1) {
            const uint64_t mid = lo + (hi - lo) / 2;
            const unsigned long long c = pass(as_double(mid), false);
            if (c > cap) {
                lo = mid;
            } else if (c < take) {
                hi = mid;
            } else {
                thr = mid;
                found = true;
                break;
            }
        }
        if (!found) thr = lo;  // more than `cap` pairs tied at one amount: keep them all
        B.list.resize(pass(as_double(thr), false));
        count = pass(as_double(thr), true);
        if (count > B.list.n) throw Failure{FCVBW_GPU_ERROR, "violation scan: candidate list overflow"};
    }
    std::vector<Violation> v(count);
    if (count) B.list.get(v.data(), count);
    const size_t k = std::min<size_t>(take, v.size());
    std::partial_sort(v.begin(), v.begin() + k, v.end(), [](const Violation& x, const Violation& y) {
        return x.amount != y.amount ? x.amount > y.amount : std::tie(x.triple, x.facet) < std::tie(y.triple, y.facet);
    });
    v.resize(k);
    return v;
}

struct SweepOut {
    std::vector<double> cell_max;  // [num_b][M]
    std::vector<int> cell_gi;
    std::vector<double> cell_pass, cell_stop;  // with bands = true
    double max_abs = 0.0;
    Triple worst{-1, -1, -1};
    std::vector<Hit> hits;
};

// sweep_true_error (design.hpp:203-269) at profile v, collecting every point with |E| > thr.
SweepOut sweep(Problem& P, const double* v, double thr, bool bands = false) {
    const int N = P.N, M = P.M;
    const int64_t kk = int64_t(P.grid.omega.size());
    SweepOut out;
    out.cell_max.assign(size_t(P.num_b) * M, -1.0);
    out.cell_gi.assign(size_t(P.num_b) * M, -1);
    Dev<double> cmax(size_t(P.num_b) * M);
    Dev<int> cgi(size_t(P.num_b) * M);
    Dev<double> cpass(bands ? size_t(P.num_b) * M : 1), cstop(bands ? size_t(P.num_b) * M : 1);
    const size_t per_b_err = size_t(kk) * M;
    const int batch = int(std::max<size_t>(1, std::min<size_t>(size_t(P.num_b), (size_t(1) << 30) / (per_b_err * 8))));
    Dev<double> err(size_t(batch) * per_b_err);
    P.base.resize(size_t(batch) * N);
    unsigned long long cap = 1ull << 20;
    Dev<Hit> hits(cap);
    Dev<unsigned long long> nh(1);
    for (int b0 = 0; b0 < P.num_b; b0 += batch) {
        const int nb = std::min(batch, P.num_b - b0);
        std::vector<cd> tabs(size_t(nb) * N);
        for (int i = 0; i < nb; ++i) P.assemble_table(v, P.blo + b0 + i, tabs.data() + size_t(i) * N);
        P.base_rows(nb, tabs, P.base.p);
        for (;;) {
            ck(cudaMemset(nh.p, 0, sizeof(unsigned long long)), "memset");
            for (int64_t g0 = 0; g0 < kk; g0 += 65535) {  // gridDim.y <= 65535 grid points per launch
                const unsigned gy = unsigned(std::min<int64_t>(65535, kk - g0));
                sweep_eval_kernel<<<dim3((M + 127) / 128, gy, nb), 128>>>(
                    N, M, P.step, int(kk), int(g0), b0, P.base.p, P.ph.p, P.des_pass.p, P.d_omega.p, P.d_region.p,
                    P.blo, P.delta, thr, err.p, hits.p, nh.p, cap);
                ck(cudaGetLastError(), "sweep_eval_kernel");
            }
            unsigned long long count = 0;
            nh.get(&count, 1);
            if (count <= cap) {
                const size_t h0 = out.hits.size();
                out.hits.resize(h0 + count);
                if (count) hits.get(out.hits.data() + h0, count);
                break;
            }
            cap = count + (count >> 2);
            hits.resize(cap);
        }
        sweep_reduce_kernel<<<dim3((M + 127) / 128, nb), 128>>>(M, int(kk), nb, b0, err.p, cmax.p, cgi.p,
                                                                bands ? P.d_region.p : nullptr, cpass.p, cstop.p);
        ck(cudaGetLastError(), "sweep_reduce_kernel");
    }
    cmax.get(out.cell_max.data(), out.cell_max.size());
    cgi.get(out.cell_gi.data(), out.cell_gi.size());
    if (bands) {
        out.cell_pass.resize(out.cell_max.size());
        out.cell_stop.resize(out.cell_max.size());
        cpass.get(out.cell_pass.data(), out.cell_pass.size());
        cstop.get(out.cell_stop.data(), out.cell_stop.size());
    }
    for (int bi = 0; bi < P.num_b; ++bi)
        for (int n = 0; n < M; ++n) {
            const double m = out.cell_max[size_t(bi) * M + n];
            if (m > out.max_abs) {
                out.max_abs = m;
                out.worst = {n, P.blo + bi, out.cell_gi[size_t(bi) * M + n]};
            }
        }
    return out;
}

// Problem setup shared by solve_minimax and the exact verify: BinSpec validation, grid, host-libm
// tables, device copies; the per-band affine bases only when `band_tables`.
void init_problem(Problem& P, const fcvbw_gpu_design* g, int grid_points, int step, int device, bool band_tables,
                  std::vector<cd>& ph_host) {
    P.N = g->fft_length;
    P.L = g->filter_length;
    P.M = g->block_length;
    P.dn = g->transition_width_bins;
    P.blo = g->b_low;
    P.bhi = g->b_high;
    P.num_b = P.bhi - P.blo + 1;
    P.lv = P.dn - 1;
    P.step = step;
    const int N = P.N, M = P.M;
    if (N < 8 || (N & (N - 1))) validation("BinSpec: N must be 2^Q with Q >= 3");
    if (P.L < 1 || P.L > N || M != N - P.L + 1 || P.dn < 2 || P.dn % 2 ||
        !(P.dn / 2 <= P.blo && P.blo <= P.bhi && P.bhi <= N / 2 - P.dn / 2 - 1))
        validation("BinSpec: invalid geometry");
    if (grid_points < 2 * N) validation("FrequencyGrid: need K >= 2N grid points");
    if (step != 1 && step != -1) validation("shift step must be +-1");
    ck(cudaSetDevice(device), "cudaSetDevice");
    P.delta = P.dn * 2.0 * kPi / N;
    P.grid = build_grid(N, P.dn, P.blo, P.bhi, grid_points);
    const size_t kk = P.grid.omega.size();
    P.phase = phase_table(N, P.L);
    P.roots = unit_roots(N);
    ph_host.assign(kk * size_t(N), cd{0.0, 0.0});
    fill_phasor_table(P.grid.omega, N, ph_host.data());
    std::vector<cd> des(kk);
    const double gd = (P.L - 1) / 2.0 + (M - 1);
    for (size_t i = 0; i < kk; ++i) {
        const double ang = -P.grid.omega[i] * gd;
        des[i] = {std::cos(ang), std::sin(ang)};
    }
    P.ph.resize(ph_host.size());
    P.ph.put(reinterpret_cast<const double2*>(ph_host.data()), ph_host.size());
    P.des_pass.resize(kk);
    P.des_pass.put(reinterpret_cast<const double2*>(des.data()), kk);
    P.d_roots.resize(N);
    P.d_roots.put(reinterpret_cast<const double2*>(P.roots.data()), N);
    P.d_omega.resize(kk);
    P.d_omega.put(P.grid.omega.data(), kk);
    P.d_region.resize(P.grid.region.size());
    P.d_region.put(P.grid.region.data(), P.grid.region.size());
    P.bad.resize(1);
    if (band_tables) P.build_band_tables();
    ck(cudaDeviceSynchronize(), "tables");
}

}  // namespace design_impl

using namespace design_impl;

extern "C" int fcvbw_gpu_solve_minimax(const fcvbw_gpu_design* geometry, const fcvbw_gpu_solve_options* opt,
                                       int step, int device, double* v_out, fcvbw_gpu_solve_result* result) {
    try {
        if (!geometry || !opt || !v_out || !result) validation("solve_minimax: null argument");
        Problem P;
        std::vector<cd> ph_host;
        if (opt->facets < 8 || opt->facets % 2 != 0) validation("DesignProblem: facets must be even and >= 8");
        if (!(opt->exchange_tol > 0.0)) validation("DesignProblem: exchange_tol must be > 0");
        if (opt->max_rounds < 1) validation("DesignProblem: max_rounds must be >= 1");
        if (opt->seed_stride < 1) validation("DesignProblem: seed_stride must be >= 1");
        Clock clk;
        double t_tab = 0, t_asm = 0, t_lp = 0, t_sw = 0;
        init_problem(P, geometry, opt->grid_points, step, device, true, ph_host);
        const int M = P.M;
        const size_t kk = P.grid.omega.size();
        t_tab += clk.lap();

        // ---- seeds: every seed_stride-th masked point per (n, b) (design.hpp:290-306)
        const int lv = P.lv, facets = opt->facets;
        std::vector<Triple> seeds;
        for (int b = P.blo; b <= P.bhi; ++b) {
            const int8_t* region = P.grid.region.data() + size_t(b - P.blo) * kk;
            std::vector<int> masked;
            for (size_t g = 0; g < kk; ++g)
                if (region[g] != 2) masked.push_back(int(g));
            for (int n = 0; n < M; ++n)
                for (size_t j = 0; j < masked.size(); j += size_t(opt->seed_stride)) seeds.push_back({n, b, masked[j]});
        }
        std::sort(seeds.begin(), seeds.end(), by_bng);
        System S;
        S.lv = lv;
        S.dev.lv = lv;
        S.dev.facets = facets;
        append_constraints(P, S, seeds);
        verify_constraints(P, S, ph_host);
        t_asm += clk.lap();
        std::unordered_set<uint64_t> active;
        active.reserve(seeds.size() * 2);
        for (const Triple& t : seeds) active.insert(key_of(t));

        std::vector<double> cos_f(facets), sin_f(facets);
        for (int p = 0; p < facets; ++p) {
            cos_f[p] = std::cos(2.0 * kPi * p / facets);
            sin_f[p] = std::sin(2.0 * kPi * p / facets);
        }
        LpRows rows;
        rows.nv = lv;
        std::vector<double> tmp(static_cast<size_t>(lv));
        auto push_facet = [&](size_t t, int p) {
            const cd* at = S.a.data() + t * size_t(lv);
            for (int r = 0; r < lv; ++r) tmp[r] = cos_f[p] * at[r].x - sin_f[p] * at[r].y;
            rows.push(tmp.data(), 1.0, -(cos_f[p] * S.c[t].x - sin_f[p] * S.c[t].y));
        };
        constexpr double kProfileBox = 16.0;
        for (int r = 0; r < lv; ++r) {
            std::fill(tmp.begin(), tmp.end(), 0.0);
            tmp[r] = 1.0;
            rows.push(tmp.data(), 0.0, kProfileBox);
            tmp[r] = -1.0;
            rows.push(tmp.data(), 0.0, kProfileBox);
        }
        ChebyshevLp solver(lv);
        SpinPool pool(int(std::min(16u, std::max(1u, std::thread::hardware_concurrency()))));
        solver.set_pool(&pool);
        for (int p = 0; p < facets; ++p) push_facet(0, p);
        ck(cudaMemset(S.dev.added, 1, size_t(facets)), "memset added");
        Dev<double> d_cos(facets), d_sin(facets);
        d_cos.put(cos_f.data(), facets);
        d_sin.put(sin_f.data(), facets);
        ScanBuffers d_scan;
        Dev<int64_t> d_marks;

        std::vector<double> profile(size_t(lv), 0.0);
        double delta = 0.0, lp_delta = 0.0;
        int rounds = 0;
        int64_t lp_iterations = 0;
        for (int round = 1;; ++round) {
            if (round > opt->max_rounds)
                nonconvergence("solve_minimax: exchange did not converge in " + std::to_string(opt->max_rounds) +
                               " rounds");
            LpSolution lp;
            for (;;) {  // lazy facet generation over the active triples
                lp = solver.solve(rows);
                lp_iterations += lp.iterations;
                // violation scan on the device; the host keeps only the top 256 under the
                // reference's total order (amount desc, then (triple, facet) asc)
                std::vector<Violation> viol = top_violations(S, d_scan, lp, d_cos.p, d_sin.p, 256);
                if (viol.empty()) break;
                std::vector<int64_t> marks;
                for (const Violation& x : viol) {
                    push_facet(size_t(x.triple), x.facet);
                    marks.push_back(x.triple * facets + x.facet);
                }
                d_marks.resize(marks.size());
                d_marks.put(marks.data(), marks.size());
                mark_added_kernel<<<(int(marks.size()) + 255) / 256, 256>>>(int(marks.size()), d_marks.p, S.dev.added);
                ck(cudaGetLastError(), "mark_added_kernel");
            }
            for (int r = 0; r < lv; ++r)
                if (std::abs(lp.v[r]) > kProfileBox - 1e-3) lp_error("solve_minimax: profile hit the safety box");
            t_lp += clk.lap();

            SweepOut sw = sweep(P, lp.v.data(), lp.delta + 1e-10);
            t_sw += clk.lap();
            profile = lp.v;
            lp_delta = lp.delta;
            delta = sw.max_abs;
            rounds = round;

            std::vector<Hit> unseen;
            for (const Hit& h : sw.hits)
                if (!active.count(key_of(Triple{h.n, P.blo + h.bi, h.gi}))) unseen.push_back(h);
            const bool within_tol = sw.max_abs <= lp.delta * (1.0 + opt->exchange_tol) + 1e-15;
            if (unseen.empty()) {
                if (within_tol) break;
                nonconvergence("solve_minimax: no new constraints to add; exchange_tol is below the facet bound");
            }
            std::sort(unseen.begin(), unseen.end(), [](const Hit& x, const Hit& y) {
                if (x.err != y.err) return x.err > y.err;
                return std::tie(x.bi, x.n, x.gi) < std::tie(y.bi, y.n, y.gi);
            });
            if (unseen.size() > 4096) unseen.resize(4096);
            std::vector<Triple> fresh;
            fresh.reserve(unseen.size());
            for (const Hit& h : unseen) fresh.push_back({h.n, P.blo + h.bi, h.gi});
            std::sort(fresh.begin(), fresh.end(), by_bng);
            for (const Triple& t : fresh) active.insert(key_of(t));
            append_constraints(P, S, fresh);
            t_asm += clk.lap();
        }
        std::copy(profile.begin(), profile.end(), v_out);
        result->delta = delta;
        result->lp_delta = lp_delta;
        result->rounds = rounds;
        result->lp_iterations = lp_iterations;
        result->active_triples = int64_t(S.size());
        result->lp_rows = rows.size();
        result->grid_size = int64_t(kk);
        result->seconds_tables = t_tab;
        result->seconds_assembly = t_asm;
        result->seconds_lp = t_lp;
        result->seconds_sweep = t_sw;
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

// verify() (design.hpp:601-673) evaluated the reference's way — every (b, n, omega) response by its
// own length-N sum in the reference's operation order — so that every report field is bit-identical
// to the reference's. O(num_b K M N) on the device; fcvbw_gpu_verify (verify.cu) is the
// O(num_b K (N + M)) prefix-sum variant (agrees to ~1e-14).
extern "C" int fcvbw_gpu_verify_exact(const fcvbw_gpu_design* d, int dense_points, double delta_e, int window_offset,
                                      int step, int device, double* per_b_max, double* per_n_max,
                                      fcvbw_gpu_verification* report) {
    try {
        if (!d || !report) validation("verify: null argument");
        if (d->profile_length != d->transition_width_bins - 1 || !d->profile)
            validation("verify: profile length must be delta_N - 1");
        if (dense_points < 4 * d->grid_points)
            validation("verify: dense grid must have at least 4x the design points");
        if (window_offset != 1 - d->block_length)
            validation("verify: only the overlap-save window offset 1 - M is supported");
        Problem P;
        std::vector<cd> ph_host;
        init_problem(P, d, dense_points, step, device, false, ph_host);
        const int M = P.M, num_b = P.num_b;
        const SweepOut sw = sweep(P, d->profile, std::numeric_limits<double>::infinity(), true);
        std::memset(report, 0, sizeof(*report));
        report->dense_points = dense_points;
        report->worst_b = -1;
        report->worst_n = -1;
        std::vector<double> pn(size_t(M), 0.0);
        for (int bi = 0; bi < num_b; ++bi) {
            // BandStats (design.hpp:612-619): max_abs starts at 0; the first (omega, n) in scan order
            // attaining the band maximum is the worst point
            double bmax = 0.0, bpass = 0.0, bstop = 0.0;
            int bn = -1, bg = -1;
            for (int n = 0; n < M; ++n) {
                const size_t c = size_t(bi) * M + n;
                pn[n] = std::max(pn[n], std::max(0.0, sw.cell_max[c]));
                bpass = std::max(bpass, sw.cell_pass[c]);
                bstop = std::max(bstop, sw.cell_stop[c]);
                const double m = sw.cell_max[c];
                if (m > bmax || (m == bmax && m > 0.0 && sw.cell_gi[c] < bg)) {
                    bmax = m;
                    bn = n;
                    bg = sw.cell_gi[c];
                }
            }
            if (per_b_max) per_b_max[bi] = bmax;
            report->passband_max = std::max(report->passband_max, bpass);
            report->stopband_max = std::max(report->stopband_max, bstop);
            if (bmax > report->delta) {
                report->delta = bmax;
                report->worst_b = P.blo + bi;
                report->worst_n = bn;
                report->worst_omega = P.grid.omega[size_t(bg)];
            }
        }
        if (per_n_max) std::memcpy(per_n_max, pn.data(), sizeof(double) * M);
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

// ------------------------------------------------------------------ shift-rule calibration
namespace design_impl {

__global__ void impulse_kernel(int channels, int64_t S, int M, double2* x) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= channels) return;
    double2* row = x + size_t(c) * S;
    if (c < M) {
        row[c] = make_double2(1.0, 0.0);  // probe p = c: delta at time p
    } else {                               // superposition probe 2 delta(0) + delta(M / 2)
        row[0] = make_double2(2.0, 0.0);
        row[M / 2] = make_double2(row[M / 2].x + 1.0, 0.0);
    }
}

// Per measured PTVIR row: the first circular shift s minimising max_q |meas[q] - base[(q + s) mod N]|
// (calibrate_shift_convention, ptvir.hpp:262-279). One CTA per row; rows and base in shared memory.
__global__ void best_shift_kernel(int N, const double* __restrict__ rows, const double* __restrict__ base,
                                  int* best_s, double* best_dev) {
    extern __shared__ double sh[];
    double* meas = sh;
    double* bs = sh + N;
    __shared__ double s_dev[256];
    __shared__ int s_arg[256];
    const int row = blockIdx.x;
    for (int q = threadIdx.x; q < N; q += blockDim.x) {
        meas[q] = rows[size_t(row) * N + q];
        bs[q] = base[q];
    }
    __syncthreads();
    double best = INFINITY;
    int arg = 0;
    for (int s = threadIdx.x; s < N; s += blockDim.x) {
        double dev = 0.0;
        for (int q = 0; q < N && dev < best; ++q) dev = fmax(dev, fabs(meas[q] - bs[(q + s) & (N - 1)]));
        if (dev < best) {
            best = dev;
            arg = s;
        }
    }
    s_dev[threadIdx.x] = best;
    s_arg[threadIdx.x] = arg;
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = INFINITY;
        int a = 0;
        for (int t = 0; t < int(blockDim.x); ++t)
            if (s_dev[t] < b || (s_dev[t] == b && s_arg[t] < a)) {
                b = s_dev[t];
                a = s_arg[t];
            }
        best_s[row] = a;
        best_dev[row] = b;
    }
}

}  // namespace design_impl

// calibrated_shift_rule (design.hpp:476-484) with the GPU overlap-save engine as the probed
// processor: a generic profile (SeededRng(0xca11b8), uniform(0.2, 1)) at b_low, M impulse probes of
// N + 2M samples plus the superposition probe in ONE batched engine launch (M + 1 channels), then
// calibrate_shift_convention's support / fit / verification (ptvir.hpp:225-294; measure_ptvir
// :162-214), the O(M N^2) shift search on the device.
extern "C" int fcvbw_gpu_calibrate_shift(const fcvbw_gpu_design* g, int device, int* window_offset, int* step) {
    fcvbw_gpu_engine* eng = nullptr;
    double2 *dx = nullptr, *dy = nullptr;
    auto release = [&] {
        if (eng) fcvbw_gpu_destroy(eng);
        cudaFree(dx);
        cudaFree(dy);
    };
    try {
        if (!g || !window_offset || !step) validation("calibrate: null argument");
        const int N = g->fft_length, L = g->filter_length, M = g->block_length, dn = g->transition_width_bins;
        const int lv = dn - 1;
        if (N < 8 || (N & (N - 1)) || L < 1 || L > N || M != N - L + 1 || dn < 2 || dn % 2 ||
            !(dn / 2 <= g->b_low && g->b_low <= g->b_high && g->b_high <= N / 2 - dn / 2 - 1))
            validation("BinSpec: invalid geometry");
        ck(cudaSetDevice(device), "cudaSetDevice");
        Rng rng(0xca11b8);
        std::vector<double> v(static_cast<size_t>(lv));
        for (auto& x : v) x = rng.uniform(0.2, 1.0);
        fcvbw_gpu_config cfg{N, L, M, dn, g->b_low, g->b_high, v.data(), lv, g->b_low, FCVBW_GPU_C128, device, 0u};
        int rc = fcvbw_gpu_create(&cfg, &eng);
        if (rc) throw Failure{rc, fcvbw_gpu_last_error()};

        const int total = N + 2 * M, channels = M + 1;
        const size_t cells = size_t(channels) * total;
        ck(cudaMalloc(&dx, sizeof(double2) * cells), "cudaMalloc");
        ck(cudaMalloc(&dy, sizeof(double2) * cells), "cudaMalloc");
        ck(cudaMemset(dx, 0, sizeof(double2) * cells), "memset");
        impulse_kernel<<<(channels + 127) / 128, 128>>>(channels, total, M, dx);
        ck(cudaGetLastError(), "impulse_kernel");
        rc = fcvbw_gpu_run(eng, dx, total, channels, nullptr, 0, dy, nullptr, 0u);
        if (rc) throw Failure{rc, fcvbw_gpu_last_error()};
        std::vector<double2> y(cells);
        ck(cudaMemcpy(y.data(), dy, sizeof(double2) * cells, cudaMemcpyDeviceToHost), "D2H probes");
        auto probe = [&](int p, int t) { return y[size_t(p) * total + t].x; };

        // support windows: first observed lag per output phase
        int wo = 0;
        bool known = false;
        // first / last observed lag t - p per output phase row = t mod M (scanned in memory order)
        std::vector<int> firsts(size_t(M), std::numeric_limits<int>::max()), lasts(size_t(M), std::numeric_limits<int>::min());
        for (int p = 0; p < M; ++p)
            for (int t = 0; t < total; ++t)
                if (probe(p, t) != 0.0) {
                    const int row = t % M;
                    firsts[row] = std::min(firsts[row], t - p);
                    lasts[row] = std::max(lasts[row], t - p);
                }
        for (int row = 0; row < M; ++row) {
            const int first = firsts[row], last = lasts[row];
            if (first > last) continue;
            if (last - first + 1 > N) throw Failure{FCVBW_GPU_ERROR, "calibrate_shift_convention: support wider than N samples"};
            if (last - first + 1 == N) {
                const int w0 = first - row;
                if (known && w0 != wo)
                    throw Failure{FCVBW_GPU_ERROR, "calibrate_shift_convention: inconsistent support windows"};
                wo = w0;
                known = true;
            }
        }
        if (!known) wo = 1 - M;  // default_shift_rule (ptvir.hpp:59)

        // measure_ptvir with (wo, +1): rows, unconsumed-cell energy check, superposition check
        auto fmod_ = [](int64_t a, int m) {
            int r = int(a % m);
            return r < 0 ? r + m : r;
        };
        std::vector<double> rows(size_t(M) * N);
        for (int row = 0; row < M; ++row)
            for (int q = 0; q < N; ++q) {
                const int tau = q + row + wo;
                const int p = fmod_(row - tau, M);
                const int t = p + tau;
                rows[size_t(row) * N + q] = (t >= 0 && t < total) ? probe(p, t) : 0.0;
            }
        for (int p = 0; p < M; ++p)
            for (int t = 0; t < total; ++t) {
                const int row = t % M;
                const int q = (t - p) - row - wo;
                if ((q < 0 || q >= N) && std::abs(probe(p, t)) > 1e-12)
                    throw Failure{FCVBW_GPU_ERROR, "measure_ptvir: energy outside the calibrated support window"};
            }
        for (int t = 0; t < total; ++t)
            if (std::abs(probe(M, t) - 2.0 * probe(0, t) - probe(M / 2, t)) > 1e-12)
                throw Failure{FCVBW_GPU_ERROR, "measure_ptvir: superposition check failed (nonlinear processor)"};

        // base row of the same coefficients (bit-exact IDFT), then the per-row shift fit
        const auto phase = phase_table(N, L);
        const auto roots = unit_roots(N);
        std::vector<cd> tab(static_cast<size_t>(N));
        assemble_table(N, dn, g->b_low, v.data(), phase, tab.data());
        Dev<double2> dt(static_cast<size_t>(N)), dr(static_cast<size_t>(N));
        dt.put(reinterpret_cast<const double2*>(tab.data()), size_t(N));
        dr.put(reinterpret_cast<const double2*>(roots.data()), size_t(N));
        Dev<double> dbase(static_cast<size_t>(N)), drows(rows.size()), ddev(static_cast<size_t>(M));
        Dev<int> dbad(1), ds(static_cast<size_t>(M));
        ck(cudaMemset(dbad.p, 0, sizeof(int)), "memset");
        base_rows_kernel<<<dim3((N + 127) / 128, 1), 128>>>(N, 1, dt.p, dr.p, dbase.p, dbad.p);
        drows.put(rows.data(), rows.size());
        const size_t smem = 2 * sizeof(double) * N;
        if (smem > 48 * 1024)
            ck(cudaFuncSetAttribute(best_shift_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)), "smem");
        best_shift_kernel<<<M, 256, smem>>>(N, drows.p, dbase.p, ds.p, ddev.p);
        ck(cudaGetLastError(), "best_shift_kernel");
        std::vector<int> sigma(static_cast<size_t>(M));
        std::vector<double> dev(static_cast<size_t>(M));
        ds.get(sigma.data(), sigma.size());
        ddev.get(dev.data(), dev.size());
        for (int row = 0; row < M; ++row)
            if (dev[row] > 1e-12)
                throw Failure{FCVBW_GPU_ERROR,
                              "calibrate_shift_convention: no circular shift reproduces row " + std::to_string(row)};
        int found = 0;
        for (int st : {1, -1}) {
            bool ok = true;
            for (int row = 0; row < M && ok; ++row) ok = sigma[row] == fmod_(int64_t(st) * (row - (M - 1)), N);
            if (ok) {
                found = st;
                break;
            }
        }
        if (!found) throw Failure{FCVBW_GPU_ERROR, "calibrate_shift_convention: shifts do not follow an affine rule"};
        *window_offset = wo;
        *step = found;
        release();
        fcvbw_gpu_detail::set_last_error("");
        return FCVBW_GPU_OK;
    } catch (const Failure& f) {
        release();
        fcvbw_gpu_detail::set_last_error(f.msg);
        return f.code;
    } catch (const std::exception& e) {
        release();
        fcvbw_gpu_detail::set_last_error(e.what());
        return FCVBW_GPU_ERROR;
    }
}
