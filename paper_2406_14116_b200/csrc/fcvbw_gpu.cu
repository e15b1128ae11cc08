// C-ABI implementation (include/fcvbw_gpu.h): engine handles, validation mirroring the reference,
// device-side tables, the streaming ring, the pipelined host-memory run and the coefficient dump.
// Host-side C++; every data-path byte is moved by the fused kernel (ols_kernel.cuh) or by
// cudaMemcpyAsync. There is no CPU compute fallback: without a usable CUDA device every entry
// point that needs one fails with FCVBW_GPU_ERROR.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/fcvbw_gpu.h"
#include "launch.cuh"

using namespace fcvbw_gpu;

namespace {

thread_local std::string g_last_error;

struct Failure {
    int code;
    std::string msg;
};

[[noreturn]] void validation(const std::string& m) { throw Failure{FCVBW_GPU_VALIDATION, m}; }
[[noreturn]] void error(const std::string& m) { throw Failure{FCVBW_GPU_ERROR, m}; }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) error(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        g_last_error.clear();
        return FCVBW_GPU_OK;
    } catch (const Failure& e) {
        g_last_error = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "out of host memory";
        return FCVBW_GPU_ERROR;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return FCVBW_GPU_ERROR;
    }
}

bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void reserve(size_t b) {
        if (b <= bytes) return;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        ck(cudaMalloc(&p, b), "cudaMalloc");
        bytes = b;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
};

// Page-locked host staging buffer (the streaming calls copy user spans through it, so their H2D /
// D2H transfers are truly asynchronous DMA instead of pageable copies staged by the driver).
struct PinBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void reserve(size_t b) {
        if (b <= bytes) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
        ck(cudaHostAlloc(&p, b, cudaHostAllocDefault), "cudaHostAlloc");
        bytes = b;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
    }
};

// exp(-j 2 pi e / n) in long double, exact integer argument reduction
std::complex<long double> root(int64_t e, int64_t n) {
    e %= n;
    if (e < 0) e += n;
    const long double ang = -2.0L * 3.141592653589793238462643383279502884L * (long double)e / (long double)n;
    return {cosl(ang), sinl(ang)};
}

// phase_table (spectrum.hpp:208-219), computed with the same double arithmetic as the reference
void phase_table(int n, int l, std::vector<std::complex<double>>& t) {
    const double kPi = 3.14159265358979323846;
    const int64_t order = l - 1;
    t.assign(size_t(n), {0.0, 0.0});
    for (int k = 0; k <= n / 2; ++k) {
        int64_t folded = (int64_t(k) * order) % (2 * int64_t(n));
        double ang = -kPi * static_cast<double>(folded) / n;
        t[k] = {std::cos(ang), std::sin(ang)};
    }
    for (int k = n / 2 + 1; k < n; ++k) t[k] = std::conj(t[n - k]);
}

}  // namespace

struct fcvbw_gpu_engine {
    int N = 0, L = 0, M = 0, dn = 0, blo = 0, bhi = 0, LV = 0;
    int dtype = FCVBW_GPU_C128, device = 0, mode = COEF_SHIFT;
    bool structured = true;
    int b = -1;
    int64_t blocks = 0;   // blocks_processed (engine.hpp:61)
    int64_t launches = 0;
    // op tallies (OpCounters, ops.hpp:15-30): data-dependent real multiplications by V, counted
    // analytically per processed block (2 L_V per real block, 4 L_V per complex block = two real
    // streams), and the (always zero) floating-point work of set_bandwidth
    uint64_t variable_mul = 0, retune_flops = 0;
    int64_t real_blocks = 0, complex_blocks = 0;
    bool corrupt_twiddles = false;  // FCVBW_GPU_TEST_CORRUPT_TWIDDLES (self-check test)
    int ring_real = -1;  // streaming ring sample kind: -1 unset, 0 complex, 1 real (reset clears)
    LaunchInfo li;
    size_t esize = 16;    // bytes per complex sample
    std::vector<double> V;
    DevBuf d_V, d_coef, d_tw, d_Vf64, d_phase64;  // tables in engine dtype (+ fp64 for the dump)
    // streaming state: d_hist holds [history (N - M) | pending] starting at sample hpos (a sliding
    // window: consumed blocks advance hpos, the window is moved to the front only when it reaches
    // the end of the buffer)
    DevBuf d_hist, d_hist2, d_out, d_b;
    PinBuf h_in, h_out;
    int64_t pending = 0;
    int64_t hpos = 0;
    cudaStream_t stream = nullptr;
    // pipelined host run
    static constexpr int kPipe = 3;
    cudaStream_t pstream[kPipe] = {nullptr, nullptr, nullptr};
    DevBuf p_in[kPipe], p_out[kPipe];
    DevBuf d_flag;

    void set_device() const { ck(cudaSetDevice(device), "cudaSetDevice"); }
};

namespace {

template <class R>
void upload_tables(fcvbw_gpu_engine* h, const std::vector<std::complex<double>>* coef_table) {
    using C = cx_t<R>;
    const int N = h->N;
    if (!plan_info<R>(N, &h->li)) validation("fft length " + std::to_string(N) + " not supported (2..8192)");
    const LaunchInfo& li = h->li;
    // per-thread factored twiddle base table (ols_kernel.cuh Pass::run): for pass p, butterfly m and
    // thread j, (LO - 1) values W^{i0 k} then (HI - 1) values W^{8 i1 k}, k = (j + mT) mod ns
    auto tangent = [&](std::complex<long double> w) -> C {
        // tangent form (Pass::run): W = wr (1 + j t), stored as {t, wr}. A zero real part (angle
        // +-pi/2) is replaced by a power of two far below the sample type's precision, so
        // t = wi / wr stays finite and wr * t == wi.
        const long double tiny = sizeof(R) == 4 ? 0x1p-40L : 0x1p-60L;
        long double wr = w.real();
        if (fabsl(wr) < tiny) wr = tiny;
        const R wr_r = static_cast<R>(wr);
        return C{static_cast<R>(w.imag() / (long double)wr_r), wr_r};
    };
    std::vector<C> tw(li.twc ? size_t(std::max(1, li.tw_compact))
                             : size_t(std::max(1, li.tw_per_thread)) * li.T);
    int off = 0, ns = li.radix[0];
    if (li.twc) {
        // compact layout (TWK = 4): pass p, entry i in [1, r), k in [0, ns) at off_p + (i - 1) ns + k
        for (int p = 1; p < li.passes; ++p) {
            const int r = li.radix[p];
            const int64_t unit = N / (int64_t(ns) * r);
            for (int i = 1; i < r; ++i)
                for (int k = 0; k < ns; ++k) {
                    const auto w = root(int64_t(i) * k * unit, N);
                    tw[size_t(off + (i - 1) * ns + k)] =
                        li.twt ? tangent(w) : C{static_cast<R>(w.real()), static_cast<R>(w.imag())};
                }
            off += (r - 1) * ns;
            ns *= r;
        }
    }
    for (int p = 1; p < li.passes && !li.twc; ++p) {
        const int r = li.radix[p];
        const int LO = r == 32 ? FCVBW_DFT32_A : (r >= 16 ? 4 : (r == 8 ? 2 : r)), HI = (r + LO - 1) / LO;
        const int CNT = li.twf ? r - 1 : (LO - 1) + (HI - 1);
        const int64_t unit = N / (int64_t(ns) * r);  // W_{ns r} = W_N^{unit}
        for (int m = 0; m < li.E / r; ++m)
            for (int j = 0; j < li.T; ++j) {
                const int k = (j + m * li.T) % ns;
                for (int c = 0; c < CNT; ++c) {
                    const int64_t e = li.twf ? int64_t(c + 1) * k
                                      : (c < LO - 1 ? int64_t(c + 1) * k : int64_t(LO) * (c - (LO - 1) + 1) * k);
                    const auto w = root(e * unit, N);
                    // paired layout: entries (2c', 2c' + 1) of thread j are adjacent (one float4)
                    C& dst = li.twp ? tw[(size_t(off / 2 + (m * CNT + c) / 2) * li.T + j) * 2 + ((m * CNT + c) & 1)]
                                    : tw[size_t(off + m * CNT + c) * li.T + j];
                    if (li.twt) {
                        dst = tangent(w);
                    } else {
                        dst = C{static_cast<R>(w.real()), static_cast<R>(w.imag())};
                    }
                }
            }
        off += (li.E / r) * CNT;
        ns *= r;
    }
    h->d_tw.reserve(sizeof(C) * tw.size());
    ck(cudaMemcpy(h->d_tw.p, tw.data(), sizeof(C) * tw.size(), cudaMemcpyHostToDevice), "upload twiddles");

    const double inv_n = 1.0 / N;
    if (h->structured) {
        std::vector<R> v(size_t(std::max(1, h->LV)));
        for (int i = 0; i < h->LV; ++i) v[i] = static_cast<R>(h->V[i] * inv_n);
        h->d_V.reserve(sizeof(R) * v.size());
        ck(cudaMemcpy(h->d_V.p, v.data(), sizeof(R) * v.size(), cudaMemcpyHostToDevice), "upload V");
        std::vector<std::complex<double>> ph;
        phase_table(N, h->L, ph);
        if (h->mode == COEF_PHASE) {
            std::vector<C> c(static_cast<size_t>(N));
            for (int k = 0; k < N; ++k) c[k] = C{static_cast<R>(ph[k].real()), static_cast<R>(ph[k].imag())};
            h->d_coef.reserve(sizeof(C) * N);
            ck(cudaMemcpy(h->d_coef.p, c.data(), sizeof(C) * N, cudaMemcpyHostToDevice), "upload phase");
        }
        // fp64 copies for the parity dump
        h->d_Vf64.reserve(sizeof(double) * std::max(1, h->LV));
        ck(cudaMemcpy(h->d_Vf64.p, h->V.data(), sizeof(double) * h->LV, cudaMemcpyHostToDevice), "upload V64");
        h->d_phase64.reserve(sizeof(double2) * N);
        ck(cudaMemcpy(h->d_phase64.p, ph.data(), sizeof(double2) * N, cudaMemcpyHostToDevice), "upload phase64");
    } else {
        std::vector<C> c(static_cast<size_t>(N));
        for (int k = 0; k < N; ++k)
            c[k] = C{static_cast<R>((*coef_table)[k].real() * inv_n), static_cast<R>((*coef_table)[k].imag() * inv_n)};
        h->d_coef.reserve(sizeof(C) * N);
        ck(cudaMemcpy(h->d_coef.p, c.data(), sizeof(C) * N, cudaMemcpyHostToDevice), "upload table");
    }
}

// Real-input I/O description (OlsArgs::xr): channels passed to launch_range are VIRTUAL channels.
struct RealIO {
    bool on = false;
    int io = 1;              // 1: one real block per transform (raw tables); 2: block pairs
    int64_t nblk_real = 0;   // io = 2: real blocks per channel
    bool pair = true;        // io = 2: pair consecutive blocks (false: one real block per transform)
};

// Internal launches (mask dump, construction self-check): a mask dump buffer, and a coefficient
// mode / table other than the engine's own. Not counted in the op tallies.
struct LaunchExtra {
    void* gdump = nullptr;
    int mode = -1;
    const void* coef = nullptr;
    bool internal = false;
};

// SeededRng (ops.hpp:62-86): xorshift64*, uniform01 = top 53 bits x 2^-53.
struct SeededRng {
    uint64_t s;
    explicit SeededRng(uint64_t seed) : s(seed ? seed : 0x9e3779b97f4a7c15ULL) {}
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

void launch_any(fcvbw_gpu_engine* h, const void* x, int64_t x_first, int64_t x_cs, int64_t S, int channels,
                const int32_t* bs, int64_t b_cs, void* y, int64_t y_first, int64_t y_cs, int64_t b0, int64_t b1,
                cudaStream_t st, const RealIO& rio = RealIO{}, const LaunchExtra& ex = LaunchExtra{});

// Construction-time self-check, the GPU form of OlsEngine::check_provider (engine.hpp:126-137):
// the seeded uniform(-1, 1) vector (seed 0x7ab1e5eed) of N samples goes through the engine's own
// FFT plan, twiddle tables and framing with an all-pass table (the identity filter:
// IFFT(FFT(segment) x 1/N) = segment), and must come back within the round-trip bound: 1e-12
// absolute per sample in fp64 (the reference's), 1e-5 in fp32 (a few ulp x log2 N at |x| <= 1).
// A miscompiled plan or a broken twiddle upload fails construction with status 2.
template <class R>
void self_check(fcvbw_gpu_engine* h) {
    using C = cx_t<R>;
    const int N = h->N;
    SeededRng rng(0x7ab1e5eedULL);
    std::vector<C> x(static_cast<size_t>(N)), y(static_cast<size_t>(N)), ones(static_cast<size_t>(N));
    for (auto& v : x) v = C{static_cast<R>(rng.uniform(-1.0, 1.0)), R(0)};
    for (auto& v : ones) v = C{static_cast<R>(1.0 / N), R(0)};
    DevBuf dx, dy, dt;
    dx.reserve(sizeof(C) * N);
    dy.reserve(sizeof(C) * N);
    dt.reserve(sizeof(C) * N);
    ck(cudaMemcpyAsync(dx.p, x.data(), sizeof(C) * N, cudaMemcpyHostToDevice, h->stream), "self-check H2D");
    ck(cudaMemcpyAsync(dt.p, ones.data(), sizeof(C) * N, cudaMemcpyHostToDevice, h->stream), "self-check H2D");
    LaunchExtra ex;
    ex.mode = COEF_RAW;
    ex.coef = dt.p;
    ex.internal = true;
    const int64_t nb = (N + h->M - 1) / h->M;
    launch_any(h, dx.p, 0, N, N, 1, nullptr, 0, dy.p, 0, N, 0, nb, h->stream, RealIO{}, ex);
    ck(cudaMemcpyAsync(y.data(), dy.p, sizeof(C) * N, cudaMemcpyDeviceToHost, h->stream), "self-check D2H");
    ck(cudaStreamSynchronize(h->stream), "self-check sync");
    const double tol = sizeof(R) == 8 ? 1e-12 : 1e-5;
    for (int i = 0; i < N; ++i) {
        const double dr = double(y[i].x) - double(x[i].x), di = double(y[i].y);
        if (!(std::fabs(dr) <= tol && std::fabs(di) <= tol))
            validation("engine: transform provider failed the round-trip check (sample " + std::to_string(i) +
                       ", error " + std::to_string(std::max(std::fabs(dr), std::fabs(di))) + ")");
    }
}

void init_device(fcvbw_gpu_engine* h, const std::vector<std::complex<double>>* raw) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        error(std::string("no CUDA device available (") + cudaGetErrorString(e) + "); the GPU engine has no CPU fallback");
    if (h->device < 0 || h->device >= count) validation("device ordinal out of range");
    h->set_device();
    h->esize = h->dtype == FCVBW_GPU_C64 ? 8 : 16;
    if (h->dtype == FCVBW_GPU_C64)
        upload_tables<float>(h, raw);
    else
        upload_tables<double>(h, raw);
    ck(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    if (h->corrupt_twiddles) {  // fault injection for the self-check test only
        const double bad[2] = {0.5, 0.5};
        ck(cudaMemcpy(h->d_tw.p, bad, h->esize, cudaMemcpyHostToDevice), "corrupt");
    }
    if (h->dtype == FCVBW_GPU_C64)
        self_check<float>(h);
    else
        self_check<double>(h);
}

void destroy_engine(fcvbw_gpu_engine* h) {
    if (!h) return;
    cudaSetDevice(h->device);
    for (DevBuf* b : {&h->d_V, &h->d_coef, &h->d_tw, &h->d_Vf64, &h->d_phase64, &h->d_hist, &h->d_hist2,
                      &h->d_out, &h->d_b, &h->d_flag})
        b->release();
    h->h_in.release();
    h->h_out.release();
    for (int i = 0; i < fcvbw_gpu_engine::kPipe; ++i) {
        h->p_in[i].release();
        h->p_out[i].release();
        if (h->pstream[i]) cudaStreamDestroy(h->pstream[i]);
    }
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
}

// One fused launch over global blocks [b0, b1) of `channels` (virtual) channels.
template <class R>
void launch_range(fcvbw_gpu_engine* h, const void* x, int64_t x_first, int64_t x_cs, int64_t S, int channels,
                  const int32_t* bs, int64_t b_cs, void* y, int64_t y_first, int64_t y_cs, int64_t b0, int64_t b1,
                  cudaStream_t st, const RealIO& rio = RealIO{}, const LaunchExtra& ex = LaunchExtra{}) {
    if (b1 <= b0 || channels <= 0) return;
    const size_t es = rio.on ? sizeof(R) : sizeof(cx_t<R>);  // bytes per element of x / y
    // keep channels * blocks per launch below 2^31 (32-bit work indices in the kernel)
    const int64_t max_items = int64_t(1) << 30;
    if ((b1 - b0) * int64_t(channels) > max_items) {
        if (b1 - b0 > max_items) {
            const int64_t mid = b0 + (b1 - b0) / 2;
            launch_range<R>(h, x, x_first, x_cs, S, channels, bs, b_cs, y, y_first, y_cs, b0, mid, st, rio, ex);
            launch_range<R>(h, x, x_first, x_cs, S, channels, bs, b_cs, y, y_first, y_cs, mid, b1, st, rio, ex);
        } else {
            const int half = channels / 2;
            launch_range<R>(h, x, x_first, x_cs, S, half, bs, b_cs, y, y_first, y_cs, b0, b1, st, rio, ex);
            launch_range<R>(h, static_cast<const char*>(x) + es * x_cs * half, x_first, x_cs, S, channels - half,
                            bs ? bs + b_cs * half : nullptr, b_cs, static_cast<char*>(y) + es * y_cs * half, y_first,
                            y_cs, b0, b1, st, rio, ex);
        }
        return;
    }
    OlsArgs<R> a{};
    a.x = static_cast<const cx_t<R>*>(x);
    a.y = static_cast<cx_t<R>*>(y);
    a.xr = static_cast<const R*>(x);
    a.yr = static_cast<R*>(y);
    a.nblk_real = rio.nblk_real;
    a.pair_real = rio.pair ? 1 : 0;
    a.x_first = x_first;
    a.y_first = y_first;
    a.x_cs = x_cs;
    a.y_cs = y_cs;
    a.S = S;
    a.blk_begin = b0;
    a.nblk = int(b1 - b0);
    a.total = int((b1 - b0) * channels);
    {
        // TMA-eligible relative blocks: segment [m M - (N - M), m M + M) inside [0, S) and 16-byte
        // aligned for every channel (alignment is uniform when all offsets are even multiples)
        const int64_t N = h->N, M = h->M;
        const int64_t first = (N - M + M - 1) / M;            // smallest m with m M - (N - M) >= 0
        const int64_t last = S >= N ? (S - N + (N - M)) / M : -1;  // largest m with m M + M <= S
        const uintptr_t base = reinterpret_cast<uintptr_t>(x);
        const bool aligned = !rio.on && (base % 16 == 0) && ((es * size_t(x_cs)) % 16 == 0 || channels == 1) &&
                             ((int64_t(es) * x_first) % 16 == 0) && ((int64_t(es) * M) % 16 == 0) &&
                             ((int64_t(es) * (N - M)) % 16 == 0);
        a.tma_lo = int(std::max<int64_t>(0, first - b0));
        a.tma_hi = aligned ? int(std::min<int64_t>(b1 - 1, last) - b0) : -1;
        if (a.tma_hi < a.tma_lo) {
            a.tma_lo = 1;
            a.tma_hi = 0;
        }
    }
    a.bsched = bs;
    a.b_cs = b_cs;
    a.b_const = h->b;
    a.M = h->M;
    a.half_dn = h->dn / 2;
    a.LV = h->LV;
    a.shift = (h->L - 1) / 2;
    a.V = static_cast<const R*>(h->d_V.p);
    a.coef = static_cast<const cx_t<R>*>(ex.coef ? ex.coef : h->d_coef.p);
    a.tw = static_cast<const cx_t<R>*>(h->d_tw.p);
    a.inv_n = static_cast<R>(1.0 / h->N);
    a.gdump = static_cast<R*>(ex.gdump);
    const int mode = ex.mode >= 0 ? ex.mode : h->mode;
    // shared memory behind the plan's own: the mask table of the plans that carry one (+ 16 bytes
    // of alignment slack), and V
    const size_t extra =
        mode != COEF_RAW
            ? 16 + sizeof(R) * (size_t(std::max(1, h->LV)) +
                                (h->li.mask_table ? mask_table_words(h->N, h->li.T, h->li.E, h->dn / 2, h->li.mask_table4) : 0))
            : 0;
    const int io = rio.on ? rio.io : (ex.gdump ? 3 : 0);
    ck(launch_ols<R>(h->N, mode, io, a, extra, 0, st, nullptr), "fused OLS launch");
    if (ex.internal) return;
    ++h->launches;
    // op tallies: blocks of this launch (a block-pair item carries up to two real blocks)
    const int64_t blocks = rio.on && rio.io == 2 ? std::min(2 * b1, rio.nblk_real) - 2 * b0 : b1 - b0;
    const int64_t n = blocks * int64_t(channels);
    if (rio.on) h->real_blocks += n;
    else h->complex_blocks += n;
    if (h->structured) h->variable_mul += uint64_t(n) * uint64_t(2 * h->LV) * (rio.on ? 1u : 2u);
}

void launch_any(fcvbw_gpu_engine* h, const void* x, int64_t x_first, int64_t x_cs, int64_t S, int channels,
                const int32_t* bs, int64_t b_cs, void* y, int64_t y_first, int64_t y_cs, int64_t b0, int64_t b1,
                cudaStream_t st, const RealIO& rio, const LaunchExtra& ex) {
    if (h->dtype == FCVBW_GPU_C64)
        launch_range<float>(h, x, x_first, x_cs, S, channels, bs, b_cs, y, y_first, y_cs, b0, b1, st, rio, ex);
    else
        launch_range<double>(h, x, x_first, x_cs, S, channels, bs, b_cs, y, y_first, y_cs, b0, b1, st, rio, ex);
}

__global__ void schedule_check_kernel(const int32_t* b, int rows, int64_t row_stride, int64_t count, int lo, int hi,
                                      int* bad) {
    const int64_t total = int64_t(rows) * count;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / count, i = e - r * count;
        const int v = b[r * row_stride + i];
        if (v < lo || v > hi) atomicExch(bad, 1);
    }
}

// Range check of a device schedule covering global blocks [b0, b1) of every channel (one launch).
void check_device_schedule(fcvbw_gpu_engine* h, const int32_t* bs, int64_t b_cs, int channels, int64_t b0,
                           int64_t b1, cudaStream_t st) {
    h->d_flag.reserve(sizeof(int));
    ck(cudaMemsetAsync(h->d_flag.p, 0, sizeof(int), st), "memset flag");
    const int rows = b_cs == 0 ? 1 : channels;
    schedule_check_kernel<<<296, 256, 0, st>>>(bs + b0, rows, b_cs, b1 - b0, h->blo, h->bhi,
                                               static_cast<int*>(h->d_flag.p));
    ck(cudaGetLastError(), "schedule check");
    int bad = 0;
    ck(cudaMemcpyAsync(&bad, h->d_flag.p, sizeof(int), cudaMemcpyDeviceToHost, st), "flag readback");
    ck(cudaStreamSynchronize(st), "schedule check sync");
    if (bad)
        validation("run: schedule requests b_N outside the design range [" + std::to_string(h->blo) + ", " +
                   std::to_string(h->bhi) + "]");
}

void check_host_schedule(const fcvbw_gpu_engine* h, const int32_t* bs, int64_t b_cs, int channels, int64_t nb) {
    const int rows = b_cs == 0 ? 1 : channels;
    for (int c = 0; c < rows; ++c)
        for (int64_t m = 0; m < nb; ++m) {
            const int b = bs[c * b_cs + m];
            if (b < h->blo || b > h->bhi)
                validation("schedule entry (" + std::to_string(m) + "," + std::to_string(b) +
                           ") requests b_N outside the design range [" + std::to_string(h->blo) + ", " +
                           std::to_string(h->bhi) + "]");
        }
}

// Bytes per streamed sample: complex samples of the engine dtype, or its real type for a real
// stream (fcvbw_gpu_*_real: the reference's own real-valued signature, engine.hpp:82,92).
size_t ring_es(const fcvbw_gpu_engine* h) { return h->ring_real == 1 ? h->esize / 2 : h->esize; }

// Fix the streaming ring's sample kind on first use; reset() clears it.
void ring_kind(fcvbw_gpu_engine* h, bool real) {
    const int want = real ? 1 : 0;
    if (h->ring_real == -1) h->ring_real = want;
    if (h->ring_real != want)
        validation("engine: streaming input mixes real and complex samples; reset() the engine first");
}

// Streaming step: the pending region of d_hist (after the N - M history) has grown to `avail`
// samples; run every complete block, copy its output to y_host, keep the tail. If `pad_to_block`
// the pending samples are first zero-padded to one full block (flush, engine.hpp:107-115) and
// only `emit_limit` output samples are returned. Real streams run as block pairs (IO = 2) in a
// virtual block numbering shifted by `off` blocks so that the first new block is even (pairs are
// (2p, 2p + 1)) and its history lies at non-negative virtual sample indices (the kernel zero-fills
// below 0, which is right only for the zero-primed start).
int64_t stream_step(fcvbw_gpu_engine* h, int64_t avail, void* y_host, int64_t y_cap, int64_t emit_limit) {
    const int64_t M = h->M, H = h->N - h->M;
    const int64_t nb = avail / M;
    if (nb == 0) return 0;
    const int64_t nout = nb * M;
    const int64_t emit = std::min(nout, emit_limit);
    if (emit > y_cap) validation("feed: output buffer too small");
    const size_t es = ring_es(h);
    h->d_out.reserve(es * size_t(nout));
    void* win = static_cast<char*>(h->d_hist.p) + es * size_t(h->hpos);  // the window [history | pending]
    // win[0] is global sample blocks*M - H; blocks [blocks, blocks + nb) are all complete
    const int64_t g0 = h->blocks * M - H;
    if (h->ring_real != 1) {
        const int64_t S_eff = h->blocks * M + nout;  // every read is inside the buffer
        launch_any(h, win, g0, 0, S_eff, 1, nullptr, 0, h->d_out.p, h->blocks * M, 0, h->blocks, h->blocks + nb,
                   h->stream);
    } else {
        int64_t off = 0;
        if (h->blocks > 0) {
            while ((h->blocks + off) * M < H) ++off;
            if ((h->blocks + off) & 1) ++off;
        }
        const int64_t vb = h->blocks + off;  // virtual index of the first new block (even, or 0)
        RealIO rio;
        rio.on = true;
        if (h->structured) {
            rio.io = 2;
            rio.pair = false;  // batching-invariant, bit-identical to the complex path on x + 0j
            rio.nblk_real = vb + nb;
            launch_any(h, win, g0 + off * M, 0, (vb + nb) * M, 1, nullptr, 0, h->d_out.p, vb * M, 0, vb / 2,
                       (vb + nb + 1) / 2, h->stream, rio);
        } else {
            rio.io = 1;
            launch_any(h, win, g0 + off * M, 0, (vb + nb) * M, 1, nullptr, 0, h->d_out.p, vb * M, 0, vb, vb + nb,
                       h->stream, rio);
        }
    }
    if (emit > 0) {
        h->h_out.reserve(es * size_t(emit));
        ck(cudaMemcpyAsync(h->h_out.p, h->d_out.p, es * size_t(emit), cudaMemcpyDeviceToHost, h->stream),
           "D2H output");
    }
    ck(cudaStreamSynchronize(h->stream), "stream sync");
    if (emit > 0) std::memcpy(y_host, h->h_out.p, es * size_t(emit));
    // the window now starts nout samples later: [history (the last H samples) | leftover pending]
    h->hpos += nout;
    h->blocks += nb;
    h->pending = avail - nout;
    return emit;
}

// Append n new samples after the window; the window moves to the front of the buffer (one D2D
// copy of H + pending samples) only when the buffer's end is reached, and the buffer grows
// geometrically when the window itself does not fit.
void stream_append(fcvbw_gpu_engine* h, const void* x_host, int64_t n) {
    const int64_t H = h->N - h->M;
    const size_t es = ring_es(h);
    const int64_t win = H + h->pending;  // samples in the current window
    const size_t need = es * size_t(h->hpos + win + n);
    if (need > h->d_hist.bytes) {
        const size_t want = es * size_t(win + n);
        DevBuf nb;
        nb.reserve(std::max(2 * want, size_t(es) * size_t(64 * h->N)));
        if (h->d_hist.p)
            ck(cudaMemcpyAsync(nb.p, static_cast<char*>(h->d_hist.p) + es * size_t(h->hpos), es * size_t(win),
                               cudaMemcpyDeviceToDevice, h->stream),
               "move window");
        else  // zero-primed history (engine.hpp:118-124): see fcvbw_gpu_reset
            ck(cudaMemsetAsync(nb.p, 0, es * size_t(H), h->stream), "zero history");
        ck(cudaStreamSynchronize(h->stream), "window sync");
        h->d_hist.release();
        h->d_hist = nb;
        h->hpos = 0;
    }
    if (n > 0) {
        h->h_in.reserve(es * size_t(n));
        std::memcpy(h->h_in.p, x_host, es * size_t(n));
        ck(cudaMemcpyAsync(static_cast<char*>(h->d_hist.p) + es * size_t(h->hpos + win), h->h_in.p, es * size_t(n),
                           cudaMemcpyHostToDevice, h->stream),
           "H2D input");
    }
}

int feed_impl(fcvbw_gpu_engine* h, const void* x_host, int64_t n, void* y_host, int64_t y_cap, int64_t* n_out,
              bool real) {
    if (n_out) *n_out = 0;
    return guarded([&] {
        if (!h) validation("null engine");
        if (n < 0 || (n > 0 && !x_host)) validation("feed: bad input span");
        ring_kind(h, real);
        // the whole output must fit before any state changes (a failed feed leaves the engine as it was)
        if ((h->pending + n) / h->M * h->M > y_cap) validation("feed: output buffer too small");
        h->set_device();
        stream_append(h, x_host, n);
        const int64_t emitted = stream_step(h, h->pending + n, y_host, y_cap, INT64_MAX);
        if (emitted == 0) {
            h->pending += n;
            ck(cudaStreamSynchronize(h->stream), "feed sync");
        }
        if (n_out) *n_out = emitted;
    });
}

int process_block_impl(fcvbw_gpu_engine* h, const void* x_host, int64_t n, void* y_host, bool real) {
    return guarded([&] {
        if (!h) validation("null engine");
        if (n != h->M) validation("engine: block must contain exactly M samples");
        if (h->pending != 0) validation("engine: pending partial input; feed() or flush() it first");
        if (!x_host || !y_host) validation("process_block: null buffer");
        ring_kind(h, real);
        h->set_device();
        stream_append(h, x_host, n);
        stream_step(h, n, y_host, n, INT64_MAX);
    });
}

int flush_impl(fcvbw_gpu_engine* h, void* y_host, int64_t y_cap, int64_t* n_out, bool real) {
    if (n_out) *n_out = 0;
    return guarded([&] {
        if (!h) validation("null engine");
        if (h->pending == 0) return;  // a second flush returns nothing (engine.hpp:108)
        ring_kind(h, real);
        if (h->pending > y_cap) validation("flush: output buffer too small");
        h->set_device();
        const int64_t real_n = h->pending, H = h->N - h->M;
        const size_t es = ring_es(h);
        // zero-pad the pending block to M samples (engine.hpp:110): make room for M - real_n more
        // samples after the window (stream_append with no data), then clear them
        h->pending = real_n;
        {
            const size_t need = es * size_t(h->hpos + H + h->M);
            if (need > h->d_hist.bytes) {
                const int64_t keep = H + real_n;
                DevBuf nb;
                nb.reserve(std::max(2 * es * size_t(H + h->M), size_t(es) * size_t(64 * h->N)));
                ck(cudaMemcpyAsync(nb.p, static_cast<char*>(h->d_hist.p) + es * size_t(h->hpos), es * size_t(keep),
                                   cudaMemcpyDeviceToDevice, h->stream),
                   "move window");
                ck(cudaStreamSynchronize(h->stream), "window sync");
                h->d_hist.release();
                h->d_hist = nb;
                h->hpos = 0;
            }
        }
        ck(cudaMemsetAsync(static_cast<char*>(h->d_hist.p) + es * size_t(h->hpos + H + real_n), 0,
                           es * size_t(h->M - real_n), h->stream),
           "zero pad");
        const int64_t emitted = stream_step(h, h->M, y_host, y_cap, real_n);
        if (n_out) *n_out = emitted;
    });
}

}  // namespace

// shared with the other translation units of the library (verify.cu)
namespace fcvbw_gpu_detail {
void set_last_error(const std::string& m) { g_last_error = m; }
}  // namespace fcvbw_gpu_detail

extern "C" {

const char* fcvbw_gpu_last_error(void) { return g_last_error.c_str(); }
const char* fcvbw_gpu_version(void) { return "fcvbw_gpu 0.1.0 (sm_100a)"; }

int fcvbw_gpu_create(const fcvbw_gpu_config* cfg, fcvbw_gpu_engine** out) {
    if (out) *out = nullptr;
    fcvbw_gpu_engine* h = nullptr;
    int rc = guarded([&] {
        if (!cfg || !out) validation("create: null argument");
        // BinSpec::validate (spectrum.hpp:63-76)
        const int N = cfg->fft_length, L = cfg->filter_length, M = cfg->block_length, dn = cfg->transition_width_bins;
        if (N < 8 || !is_pow2(N)) validation("BinSpec: N must be 2^Q with Q >= 3");
        if (L < 1 || L > N) validation("BinSpec: L must satisfy 1 <= L <= N");
        if (M != N - L + 1) validation("BinSpec: M must equal N - L + 1");
        if (dn < 2 || dn % 2 != 0) validation("BinSpec: delta_N must be a positive even integer");
        const int half = dn / 2;
        if (!(half <= cfg->b_low && cfg->b_low <= cfg->b_high && cfg->b_high <= N / 2 - half - 1))
            validation("BinSpec: need delta_N/2 <= b_low <= b_high <= N/2 - delta_N/2 - 1");
        if (N > 8192) validation("fft length above 8192 is not supported by the GPU engine");
        // profile length (engine.hpp:40-41)
        if (cfg->profile_length != dn - 1 || (!cfg->profile && dn > 1))
            validation("engine: profile length must be delta_N - 1");
        if (cfg->dtype != FCVBW_GPU_C64 && cfg->dtype != FCVBW_GPU_C128) validation("create: unknown dtype");
        h = new fcvbw_gpu_engine();
        h->N = N;
        h->L = L;
        h->M = M;
        h->dn = dn;
        h->blo = cfg->b_low;
        h->bhi = cfg->b_high;
        h->LV = dn - 1;
        h->V.assign(cfg->profile, cfg->profile + h->LV);
        h->dtype = cfg->dtype;
        h->device = cfg->device;
        h->structured = true;
        const bool shift_ok = ((L - 1) % 2) == 0;
        h->mode = (shift_ok && !(cfg->flags & FCVBW_GPU_FORCE_PHASE_MULTIPLY)) ? COEF_SHIFT : COEF_PHASE;
        if (h->mode == COEF_SHIFT && 4 * (L - 1) == N) h->mode = COEF_SHIFT_Q;  // BASELINE geometry
        // set_bandwidth(initial_b) (engine.hpp:42, 72-75)
        if (cfg->initial_b < h->blo || cfg->initial_b > h->bhi)
            validation("engine: bandwidth " + std::to_string(cfg->initial_b) + " outside design range [" +
                       std::to_string(h->blo) + ", " + std::to_string(h->bhi) + "]");
        h->b = cfg->initial_b;
        h->corrupt_twiddles = (cfg->flags & FCVBW_GPU_TEST_CORRUPT_TWIDDLES) != 0;
        init_device(h, nullptr);
        *out = h;
    });
    if (rc != FCVBW_GPU_OK && h) destroy_engine(h);
    return rc;
}

int fcvbw_gpu_create_raw(int fft_length, int block_length, const double* table, int dtype, int device,
                         fcvbw_gpu_engine** out) {
    if (out) *out = nullptr;
    fcvbw_gpu_engine* h = nullptr;
    int rc = guarded([&] {
        if (!out || !table) validation("create_raw: null argument");
        if (fft_length < 2 || !is_pow2(fft_length)) validation("fft: size must be a power of two >= 2");
        if (fft_length > 8192) validation("fft length above 8192 is not supported by the GPU engine");
        if (block_length < 1 || block_length > fft_length) validation("engine: need 1 <= M <= N");
        if (dtype != FCVBW_GPU_C64 && dtype != FCVBW_GPU_C128) validation("create: unknown dtype");
        h = new fcvbw_gpu_engine();
        h->N = fft_length;
        h->M = block_length;
        h->L = fft_length - block_length + 1;
        h->dtype = dtype;
        h->device = device;
        h->structured = false;
        h->mode = COEF_RAW;
        std::vector<std::complex<double>> t(static_cast<size_t>(fft_length));
        for (int k = 0; k < fft_length; ++k) t[k] = {table[2 * k], table[2 * k + 1]};
        init_device(h, &t);
        *out = h;
    });
    if (rc != FCVBW_GPU_OK && h) destroy_engine(h);
    return rc;
}

void fcvbw_gpu_destroy(fcvbw_gpu_engine* h) { destroy_engine(h); }

int fcvbw_gpu_block_length(const fcvbw_gpu_engine* h) { return h ? h->M : -1; }
int fcvbw_gpu_fft_length(const fcvbw_gpu_engine* h) { return h ? h->N : -1; }
int fcvbw_gpu_current_b(const fcvbw_gpu_engine* h) { return h ? h->b : -1; }
int64_t fcvbw_gpu_blocks_processed(const fcvbw_gpu_engine* h) { return h ? h->blocks : -1; }
int fcvbw_gpu_dtype(const fcvbw_gpu_engine* h) { return h ? h->dtype : -1; }
int64_t fcvbw_gpu_kernel_launches(const fcvbw_gpu_engine* h) { return h ? h->launches : -1; }

int fcvbw_gpu_set_bandwidth(fcvbw_gpu_engine* h, int b) {
    return guarded([&] {
        if (!h) validation("null engine");
        if (!h->structured) validation("engine: raw-table engine has no bandwidth");
        if (b < h->blo || b > h->bhi)
            validation("engine: bandwidth " + std::to_string(b) + " outside design range [" + std::to_string(h->blo) +
                       ", " + std::to_string(h->bhi) + "]");
        h->b = b;  // index update only (engine.hpp:76-79)
    });
}

int fcvbw_gpu_reset(fcvbw_gpu_engine* h) {
    return guarded([&] {
        if (!h) validation("null engine");
        h->pending = 0;
        h->blocks = 0;
        h->hpos = 0;
        h->ring_real = -1;
        // zero history (ring priming, engine.hpp:118-124). The complex path zero-fills global
        // indices below 0 in the kernel anyway; the real path's shifted block numbering reads the
        // history from the ring, so the ring must hold the zeros.
        if (h->d_hist.p) {
            h->set_device();
            const size_t hb = std::min(h->d_hist.bytes, h->esize * size_t(h->N - h->M));
            ck(cudaMemsetAsync(h->d_hist.p, 0, hb, h->stream), "reset history");
            ck(cudaStreamSynchronize(h->stream), "reset sync");
        }
    });
}

int fcvbw_gpu_feed(fcvbw_gpu_engine* h, const void* x_host, int64_t n, void* y_host, int64_t y_cap,
                   int64_t* n_out) {
    return feed_impl(h, x_host, n, y_host, y_cap, n_out, false);
}

int fcvbw_gpu_process_block(fcvbw_gpu_engine* h, const void* x_host, int64_t n, void* y_host) {
    return process_block_impl(h, x_host, n, y_host, false);
}

int fcvbw_gpu_flush(fcvbw_gpu_engine* h, void* y_host, int64_t y_cap, int64_t* n_out) {
    return flush_impl(h, y_host, y_cap, n_out, false);
}

int fcvbw_gpu_feed_real(fcvbw_gpu_engine* h, const void* x_host, int64_t n, void* y_host, int64_t y_cap,
                        int64_t* n_out) {
    return feed_impl(h, x_host, n, y_host, y_cap, n_out, true);
}

int fcvbw_gpu_process_block_real(fcvbw_gpu_engine* h, const void* x_host, int64_t n, void* y_host) {
    return process_block_impl(h, x_host, n, y_host, true);
}

int fcvbw_gpu_flush_real(fcvbw_gpu_engine* h, void* y_host, int64_t y_cap, int64_t* n_out) {
    return flush_impl(h, y_host, y_cap, n_out, true);
}

int fcvbw_gpu_op_counts(const fcvbw_gpu_engine* h, fcvbw_gpu_ops* out) {
    return guarded([&] {
        if (!h || !out) validation("op_counts: null argument");
        out->variable_mul = h->variable_mul;
        out->retune_flops = h->retune_flops;
        out->real_blocks = h->real_blocks;
        out->complex_blocks = h->complex_blocks;
    });
}

int fcvbw_gpu_run_range(fcvbw_gpu_engine* h, const void* x_dev, int64_t x_first, int64_t x_cs, int64_t S,
                        int channels, const int32_t* b_sched_dev, int64_t b_cs, void* y_dev, int64_t y_first,
                        int64_t y_cs, int64_t blk_begin, int64_t blk_end, void* stream, unsigned flags) {
    return guarded([&] {
        if (!h) validation("null engine");
        if (S < 0 || channels < 0 || blk_begin < 0 || blk_end < blk_begin) validation("run: bad extents");
        const int64_t nb = (S + h->M - 1) / h->M;
        if (blk_end > nb) validation("run: block range beyond the input stream");
        if (b_sched_dev && !h->structured) validation("engine: raw-table engine has no bandwidth");
        if (b_cs < 0) validation("run: negative schedule stride");
        if (blk_end == blk_begin || channels == 0) return;
        if (!x_dev || !y_dev) validation("run: null buffer");
        h->set_device();
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (b_sched_dev && !(flags & FCVBW_GPU_RUN_TRUSTED_SCHEDULE))
            check_device_schedule(h, b_sched_dev, b_cs, channels, blk_begin, blk_end, st);
        launch_any(h, x_dev, x_first, x_cs, S, channels, b_sched_dev, b_cs, y_dev, y_first, y_cs, blk_begin, blk_end,
                   st);
    });
}

int fcvbw_gpu_run(fcvbw_gpu_engine* h, const void* x_dev, int64_t S, int channels, const int32_t* b_sched_dev,
                  int64_t b_cs, void* y_dev, void* stream, unsigned flags) {
    if (!h) {
        g_last_error = "null engine";
        return FCVBW_GPU_VALIDATION;
    }
    const int64_t nb = S > 0 ? (S + h->M - 1) / h->M : 0;
    return fcvbw_gpu_run_range(h, x_dev, 0, S, S, channels, b_sched_dev, b_cs, y_dev, 0, S, 0, nb, stream, flags);
}

int fcvbw_gpu_run_real(fcvbw_gpu_engine* h, const void* x_dev, int64_t S, int channels, const int32_t* b_sched_dev,
                       int64_t b_cs, void* y_dev, void* stream, unsigned flags) {
    return guarded([&] {
        if (!h) validation("null engine");
        if (S < 0 || channels < 0 || b_cs < 0) validation("run: bad extents");
        if (b_sched_dev && !h->structured) validation("engine: raw-table engine has no bandwidth");
        const int64_t nb = S > 0 ? (S + h->M - 1) / h->M : 0;
        if (nb == 0 || channels == 0) return;
        if (!x_dev || !y_dev) validation("run: null buffer");
        h->set_device();
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (b_sched_dev && !(flags & FCVBW_GPU_RUN_TRUSTED_SCHEDULE))
            check_device_schedule(h, b_sched_dev, b_cs, channels, 0, nb, st);
        RealIO rio;
        rio.on = true;
        if (h->structured) {
            // block pairs (2p, 2p + 1) of each real channel share one complex transform (exact, H is
            // conjugate-symmetric; pairs whose b differ combine the two masks, see ols_kernel.cuh)
            rio.io = 2;
            rio.nblk_real = nb;
            rio.pair = !(flags & FCVBW_GPU_RUN_ONE_BLOCK_PER_TRANSFORM);
            launch_any(h, x_dev, 0, S, S, channels, b_sched_dev, b_cs, y_dev, 0, S, 0, (nb + 1) / 2, st, rio);
        } else {
            // raw tables may be asymmetric (the reference keeps Re(IFFT), fft.hpp:68-78): Im = 0
            rio.io = 1;
            launch_any(h, x_dev, 0, S, S, channels, nullptr, 0, y_dev, 0, S, 0, nb, st, rio);
        }
        (void)flags;
    });
}

}  // extern "C"

namespace {

// Host-memory whole-stream run, complex or real samples: (channel, block range) chunks of about
// 2^21 samples through a 3-deep H2D / fused kernel / D2H pipeline on three CUDA streams.
int run_host_impl(fcvbw_gpu_engine* h, const void* x_host, int64_t S, int channels, const int32_t* bs_host,
                  int64_t b_cs, void* y_host, bool real) {
    return guarded([&] {
        if (!h) validation("null engine");
        if (S < 0 || channels < 0 || b_cs < 0) validation("run: bad extents");
        if (bs_host && !h->structured) validation("engine: raw-table engine has no bandwidth");
        const int64_t M = h->M, H = h->N - h->M;
        const int64_t nb = (S + M - 1) / M;
        if (S == 0 || channels == 0) return;
        if (!x_host || !y_host) validation("run: null buffer");
        if (bs_host) check_host_schedule(h, bs_host, b_cs, channels, nb);
        h->set_device();
        const int rows = bs_host ? (b_cs == 0 ? 1 : channels) : 0;
        if (rows) {
            h->d_b.reserve(sizeof(int32_t) * size_t(rows) * size_t(nb));
            for (int c = 0; c < rows; ++c)
                ck(cudaMemcpyAsync(static_cast<int32_t*>(h->d_b.p) + c * nb, bs_host + c * b_cs, sizeof(int32_t) * nb,
                                   cudaMemcpyHostToDevice, h->stream),
                   "H2D schedule");
            ck(cudaStreamSynchronize(h->stream), "schedule sync");
        }
        const int32_t* dbs = rows ? static_cast<const int32_t*>(h->d_b.p) : nullptr;
        const int64_t dbcs = rows > 1 ? nb : 0;
        const size_t es = real ? h->esize / 2 : h->esize;  // bytes per host sample
        // chunk = (channel, block range); an even block count keeps real block pairs inside a chunk.
        // Channels shorter than one chunk are grouped: g whole channels per chunk (one copy each way
        // and one multi-channel launch), so that per-copy and per-launch overheads stay small.
        // Sized in bytes (16 MB per chunk, 32 MB per channel group), so that real streams (4 or 8 B
        // per sample) move as much per copy as complex ones.
        int64_t chunk_blocks = std::max<int64_t>(2, (int64_t(1) << 24) / (int64_t(es) * M));
        chunk_blocks += chunk_blocks & 1;
        const int64_t chunks_per_ch = (nb + chunk_blocks - 1) / chunk_blocks;
        const int group = chunks_per_ch == 1
                              ? int(std::max<int64_t>(1, std::min<int64_t>(channels, (int64_t(1) << 25) / (int64_t(es) * S))))
                              : 1;
        const size_t in_bytes = group > 1 ? es * size_t(group) * size_t(S) : es * size_t(chunk_blocks * M + H);
        const size_t out_bytes = group > 1 ? es * size_t(group) * size_t(S) : es * size_t(chunk_blocks * M);
        for (int i = 0; i < fcvbw_gpu_engine::kPipe; ++i) {
            if (!h->pstream[i]) ck(cudaStreamCreateWithFlags(&h->pstream[i], cudaStreamNonBlocking), "stream");
            h->p_in[i].reserve(in_bytes);
            h->p_out[i].reserve(out_bytes);
        }
        const char* xh = static_cast<const char*>(x_host);
        char* yh = static_cast<char*>(y_host);
        auto launch_chunk = [&](cudaStream_t st, int s, int64_t x_first, int64_t cs, int nch, const int32_t* bsc,
                                int64_t bcs, int64_t y_first, int64_t b0, int64_t b1) {
            if (!real) {
                launch_any(h, h->p_in[s].p, x_first, cs, S, nch, bsc, bcs, h->p_out[s].p, y_first, cs, b0, b1, st);
            } else {
                RealIO rio;
                rio.on = true;
                if (h->structured) {
                    rio.io = 2;
                    rio.nblk_real = nb;
                    launch_any(h, h->p_in[s].p, x_first, cs, S, nch, bsc, bcs, h->p_out[s].p, y_first, cs, b0 / 2,
                               (b1 + 1) / 2, st, rio);
                } else {
                    rio.io = 1;
                    launch_any(h, h->p_in[s].p, x_first, cs, S, nch, nullptr, 0, h->p_out[s].p, y_first, cs, b0, b1,
                               st, rio);
                }
            }
        };
        int64_t u = 0;
        if (group > 1) {
            for (int c = 0; c < channels; c += group, ++u) {
                const int gc = std::min(group, channels - c);
                const int s = int(u % fcvbw_gpu_engine::kPipe);
                cudaStream_t st = h->pstream[s];
                const size_t bytes = es * size_t(gc) * size_t(S);
                ck(cudaMemcpyAsync(h->p_in[s].p, xh + es * size_t(c) * size_t(S), bytes, cudaMemcpyHostToDevice, st),
                   "H2D chunk");
                const int32_t* bsc = dbs ? dbs + (rows > 1 ? c * dbcs : 0) : nullptr;
                launch_chunk(st, s, 0, S, gc, bsc, rows > 1 ? dbcs : 0, 0, 0, nb);
                ck(cudaMemcpyAsync(yh + es * size_t(c) * size_t(S), h->p_out[s].p, bytes, cudaMemcpyDeviceToHost, st),
                   "D2H chunk");
            }
        } else {
            for (int c = 0; c < channels; ++c)
                for (int64_t k = 0; k < chunks_per_ch; ++k, ++u) {
                    const int s = int(u % fcvbw_gpu_engine::kPipe);
                    cudaStream_t st = h->pstream[s];
                    const int64_t b0 = k * chunk_blocks, b1 = std::min(nb, b0 + chunk_blocks);
                    const int64_t i0 = std::max<int64_t>(0, b0 * M - H), i1 = std::min(S, b1 * M);
                    const int64_t o0 = b0 * M;
                    const char* xc = xh + es * size_t(c) * size_t(S);
                    char* yc = yh + es * size_t(c) * size_t(S);
                    const int32_t* bsc = dbs ? dbs + (rows > 1 ? c * dbcs : 0) : nullptr;
                    ck(cudaMemcpyAsync(h->p_in[s].p, xc + es * i0, es * size_t(i1 - i0), cudaMemcpyHostToDevice, st),
                       "H2D chunk");
                    launch_chunk(st, s, i0, 0, 1, bsc, 0, o0, b0, b1);
                    ck(cudaMemcpyAsync(yc + es * o0, h->p_out[s].p, es * size_t(i1 - o0), cudaMemcpyDeviceToHost, st),
                       "D2H chunk");
                }
        }
        for (int i = 0; i < fcvbw_gpu_engine::kPipe; ++i) ck(cudaStreamSynchronize(h->pstream[i]), "pipeline sync");
    });
}

}  // namespace

extern "C" {

int fcvbw_gpu_run_host(fcvbw_gpu_engine* h, const void* x_host, int64_t S, int channels, const int32_t* bs_host,
                       int64_t b_cs, void* y_host) {
    return run_host_impl(h, x_host, S, channels, bs_host, b_cs, y_host, false);
}

int fcvbw_gpu_run_real_host(fcvbw_gpu_engine* h, const void* x_host, int64_t S, int channels,
                            const int32_t* bs_host, int64_t b_cs, void* y_host) {
    return run_host_impl(h, x_host, S, channels, bs_host, b_cs, y_host, true);
}

int fcvbw_gpu_mask_dump(fcvbw_gpu_engine* h, const int32_t* b_host, int n_b, double* g_out) {
    return guarded([&] {
        if (!h) validation("null engine");
        if (!h->structured) validation("mask_dump: raw-table engine has no structured coefficients");
        if (n_b < 0 || (n_b > 0 && (!b_host || !g_out))) validation("mask_dump: bad arguments");
        for (int i = 0; i < n_b; ++i)
            if (b_host[i] < h->blo || b_host[i] > h->bhi) validation("transition_bins: b out of declared range");
        if (n_b == 0) return;
        h->set_device();
        // n_b blocks of one zero stream, block m using b_host[m]: the production kernel (same plan,
        // same instantiation as fcvbw_gpu_run) with its mask dump pointer set
        const int64_t S = int64_t(n_b) * h->M;
        const size_t cells = size_t(n_b) * h->N;
        const size_t rs = h->esize / 2;  // bytes of the engine's real type
        DevBuf dx, dy, db, dg;
        dx.reserve(h->esize * size_t(S));
        dy.reserve(h->esize * size_t(S));
        db.reserve(sizeof(int32_t) * n_b);
        dg.reserve(rs * cells);
        ck(cudaMemsetAsync(dx.p, 0, h->esize * size_t(S), h->stream), "mask dump zero input");
        ck(cudaMemcpyAsync(db.p, b_host, sizeof(int32_t) * n_b, cudaMemcpyHostToDevice, h->stream), "H2D b");
        LaunchExtra ex;
        ex.gdump = dg.p;
        ex.internal = true;
        launch_any(h, dx.p, 0, S, S, 1, static_cast<const int32_t*>(db.p), 0, dy.p, 0, S, 0, n_b, h->stream,
                   RealIO{}, ex);
        if (rs == 8) {
            ck(cudaMemcpyAsync(g_out, dg.p, rs * cells, cudaMemcpyDeviceToHost, h->stream), "D2H mask");
            ck(cudaStreamSynchronize(h->stream), "mask dump sync");
        } else {
            std::vector<float> g(cells);
            ck(cudaMemcpyAsync(g.data(), dg.p, rs * cells, cudaMemcpyDeviceToHost, h->stream), "D2H mask");
            ck(cudaStreamSynchronize(h->stream), "mask dump sync");
            for (size_t i = 0; i < cells; ++i) g_out[i] = double(g[i]);  // exact widening
        }
    });
}

int fcvbw_gpu_coeff_dump(fcvbw_gpu_engine* h, const int32_t* b_host, int n_b, int8_t* region, int16_t* v_index,
                         double* H) {
    return guarded([&] {
        if (!h) validation("null engine");
        if (!h->structured) validation("coeff_dump: raw-table engine has no structured coefficients");
        if (n_b < 0 || (n_b > 0 && !b_host)) validation("coeff_dump: bad b list");
        for (int i = 0; i < n_b; ++i)
            if (b_host[i] < h->blo || b_host[i] > h->bhi) validation("transition_bins: b out of declared range");
        if (n_b == 0) return;
        h->set_device();
        const size_t cells = size_t(n_b) * h->N;
        DevBuf db, dr, dv, dh;
        db.reserve(sizeof(int32_t) * n_b);
        if (region) dr.reserve(cells);
        if (v_index) dv.reserve(sizeof(int16_t) * cells);
        if (H) dh.reserve(sizeof(double2) * cells);
        ck(cudaMemcpyAsync(db.p, b_host, sizeof(int32_t) * n_b, cudaMemcpyHostToDevice, h->stream), "H2D b");
        coeff_dump_kernel<<<148, 256, 0, h->stream>>>(h->N, static_cast<int*>(db.p), n_b, h->dn / 2,
                                                     static_cast<const double*>(h->d_Vf64.p),
                                                     static_cast<const double2*>(h->d_phase64.p),
                                                     static_cast<int8_t*>(dr.p), static_cast<int16_t*>(dv.p),
                                                     static_cast<double2*>(dh.p));
        ck(cudaGetLastError(), "coeff dump launch");
        if (region) ck(cudaMemcpyAsync(region, dr.p, cells, cudaMemcpyDeviceToHost, h->stream), "D2H region");
        if (v_index)
            ck(cudaMemcpyAsync(v_index, dv.p, sizeof(int16_t) * cells, cudaMemcpyDeviceToHost, h->stream), "D2H vidx");
        if (H) ck(cudaMemcpyAsync(H, dh.p, sizeof(double2) * cells, cudaMemcpyDeviceToHost, h->stream), "D2H H");
        ck(cudaStreamSynchronize(h->stream), "coeff dump sync");
        db.release();
        dr.release();
        dv.release();
        dh.release();
    });
}

}  // extern "C"
