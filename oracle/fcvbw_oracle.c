/* TEST INFRASTRUCTURE ONLY — the CPU oracle (checker) for the GPU overlap-save path.
 *
 * A plain-C restatement of the reference algorithm (arxiv 2406.14116 / `fcvbw`, read-only at
 * /root/reference). Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library; the product path (paper_2406_14116_b200/libfcvbw_gpu.so) never does.
 *
 * Parity pin: tests/test_oracle_golden.py checks this restatement bit-for-bit against
 * oracle/_ref/libfcvbw_ref.so (the reference headers compiled in place) and against the committed
 * golden vectors in tests/golden/ (generated from the reference by tests/golden/make_golden.py),
 * including the reference's own known-answer pins (proj/tests/test_spectrum.cpp:62-126,
 * proj/tests/test_oracle_engine.cpp:85-161).
 *
 * Each function cites the reference file:line it restates (paths relative to /root/reference).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

typedef struct { double re, im; } cpx;

/* (a)(b) with the operand order of std::complex<double>::operator* (libstdc++ builtin). */
static inline cpx cmul(cpx a, cpx b) {
    cpx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
    return r;
}

/* ---------------------------------------------------------------- SeededRng
 * xorshift64* with the reference's double mapping: proj/include/fcvbw/ops.hpp:62-86. */
typedef struct { uint64_t s; } orc_rng;

static void rng_init(orc_rng* r, uint64_t seed) { r->s = seed ? seed : 0x9e3779b97f4a7c15ULL; }
static uint64_t rng_next(orc_rng* r) {
    uint64_t x = r->s;
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    r->s = x;
    return x * 0x2545F4914F6CDD1DULL;
}
static double rng_u01(orc_rng* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }

void orc_rng_uniform(uint64_t seed, double lo, double hi, double* out, int64_t count) {
    orc_rng r;
    rng_init(&r, seed);
    for (int64_t i = 0; i < count; ++i) out[i] = lo + (hi - lo) * rng_u01(&r);
}
void orc_rng_uniform_int(uint64_t seed, int lo, int hi, int* out, int64_t count) {
    orc_rng r;
    rng_init(&r, seed);
    for (int64_t i = 0; i < count; ++i)
        out[i] = lo + (int)(rng_next(&r) % (uint64_t)(hi - lo + 1));
}

/* ---------------------------------------------------------------- BinSpec
 * BinSpec::validate (spectrum.hpp:63-76) + profile length (engine.hpp:39-41).
 * Returns 0 ok, 2 validation error (the reference's ValidationError exit code). */
int orc_validate(int n, int l, int m, int dn, int blo, int bhi, int lv) {
    if (n < 8 || (n & (n - 1)) != 0) return 2;
    if (l < 1 || l > n) return 2;
    if (m != n - l + 1) return 2;
    if (dn < 2 || dn % 2 != 0) return 2;
    int half = dn / 2;
    if (!(half <= blo && blo <= bhi && bhi <= n / 2 - half - 1)) return 2;
    if (lv != dn - 1) return 2;
    return 0;
}

/* transition_bins (spectrum.hpp:161-165). */
static void transition_bins(int dn, int b, int* k1, int* k2) {
    *k1 = b - dn / 2 + 1;
    *k2 = b + dn / 2 - 1;
}

/* phase_table (spectrum.hpp:208-219): e^{-j pi ((k (L-1)) mod 2N) / N} on [0, N/2], conj mirror. */
void orc_phase_table(int n, int l, double* out /* 2n */) {
    const int64_t order = l - 1;
    for (int k = 0; k <= n / 2; ++k) {
        int64_t folded = ((int64_t)k * order) % (2 * (int64_t)n);
        double ang = -M_PI * (double)folded / n;
        out[2 * k] = cos(ang);
        out[2 * k + 1] = sin(ang);
    }
    for (int k = n / 2 + 1; k < n; ++k) {
        out[2 * k] = out[2 * (n - k)];
        out[2 * k + 1] = -out[2 * (n - k) + 1];
    }
}

/* magnitude_samples (spectrum.hpp:170-187), bin_region (spectrum.hpp:194-202) and
 * assemble_dft_coefficients (spectrum.hpp:221-242) for one b. region: 0 pass, 1 transition,
 * 2 stop. Any output pointer may be NULL. */
int orc_coefficients(int n, int l, int dn, int blo, int bhi, const double* v, int b, double* mag,
                     int* region, double* table) {
    if (orc_validate(n, l, n - l + 1, dn, blo, bhi, dn - 1)) return 2;
    if (b < blo || b > bhi) return 2;
    int k1, k2;
    transition_bins(dn, b, &k1, &k2);
    double* mg = (double*)calloc((size_t)n, sizeof(double));
    mg[0] = 1.0;
    for (int k = 1; k < k1; ++k) mg[k] = mg[n - k] = 1.0;
    for (int r = 0; r <= k2 - k1; ++r) mg[k1 + r] = mg[n - (k1 + r)] = v[r];
    if (mag) memcpy(mag, mg, sizeof(double) * (size_t)n);
    if (region) {
        for (int k = 0; k < n; ++k) {
            int f = k < n - k ? k : n - k;
            region[k] = f < k1 ? 0 : (f <= k2 ? 1 : 2);
        }
    }
    if (table) {
        double* ph = (double*)malloc(sizeof(double) * 2 * (size_t)n);
        orc_phase_table(n, l, ph);
        /* magnitude[k] * phase[k]: real * complex multiplies both parts (spectrum.hpp:234) */
        for (int k = 0; k < n; ++k) {
            table[2 * k] = mg[k] * ph[2 * k];
            table[2 * k + 1] = mg[k] * ph[2 * k + 1];
        }
        free(ph);
    }
    free(mg);
    return 0;
}

/* ---------------------------------------------------------------- Radix2Fft
 * Iterative radix-2 DIT with bit-reverse and twiddle tables: fft.hpp:35-51 (ctor), :95-108 (run),
 * :55-59 (real forward), :70-78 (real-out inverse, conj trick, 1/N). */
typedef struct {
    int n, log2n;
    int* bitrev;
    cpx* tw;
    cpx* scratch;
} fft_plan;

static void fft_init(fft_plan* p, int n) {
    p->n = n;
    p->log2n = 0;
    while ((1 << p->log2n) < n) ++p->log2n;
    p->bitrev = (int*)malloc(sizeof(int) * (size_t)n);
    for (int i = 0; i < n; ++i) {
        int r = 0;
        for (int b = 0; b < p->log2n; ++b) r |= ((i >> b) & 1) << (p->log2n - 1 - b);
        p->bitrev[i] = r;
    }
    p->tw = (cpx*)malloc(sizeof(cpx) * (size_t)(n / 2 > 0 ? n / 2 : 1));
    for (int k = 0; k < n / 2; ++k) {
        double ang = -2.0 * M_PI * (double)k / (double)n;
        p->tw[k].re = cos(ang);
        p->tw[k].im = sin(ang);
    }
    p->scratch = (cpx*)malloc(sizeof(cpx) * (size_t)n);
}
static void fft_free(fft_plan* p) {
    free(p->bitrev);
    free(p->tw);
    free(p->scratch);
}
static void fft_run(const fft_plan* p, cpx* a) {
    const int n = p->n;
    for (int len = 2, half = 1; len <= n; len <<= 1, half <<= 1) {
        int step = n / len;
        for (int blk = 0; blk < n; blk += len) {
            for (int j = 0; j < half; ++j) {
                cpx w = p->tw[j * step];
                cpx t = cmul(w, a[blk + j + half]);
                a[blk + j + half].re = a[blk + j].re - t.re;
                a[blk + j + half].im = a[blk + j].im - t.im;
                a[blk + j].re += t.re;
                a[blk + j].im += t.im;
            }
        }
    }
}
static void fft_forward_real(const fft_plan* p, const double* x, cpx* spec) {
    for (int i = 0; i < p->n; ++i) {
        spec[p->bitrev[i]].re = x[i];
        spec[p->bitrev[i]].im = 0.0;
    }
    fft_run(p, spec);
}
static void fft_inverse_real(fft_plan* p, const cpx* spec, double* out) {
    for (int i = 0; i < p->n; ++i) {
        p->scratch[p->bitrev[i]].re = spec[i].re;
        p->scratch[p->bitrev[i]].im = -spec[i].im;
    }
    fft_run(p, p->scratch);
    const double scale = 1.0 / (double)p->n;
    for (int i = 0; i < p->n; ++i) out[i] = p->scratch[i].re * scale;
}

/* ---------------------------------------------------------------- OlsEngine
 * Streaming overlap-save engine, structured and raw-table modes: engine.hpp:28-192.
 * run_block restates engine.hpp:139-172 (framing :142-143, forward :145-146, structured multiply
 * :147-162, raw multiply :163-165, inverse :166-167, ring update :169, discard :171). */
typedef struct {
    int n, m, structured;
    int dn, blo, bhi, k1, k2, b;
    const double* v;    /* profile, dn - 1 values (borrowed) */
    cpx* phase;         /* phase_table(N, L) */
    const double* raw;  /* raw table, 2N doubles (borrowed) */
    fft_plan fft;
    double* ring;       /* N - M */
    double* segment;    /* N */
    cpx* spectrum;
    cpx* filtered;
    double* time_out;
} ols_engine;

static void eng_init_common(ols_engine* e, int n, int m) {
    e->n = n;
    e->m = m;
    fft_init(&e->fft, n);
    e->ring = (double*)calloc((size_t)(n - m > 0 ? n - m : 1), sizeof(double));
    e->segment = (double*)malloc(sizeof(double) * (size_t)n);
    e->spectrum = (cpx*)malloc(sizeof(cpx) * (size_t)n);
    e->filtered = (cpx*)malloc(sizeof(cpx) * (size_t)n);
    e->time_out = (double*)malloc(sizeof(double) * (size_t)n);
    e->phase = NULL;
    e->raw = NULL;
}
static void eng_free(ols_engine* e) {
    fft_free(&e->fft);
    free(e->ring);
    free(e->segment);
    free(e->spectrum);
    free(e->filtered);
    free(e->time_out);
    free(e->phase);
}
/* set_bandwidth (engine.hpp:70-80): index update only. */
static int eng_set_bandwidth(ols_engine* e, int b) {
    if (!e->structured || b < e->blo || b > e->bhi) return 2;
    e->b = b;
    transition_bins(e->dn, b, &e->k1, &e->k2);
    return 0;
}
static void eng_run_block(ols_engine* e, const double* input, double* out /* M */) {
    const int n = e->n, overlap = n - e->m;
    memcpy(e->segment, e->ring, sizeof(double) * (size_t)overlap);
    memcpy(e->segment + overlap, input, sizeof(double) * (size_t)e->m);
    fft_forward_real(&e->fft, e->segment, e->spectrum);
    if (e->structured) {
        for (int k = 0; k <= n / 2; ++k) {
            cpx value = e->spectrum[k];
            if (k >= e->k1 && k <= e->k2) {
                const double v = e->v[k - e->k1];
                value.re *= v;
                value.im *= v;
            } else if (k > e->k2) {
                e->filtered[k].re = 0.0;
                e->filtered[k].im = 0.0;
                continue;
            }
            e->filtered[k] = cmul(value, e->phase[k]);
        }
        for (int k = 1; k < n / 2; ++k) {
            e->filtered[n - k].re = e->filtered[k].re;
            e->filtered[n - k].im = -e->filtered[k].im;
        }
    } else {
        for (int k = 0; k < n; ++k) {
            cpx h = {e->raw[2 * k], e->raw[2 * k + 1]};
            e->filtered[k] = cmul(e->spectrum[k], h);
        }
    }
    fft_inverse_real(&e->fft, e->filtered, e->time_out);
    memcpy(e->ring, e->segment + (n - overlap), sizeof(double) * (size_t)overlap);
    memcpy(out, e->time_out + overlap, sizeof(double) * (size_t)e->m);
}

/* Whole-stream driver = the reference CLI block loop (fcvbw_cli.cpp:95-113): the schedule value
 * for block m is applied before that block; a partial tail is zero-padded and truncated exactly
 * like feed + flush (engine.hpp:92-115). Blocks [b0, b1) are produced; the engine is primed by
 * re-running the preceding ceil((N-M)/M) blocks with output discarded (exact: a block depends
 * only on its N-sample segment). */
static int eng_stream(ols_engine* e, const double* x, int64_t s, const int* bs, int64_t b0,
                      int64_t b1, double* y) {
    const int m = e->m;
    const int64_t prime = (e->n - m + m - 1) / m;
    int64_t start = b0 - prime;
    if (start < 0) start = 0;
    double* blk_in = (double*)malloc(sizeof(double) * (size_t)m);
    double* blk_out = (double*)malloc(sizeof(double) * (size_t)m);
    int rc = 0;
    for (int64_t blk = start; blk < b1; ++blk) {
        if (bs && (rc = eng_set_bandwidth(e, bs[blk])) != 0) break;
        int64_t pos = blk * m;
        int64_t take = s - pos < m ? s - pos : m;
        for (int i = 0; i < m; ++i) blk_in[i] = i < take ? x[pos + i] : 0.0;
        eng_run_block(e, blk_in, blk_out);
        if (blk >= b0) memcpy(y + pos, blk_out, sizeof(double) * (size_t)take);
    }
    free(blk_in);
    free(blk_out);
    return rc;
}

static int eng_init_structured(ols_engine* e, int n, int l, int dn, int blo, int bhi,
                               const double* v, int b) {
    if (orc_validate(n, l, n - l + 1, dn, blo, bhi, dn - 1)) return 2;
    eng_init_common(e, n, n - l + 1);
    e->structured = 1;
    e->dn = dn;
    e->blo = blo;
    e->bhi = bhi;
    e->v = v;
    e->phase = (cpx*)malloc(sizeof(cpx) * (size_t)n);
    orc_phase_table(n, l, (double*)e->phase);
    if (eng_set_bandwidth(e, b)) {
        eng_free(e);
        return 2;
    }
    return 0;
}

/* Real stream, structured engine (single thread). bs: one b per block, or NULL (b0 fixed). */
int orc_ols_real(int n, int l, int dn, int blo, int bhi, const double* v, const double* x,
                 int64_t s, const int* bs, int b0, double* y) {
    ols_engine e;
    int rc = eng_init_structured(&e, n, l, dn, blo, bhi, v, bs ? bs[0] : b0);
    if (rc) return rc;
    int64_t nb = (s + e.m - 1) / e.m;
    rc = eng_stream(&e, x, s, bs, 0, nb, y);
    eng_free(&e);
    return rc;
}

/* Raw-table engine over a real stream (engine.hpp:47-56 + feed/flush). */
int orc_ols_raw_real(int n, int m, const double* table, const double* x, int64_t s, double* y) {
    if (m < 1 || m > n || n < 2 || (n & (n - 1))) return 2;
    ols_engine e;
    eng_init_common(&e, n, m);
    e.structured = 0;
    e.raw = table;
    int64_t nb = (s + m - 1) / m;
    int rc = eng_stream(&e, x, s, NULL, 0, nb, y);
    eng_free(&e);
    return rc;
}

/* Complex composite: y = engine(Re x) + j engine(Im x) per channel, threads over
 * (channel, component) streams. x, y: [channels][s] interleaved complex doubles. */
typedef struct {
    int n, l, dn, blo, bhi, b0;
    const double* v;
    const double* x;
    double* y;
    int64_t s;
    int channels;
    const int* bs;
    int64_t bstride;
    int next;  /* shared work counter */
    int rc;
    pthread_mutex_t mu;
} cx_job;

static void* cx_worker(void* arg) {
    cx_job* j = (cx_job*)arg;
    double* xr = (double*)malloc(sizeof(double) * (size_t)j->s);
    double* yr = (double*)malloc(sizeof(double) * (size_t)j->s);
    for (;;) {
        pthread_mutex_lock(&j->mu);
        int st = j->next++;
        pthread_mutex_unlock(&j->mu);
        if (st >= 2 * j->channels) break;
        int ch = st / 2, comp = st % 2;
        const double* xc = j->x + 2 * (int64_t)ch * j->s;
        for (int64_t i = 0; i < j->s; ++i) xr[i] = xc[2 * i + comp];
        const int* bs = j->bs ? j->bs + ch * j->bstride : NULL;
        int rc = orc_ols_real(j->n, j->l, j->dn, j->blo, j->bhi, j->v, xr, j->s, bs, j->b0, yr);
        if (rc) {
            pthread_mutex_lock(&j->mu);
            j->rc = rc;
            pthread_mutex_unlock(&j->mu);
        }
        double* yc = j->y + 2 * (int64_t)ch * j->s;
        for (int64_t i = 0; i < j->s; ++i) yc[2 * i + comp] = yr[i];
    }
    free(xr);
    free(yr);
    return NULL;
}

int orc_ols_complex(int n, int l, int dn, int blo, int bhi, const double* v, const double* x,
                    int64_t s, int channels, const int* bs, int64_t bstride, int b0, double* y,
                    int threads) {
    cx_job j = {n, l, dn, blo, bhi, b0, v, x, y, s, channels, bs, bstride, 0, 0,
                PTHREAD_MUTEX_INITIALIZER};
    if (orc_validate(n, l, n - l + 1, dn, blo, bhi, dn - 1)) return 2;
    if (threads < 1) threads = 1;
    if (threads > 2 * channels) threads = 2 * channels;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, cx_worker, &j);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
    return j.rc;
}

/* ---------------------------------------------------------------- independent oracles
 * Neumaier-compensated sum (oracle.hpp:16-31). */
typedef struct { double sum, comp; } csum;
static void cs_add(csum* c, double x) {
    double t = c->sum + x;
    if (fabs(c->sum) >= fabs(x))
        c->comp += (c->sum - t) + x;
    else
        c->comp += (x - t) + c->sum;
    c->sum = t;
}
static double cs_val(const csum* c) { return c->sum + c->comp; }

/* naive_block_filter (oracle.hpp:36-121): O(N^2) defining DFT/IDFT per block, same framing. */
int orc_naive_block_filter(int n, int m, const double* table, const double* x, int64_t s,
                           double* y) {
    if (m < 1 || m > n) return 2;
    cpx* roots = (cpx*)malloc(sizeof(cpx) * (size_t)n);
    for (int r = 0; r < n; ++r) {
        double ang = 2.0 * M_PI * r / n;
        roots[r].re = cos(ang);
        roots[r].im = sin(ang);
    }
    double* ring = (double*)calloc((size_t)(n - m + 1), sizeof(double));
    double* seg = (double*)malloc(sizeof(double) * (size_t)n);
    cpx* spec = (cpx*)malloc(sizeof(cpx) * (size_t)n);
    for (int64_t start = 0; start < s; start += m) {
        memcpy(seg, ring, sizeof(double) * (size_t)(n - m));
        for (int i = 0; i < m; ++i) seg[n - m + i] = start + i < s ? x[start + i] : 0.0;
        for (int k = 0; k < n; ++k) {
            csum re = {0, 0}, im = {0, 0};
            for (int t = 0; t < n; ++t) {
                cpx w = roots[((int64_t)t * k) % n];
                cs_add(&re, seg[t] * w.re);
                cs_add(&im, seg[t] * -w.im);
            }
            cpx v = {cs_val(&re), cs_val(&im)};
            cpx h = {table[2 * k], table[2 * k + 1]};
            spec[k] = cmul(v, h);
        }
        for (int q = n - m; q < n; ++q) {
            csum re = {0, 0};
            for (int k = 0; k < n; ++k) {
                cpx w = roots[((int64_t)q * k) % n];
                cs_add(&re, spec[k].re * w.re - spec[k].im * w.im);
            }
            int64_t t = start + (q - (n - m));
            if (t < s) y[t] = cs_val(&re) / n;
        }
        memcpy(ring, seg + m, sizeof(double) * (size_t)(n - m));
    }
    free(roots);
    free(ring);
    free(seg);
    free(spec);
    return 0;
}

/* direct_fir_convolution (oracle.hpp:124-134). */
void orc_direct_fir(const double* taps, int nt, const double* x, int64_t s, double* y) {
    for (int64_t t = 0; t < s; ++t) {
        csum acc = {0, 0};
        for (int q = 0; q < nt && q <= t; ++q) cs_add(&acc, taps[q] * x[t - q]);
        y[t] = cs_val(&acc);
    }
}

/* ---------------------------------------------------------------- design verification
 * verify() (design.hpp:601-673) with the overlap-save engine's shift rule (window offset 1 - M,
 * step +1; ptvir.hpp:52-56): FrequencyGrid::build (ptvir.hpp:309-343), base_response_idft
 * (ptvir.hpp:100-115), ptvir_from_base (:147-160), fill_phasors / response_from_row (:346-361),
 * desired_response (:368-381). Direct O(num_b K M N) evaluation, as the reference does it.
 * out_d = {delta, passband_max, stopband_max, worst_omega, refinement_bound};
 * out_i = {dense_points, worst_b, worst_n, pass, within_bound}. */

int orc_verify(int n, int l, int dn, int blo, int bhi, const double* v, double design_delta,
               int grid_points, int facets, int dense, double delta_e, double* per_b,
               double* per_n, double* out_d, int* out_i) {
    const int m = n - l + 1, half = dn / 2, num_b = bhi - blo + 1;
    if (orc_validate(n, l, m, dn, blo, bhi, dn - 1)) return 2;
    if (dense < 4 * grid_points || dense < 2 * n) return 2;
    /* grid: uniform points, then every band edge inserted in sorted position if absent */
    size_t cap = (size_t)dense + 2 * (size_t)num_b, kk = 0;
    double* om = (double*)malloc(sizeof(double) * cap);
    for (int i = 0; i < dense; ++i) om[kk++] = M_PI * i / (dense - 1);
    for (int b = blo; b <= bhi; ++b) {
        int edges[2] = {b - half, b + half};
        for (int e = 0; e < 2; ++e) {
            double w = edges[e] * 2.0 * M_PI / n;
            size_t lo = 0, hi = kk; /* lower_bound */
            while (lo < hi) {
                size_t mid = (lo + hi) / 2;
                if (om[mid] < w) lo = mid + 1; else hi = mid;
            }
            if (lo == kk || om[lo] != w) {
                memmove(om + lo + 1, om + lo, sizeof(double) * (kk - lo));
                om[lo] = w;
                ++kk;
            }
        }
    }
    double* table = (double*)malloc(sizeof(double) * 2 * (size_t)n);
    double* base = (double*)malloc(sizeof(double) * (size_t)n);
    cpx* roots = (cpx*)malloc(sizeof(cpx) * (size_t)n);
    cpx* ph = (cpx*)malloc(sizeof(cpx) * (size_t)n);
    double* pn = (double*)calloc((size_t)m, sizeof(double));
    for (int k = 0; k < n; ++k) {
        double ang = 2.0 * M_PI * k / n;
        roots[k].re = cos(ang);
        roots[k].im = sin(ang);
    }
    double delta = 0, pass_max = 0, stop_max = 0, worst_omega = 0;
    int worst_b = -1, worst_n = -1, rc = 0;
    for (int b = blo; b <= bhi && !rc; ++b) {
        orc_coefficients(n, l, dn, blo, bhi, v, b, NULL, NULL, table);
        for (int q = 0; q < n; ++q) {
            cpx acc = {0, 0};
            for (int k = 0; k < n; ++k) {
                cpx h = {table[2 * k], table[2 * k + 1]};
                cpx t = cmul(h, roots[((int64_t)q * k) % n]);
                acc.re += t.re;
                acc.im += t.im;
            }
            if (fabs(acc.im) > 1e-12 * n) rc = 2;
            base[q] = acc.re / n;
        }
        const double b_omega = b * 2.0 * M_PI / n, dlt = dn * 2.0 * M_PI / n;
        const double pass_edge = (b - half) * 2.0 * M_PI / n, stop_edge = (b + half) * 2.0 * M_PI / n;
        double bmax = 0, bpass = 0, bstop = 0, bw_omega = 0;
        int bw_n = -1;
        for (size_t gi = 0; gi < kk; ++gi) {
            const double w = om[gi];
            const int reg = w <= pass_edge ? 0 : (w >= stop_edge ? 1 : 2);
            if (reg == 2) continue;
            for (int q = 0; q < n; ++q) {
                double ang = -w * (double)q;
                ph[q].re = cos(ang);
                ph[q].im = sin(ang);
            }
            cpx des = {0, 0};
            if (w <= b_omega - dlt / 2.0 + 1e-12) {
                double gd = (l - 1) / 2.0 + (m - 1), ang = -w * gd;
                des.re = cos(ang);
                des.im = sin(ang);
            }
            for (int row = 0; row < m; ++row) {
                int shift = row - (m - 1);
                cpx acc = {0, 0};
                for (int q = 0; q < n; ++q) {
                    int idx = (int)(((int64_t)q + shift) % n);
                    if (idx < 0) idx += n;
                    acc.re += base[idx] * ph[q].re;
                    acc.im += base[idx] * ph[q].im;
                }
                cpx hn = cmul(ph[row], acc);
                double err = hypot(hn.re - des.re, hn.im - des.im);
                if (err > pn[row]) pn[row] = err;
                if (reg == 0) { if (err > bpass) bpass = err; }
                else if (err > bstop) bstop = err;
                if (err > bmax) {
                    bmax = err;
                    bw_n = row;
                    bw_omega = w;
                }
            }
        }
        if (per_b) per_b[b - blo] = bmax;
        if (bpass > pass_max) pass_max = bpass;
        if (bstop > stop_max) stop_max = bstop;
        if (bmax > delta) {
            delta = bmax;
            worst_b = b;
            worst_n = bw_n;
            worst_omega = bw_omega;
        }
    }
    if (!rc) {
        if (per_n) memcpy(per_n, pn, sizeof(double) * (size_t)m);
        double bound = design_delta / cos(M_PI / facets) + 1e-9;
        out_d[0] = delta;
        out_d[1] = pass_max;
        out_d[2] = stop_max;
        out_d[3] = worst_omega;
        out_d[4] = bound;
        out_i[0] = dense;
        out_i[1] = worst_b;
        out_i[2] = worst_n;
        out_i[3] = delta <= delta_e;
        out_i[4] = delta <= bound;
    }
    free(om);
    free(table);
    free(base);
    free(roots);
    free(ph);
    free(pn);
    return rc;
}
