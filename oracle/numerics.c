/* CPU oracle — see numerics.h for scope and provenance. TEST INFRASTRUCTURE. */
#include "numerics.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ------------------------------------------------------------ threads --- */
static int g_threads = 0;

int oracle_threads(void) {
    if (g_threads <= 0) {
        long n = sysconf(_SC_NPROCESSORS_ONLN);
        g_threads = n > 0 ? (int)n : 1;
    }
    return g_threads;
}
void oracle_set_threads(int n) { g_threads = n; }

typedef void (*range_fn)(void* ctx, long lo, long hi);
typedef struct {
    range_fn fn;
    void* ctx;
    long lo, hi;
} job_t;

static void* run_job(void* a) {
    job_t* j = (job_t*)a;
    j->fn(j->ctx, j->lo, j->hi);
    return NULL;
}

/* Static partition of [0, total) over the worker threads. */
static void parallel_for(long total, range_fn fn, void* ctx) {
    int t = oracle_threads();
    if (total < 64 || t <= 1) {
        fn(ctx, 0, total);
        return;
    }
    if (t > total) t = (int)total;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * t);
    job_t* jobs = (job_t*)malloc(sizeof(job_t) * t);
    long per = (total + t - 1) / t;
    int used = 0;
    for (int i = 0; i < t; ++i) {
        long lo = i * per, hi = lo + per > total ? total : lo + per;
        if (lo >= hi) break;
        jobs[i] = (job_t){fn, ctx, lo, hi};
        pthread_create(&th[i], NULL, run_job, &jobs[i]);
        ++used;
    }
    for (int i = 0; i < used; ++i) pthread_join(th[i], NULL);
    free(th);
    free(jobs);
}

/* ---------------------------------------------------------------- rng --- */
static uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
static uint64_t stream_base(uint64_t seed, uint64_t tag) { return splitmix64(seed ^ splitmix64(tag)); }

void oracle_fill_uniform(float* out, size_t n, uint64_t seed, uint64_t tag, float lo, float hi) {
    const uint64_t base = stream_base(seed, tag);
    const float span = hi - lo;
    for (size_t i = 0; i < n; ++i) {
        const uint64_t bits = splitmix64(base + i);
        const float u = (float)(bits >> 40) * (1.0f / 16777216.0f);
        const float prod = span * u;
        out[i] = lo + prod;
    }
}

void oracle_fill_labels(int32_t* out, int n, int classes, uint64_t seed) {
    const uint64_t base = stream_base(seed, 0x4C4142454C53ull);
    for (int i = 0; i < n; ++i) out[i] = (int32_t)(splitmix64(base + (uint64_t)i) % (uint64_t)classes);
}

/* float -> bf16 (round to nearest even) -> float */
void oracle_round_bf16(float* p, size_t n) {
    for (size_t i = 0; i < n; ++i) {
        uint32_t u;
        memcpy(&u, &p[i], 4);
        if ((u & 0x7f800000u) == 0x7f800000u) { /* inf / nan */
            if (u & 0x007fffffu) u |= 0x00400000u;
            u &= 0xffff0000u;
        } else {
            u += 0x7fffu + ((u >> 16) & 1u);
            u &= 0xffff0000u;
        }
        memcpy(&p[i], &u, 4);
    }
}

/* --------------------------------------------------------------- conv --- */
static int out_extent(int in, int f, int pad, int stride) {
    int num = in - f + 2 * pad;
    int q = num / stride;
    if ((num % stride != 0) && (num < 0)) --q; /* floor (Eq 1) */
    return q + 1;
}

typedef struct {
    const oracle_geom* g;
    const float *a, *b, *bias, *res, *mask;
    int relu;
    double *out, *out2;
    int ho, wo;
} conv_ctx;

/* one output pixel (n, ho, wo) per unit */
static void fwd_range(void* vc, long lo, long hi) {
    conv_ctx* c = (conv_ctx*)vc;
    const oracle_geom* g = c->g;
    for (long pix = lo; pix < hi; ++pix) {
        const int n = (int)(pix / ((long)c->ho * c->wo));
        const int rem = (int)(pix % ((long)c->ho * c->wo));
        const int ho = rem / c->wo, wo = rem % c->wo;
        for (int k = 0; k < g->k; ++k) {
            double acc = 0.0;
            for (int r = 0; r < g->r; ++r) {
                const int hi_ = ho * g->stride_h - g->pad_h + r;
                if (hi_ < 0 || hi_ >= g->h) continue;
                for (int s = 0; s < g->s; ++s) {
                    const int wi = wo * g->stride_w - g->pad_w + s;
                    if (wi < 0 || wi >= g->w) continue;
                    const float* xp = c->a + (((size_t)n * g->h + hi_) * g->w + wi) * g->c;
                    const float* wp = c->b + (((size_t)k * g->r + r) * g->s + s) * g->c;
                    for (int ch = 0; ch < g->c; ++ch) acc += (double)xp[ch] * (double)wp[ch];
                }
            }
            const size_t o = (size_t)pix * g->k + k;
            if (c->bias) acc += c->bias[k];
            if (c->res) acc += c->res[o];
            if (c->relu && acc < 0) acc = 0;
            c->out[o] = acc;
        }
    }
}

void oracle_conv_fwd(const oracle_geom* g, const float* x, const float* w, const float* bias,
                     const float* residual, int relu, double* y) {
    conv_ctx c = {g, x, w, bias, residual, NULL, relu, y, NULL,
                  out_extent(g->h, g->r, g->pad_h, g->stride_h),
                  out_extent(g->w, g->s, g->pad_w, g->stride_w)};
    parallel_for((long)g->n * c.ho * c.wo, fwd_range, &c);
}

/* one input pixel (n, h, w) per unit */
static void dgrad_range(void* vc, long lo, long hi) {
    conv_ctx* c = (conv_ctx*)vc;
    const oracle_geom* g = c->g;
    double* acc = (double*)calloc((size_t)g->c, sizeof(double));
    for (long pix = lo; pix < hi; ++pix) {
        const int n = (int)(pix / ((long)g->h * g->w));
        const int rem = (int)(pix % ((long)g->h * g->w));
        const int h = rem / g->w, w = rem % g->w;
        for (int ch = 0; ch < g->c; ++ch) acc[ch] = 0.0;
        for (int r = 0; r < g->r; ++r) {
            const int hn = h + g->pad_h - r;
            if (hn < 0 || hn % g->stride_h) continue;
            const int ho = hn / g->stride_h;
            if (ho >= c->ho) continue;
            for (int s = 0; s < g->s; ++s) {
                const int wn = w + g->pad_w - s;
                if (wn < 0 || wn % g->stride_w) continue;
                const int wo = wn / g->stride_w;
                if (wo >= c->wo) continue;
                const float* dyp = c->a + (((size_t)n * c->ho + ho) * c->wo + wo) * g->k;
                for (int k = 0; k < g->k; ++k) {
                    const double d = dyp[k];
                    const float* wp = c->b + (((size_t)k * g->r + r) * g->s + s) * g->c;
                    for (int ch = 0; ch < g->c; ++ch) acc[ch] += d * (double)wp[ch];
                }
            }
        }
        for (int ch = 0; ch < g->c; ++ch) {
            const size_t o = (size_t)pix * g->c + ch;
            double v = acc[ch];
            if (c->res) v += c->res[o];
            if (c->mask && !(c->mask[o] > 0.f)) v = 0.0;
            c->out[o] = v;
        }
    }
    free(acc);
}

void oracle_conv_dgrad(const oracle_geom* g, const float* dy, const float* w,
                       const float* residual, const float* mask, double* dx) {
    conv_ctx c = {g, dy, w, NULL, residual, mask, 0, dx, NULL,
                  out_extent(g->h, g->r, g->pad_h, g->stride_h),
                  out_extent(g->w, g->s, g->pad_w, g->stride_w)};
    parallel_for((long)g->n * g->h * g->w, dgrad_range, &c);
}

/* one output channel k per unit */
static void wgrad_range(void* vc, long lo, long hi) {
    conv_ctx* c = (conv_ctx*)vc;
    const oracle_geom* g = c->g;
    const size_t rsc = (size_t)g->r * g->s * g->c;
    for (long k = lo; k < hi; ++k) {
        double* dw = c->out + (size_t)k * rsc;
        for (size_t i = 0; i < rsc; ++i) dw[i] = 0.0;
        double db = 0.0;
        for (int n = 0; n < g->n; ++n)
            for (int ho = 0; ho < c->ho; ++ho)
                for (int wo = 0; wo < c->wo; ++wo) {
                    const double d = c->a[(((size_t)n * c->ho + ho) * c->wo + wo) * g->k + k];
                    db += d;
                    if (d == 0.0) continue;
                    for (int r = 0; r < g->r; ++r) {
                        const int hi_ = ho * g->stride_h - g->pad_h + r;
                        if (hi_ < 0 || hi_ >= g->h) continue;
                        for (int s = 0; s < g->s; ++s) {
                            const int wi = wo * g->stride_w - g->pad_w + s;
                            if (wi < 0 || wi >= g->w) continue;
                            const float* xp = c->b + (((size_t)n * g->h + hi_) * g->w + wi) * g->c;
                            double* o = dw + ((size_t)r * g->s + s) * g->c;
                            for (int ch = 0; ch < g->c; ++ch) o[ch] += d * (double)xp[ch];
                        }
                    }
                }
        if (c->out2) c->out2[k] = db;
    }
}

void oracle_conv_wgrad(const oracle_geom* g, const float* dy, const float* x, double* dw,
                       double* db) {
    conv_ctx c = {g, dy, x, NULL, NULL, NULL, 0, dw, db,
                  out_extent(g->h, g->r, g->pad_h, g->stride_h),
                  out_extent(g->w, g->s, g->pad_w, g->stride_w)};
    /* parallel over k; for few channels fall back to serial */
    parallel_for(g->k, wgrad_range, &c);
}

/* -------------------------------------------------------------- pools --- */
void oracle_maxpool_fwd(const float* x, double* y, uint8_t* arg, int n, int h, int w, int c,
                        int f, int s, int p) {
    const int ho = out_extent(h, f, p, s), wo = out_extent(w, f, p, s);
    for (int b = 0; b < n; ++b)
        for (int i = 0; i < ho; ++i)
            for (int j = 0; j < wo; ++j)
                for (int ch = 0; ch < c; ++ch) {
                    float best = -INFINITY;
                    int bi = 0;
                    for (int r = 0; r < f; ++r) {
                        const int hh = i * s - p + r;
                        if (hh < 0 || hh >= h) continue;
                        for (int q = 0; q < f; ++q) {
                            const int ww = j * s - p + q;
                            if (ww < 0 || ww >= w) continue;
                            const float v = x[(((size_t)b * h + hh) * w + ww) * c + ch];
                            if (v > best) {
                                best = v;
                                bi = r * f + q;
                            }
                        }
                    }
                    const size_t o = (((size_t)b * ho + i) * wo + j) * c + ch;
                    y[o] = best;
                    if (arg) arg[o] = (uint8_t)bi;
                }
}

void oracle_maxpool_bwd(const float* dy, const uint8_t* arg, double* dx, int n, int h, int w,
                        int c, int f, int s, int p) {
    const int ho = out_extent(h, f, p, s), wo = out_extent(w, f, p, s);
    memset(dx, 0, sizeof(double) * (size_t)n * h * w * c);
    for (int b = 0; b < n; ++b)
        for (int i = 0; i < ho; ++i)
            for (int j = 0; j < wo; ++j)
                for (int ch = 0; ch < c; ++ch) {
                    const size_t o = (((size_t)b * ho + i) * wo + j) * c + ch;
                    const int r = arg[o] / f, q = arg[o] % f;
                    const int hh = i * s - p + r, ww = j * s - p + q;
                    if (hh < 0 || hh >= h || ww < 0 || ww >= w) continue;
                    dx[(((size_t)b * h + hh) * w + ww) * c + ch] += dy[o];
                }
}

void oracle_avgpool_fwd(const float* x, double* y, int n, int hw, int c) {
    for (int b = 0; b < n; ++b)
        for (int ch = 0; ch < c; ++ch) {
            double acc = 0;
            for (int i = 0; i < hw; ++i) acc += x[((size_t)b * hw + i) * c + ch];
            y[(size_t)b * c + ch] = acc / hw;
        }
}

void oracle_avgpool_bwd(const float* dy, double* dx, int n, int hw, int c) {
    for (int b = 0; b < n; ++b)
        for (int i = 0; i < hw; ++i)
            for (int ch = 0; ch < c; ++ch)
                dx[((size_t)b * hw + i) * c + ch] = (double)dy[(size_t)b * c + ch] / hw;
}

void oracle_avgpool2d_fwd(const float* x, double* y, int n, int h, int w, int c, int f, int s, int p) {
    const int ho = out_extent(h, f, p, s), wo = out_extent(w, f, p, s);
    for (int b = 0; b < n; ++b)
        for (int i = 0; i < ho; ++i)
            for (int j = 0; j < wo; ++j)
                for (int ch = 0; ch < c; ++ch) {
                    double acc = 0;
                    for (int r = 0; r < f; ++r) {
                        const int hh = i * s - p + r;
                        if (hh < 0 || hh >= h) continue;
                        for (int q = 0; q < f; ++q) {
                            const int ww = j * s - p + q;
                            if (ww < 0 || ww >= w) continue;
                            acc += x[(((size_t)b * h + hh) * w + ww) * c + ch];
                        }
                    }
                    y[(((size_t)b * ho + i) * wo + j) * c + ch] = acc / (f * f);
                }
}

void oracle_avgpool2d_bwd(const float* dy, double* dx, int n, int h, int w, int c, int f, int s, int p) {
    const int ho = out_extent(h, f, p, s), wo = out_extent(w, f, p, s);
    memset(dx, 0, sizeof(double) * (size_t)n * h * w * c);
    for (int b = 0; b < n; ++b)
        for (int i = 0; i < ho; ++i)
            for (int j = 0; j < wo; ++j)
                for (int ch = 0; ch < c; ++ch) {
                    const double g = (double)dy[(((size_t)b * ho + i) * wo + j) * c + ch] / (f * f);
                    for (int r = 0; r < f; ++r) {
                        const int hh = i * s - p + r;
                        if (hh < 0 || hh >= h) continue;
                        for (int q = 0; q < f; ++q) {
                            const int ww = j * s - p + q;
                            if (ww < 0 || ww >= w) continue;
                            dx[(((size_t)b * h + hh) * w + ww) * c + ch] += g;
                        }
                    }
                }
}

double oracle_softmax_xent(const float* z, const int32_t* labels, double* dl, int n, int classes) {
    double total = 0.0;
    for (int b = 0; b < n; ++b) {
        const float* row = z + (size_t)b * classes;
        double m = -INFINITY, sum = 0.0;
        for (int k = 0; k < classes; ++k) m = row[k] > m ? row[k] : m;
        for (int k = 0; k < classes; ++k) sum += exp((double)row[k] - m);
        for (int k = 0; k < classes; ++k)
            dl[(size_t)b * classes + k] =
                (exp((double)row[k] - m) / sum - (k == labels[b] ? 1.0 : 0.0)) / n;
        total += log(sum) + m - row[labels[b]];
    }
    return total / n;
}

/* ---------------------------------------------------------------- sgd --- */
void oracle_sgd(float* w, const float* g, float* v, size_t n, float lr, float mom, float wd,
                float gscale) {
    for (size_t i = 0; i < n; ++i) {
        const float wi = w[i];
        const float a = g[i] * gscale;
        const float b = wd * wi;
        const float gg = a + b;
        const float mv = mom * v[i];
        const float vi = mv + gg;
        const float step = lr * vi;
        v[i] = vi;
        w[i] = wi - step;
    }
}
