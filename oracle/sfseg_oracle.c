/*
 * sfseg_oracle.c — TEST INFRASTRUCTURE ONLY. CPU restatement of the SFSeg
 * power-iteration hot path of the reference (proj/src/engine.cpp,
 * proj/src/conv3d.cpp), used by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py as the checker. Nothing in the product
 * (paper_1907_02731_b200/) links, loads or calls this file.
 *
 * Arithmetic follows the reference operation by operation: float products and
 * sums rounded separately (compile with -ffp-contract=off; the reference is
 * built for baseline x86-64 without FMA), fp64 where the
 * reference uses double. Parity of this restatement is pinned against the
 * reference library itself (oracle/_ref/libsfseg_ref.so, built from
 * /root/reference/proj/src by oracle/Makefile) and against the committed
 * golden fixtures in tests/golden/ (tests/golden/make_golden.py).
 *
 * Deviation, by design: oracle_run uses the global step instead of the
 * per-frame windowed sweep (engine.cpp:290-325); test_engine.cpp:276-297 pins
 * the two bit-equal, and the oracle has no FrameTransform hook.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/sfseg_cuda.h"

#define ORACLE_OK 0
#define ORACLE_ERR_PARAMETER 1
#define ORACLE_ERR_SHAPE 2
#define ORACLE_ERR_VALIDATION 3
#define ORACLE_ERR_DEGENERATE 4
#define ORACLE_ERR_MEMORY 5

/* ---- kernel taps: conv3d.cpp:23-58 ------------------------------------- */

static void raw_taps(double sigma, int radius, double* taps) {
    /* conv3d.cpp:23-30 */
    const double inv = 1.0 / (2.0 * sigma * sigma);
    for (int i = -radius; i <= radius; ++i)
        taps[i + radius] = exp(-(double)i * (double)i * inv);
}

static double tap_sum(const double* taps, int n) { /* conv3d.cpp:32-36 */
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += taps[i];
    return s;
}

int oracle_make_kernel(const int32_t radii[3], const double sigmas[3], double* taps_t,
                       double* taps_y, double* taps_x) {
    for (int a = 0; a < 3; ++a) /* conv3d.cpp:42-45 */
        if (!(sigmas[a] > 0.0) || radii[a] < 0) return ORACLE_ERR_PARAMETER;
    raw_taps(sigmas[0], radii[0], taps_t);
    raw_taps(sigmas[1], radii[1], taps_y);
    raw_taps(sigmas[2], radii[2], taps_x);
    /* conv3d.cpp:54-57: unit mass folded into taps_t only */
    const double total = tap_sum(taps_t, 2 * radii[0] + 1) *
                         tap_sum(taps_y, 2 * radii[1] + 1) *
                         tap_sum(taps_x, 2 * radii[2] + 1);
    for (int i = 0; i < 2 * radii[0] + 1; ++i) taps_t[i] /= total;
    return ORACLE_OK;
}

/* ---- separable convolution: conv3d.cpp:80-185 -------------------------- */

static int imin(int a, int b) { return a < b ? a : b; }

static void axis_pass_x(const float* src, float* dst, uint32_t T, uint32_t H, uint32_t W,
                        const double* taps, int r) {
    float ft[64];
    for (int i = 0; i < 2 * r + 1; ++i) ft[i] = (float)taps[i]; /* conv3d.cpp:84-85 */
    const size_t rows = (size_t)T * H;
    for (size_t row = 0; row < rows; ++row) { /* conv3d.cpp:88-101 */
        const float* in = src + row * W;
        float* out = dst + row * W;
        for (uint32_t x = 0; x < W; ++x) {
            float acc = 0.0f;
            const int d_lo = -imin(r, (int)x);
            const int d_hi = imin(r, (int)(W - 1 - x));
            for (int d = d_lo; d <= d_hi; ++d) acc += ft[d + r] * in[(int)x + d];
            out[x] = acc;
        }
    }
}

static void axis_pass_y(const float* src, float* dst, uint32_t T, uint32_t H, uint32_t W,
                        const double* taps, int r) {
    float ft[64];
    for (int i = 0; i < 2 * r + 1; ++i) ft[i] = (float)taps[i]; /* conv3d.cpp:108-109 */
    const size_t plane = (size_t)H * W;
    for (size_t t = 0; t < T; ++t) { /* conv3d.cpp:113-135 */
        const float* in = src + t * plane;
        float* out = dst + t * plane;
        for (uint32_t y = 0; y < H; ++y) {
            float* orow = out + (size_t)y * W;
            const int d_lo = -imin(r, (int)y);
            const int d_hi = imin(r, (int)(H - 1 - y));
            int first = 1;
            for (int d = d_lo; d <= d_hi; ++d) {
                const float w = ft[d + r];
                const float* irow = in + (size_t)((int)y + d) * W;
                if (first) {
                    for (uint32_t x = 0; x < W; ++x) orow[x] = w * irow[x];
                    first = 0;
                } else {
                    for (uint32_t x = 0; x < W; ++x) orow[x] += w * irow[x];
                }
            }
            if (first) memset(orow, 0, sizeof(float) * W);
        }
    }
}

static void axis_pass_t(const float* src, float* dst, uint32_t T, uint32_t H, uint32_t W,
                        const double* taps, int r) {
    float ft[64];
    for (int i = 0; i < 2 * r + 1; ++i) ft[i] = (float)taps[i]; /* conv3d.cpp:142-143 */
    const size_t plane = (size_t)H * W;
    for (size_t t = 0; t < T; ++t) { /* conv3d.cpp:147-165 */
        float* out = dst + t * plane;
        const int d_lo = -imin(r, (int)t);
        const int d_hi = imin(r, (int)(T - 1 - t));
        int first = 1;
        for (int d = d_lo; d <= d_hi; ++d) {
            const float w = ft[d + r];
            const float* in = src + (size_t)((long)t + d) * plane;
            if (first) {
                for (size_t i = 0; i < plane; ++i) out[i] = w * in[i];
                first = 0;
            } else {
                for (size_t i = 0; i < plane; ++i) out[i] += w * in[i];
            }
        }
        if (first) memset(out, 0, sizeof(float) * plane);
    }
}

typedef struct {
    double t[64], y[64], x[64];
    int32_t r[3];
} oracle_kernel;

static int kernel_from(const sfseg_params* p, oracle_kernel* k) {
    for (int a = 0; a < 3; ++a) {
        if (p->radii[a] < 0 || p->radii[a] > 31) return ORACLE_ERR_PARAMETER;
        k->r[a] = p->radii[a];
    }
    return oracle_make_kernel(p->radii, p->sigmas, k->t, k->y, k->x);
}

/* convolve_separable (conv3d.cpp:171-185): x -> y -> t, two temporaries. */
int oracle_convolve_separable(uint32_t T, uint32_t H, uint32_t W, const float* v,
                              const int32_t radii[3], const double sigmas[3], float* out) {
    sfseg_params p;
    memset(&p, 0, sizeof p);
    for (int a = 0; a < 3; ++a) {
        p.radii[a] = radii[a];
        p.sigmas[a] = sigmas[a];
    }
    oracle_kernel k;
    int rc = kernel_from(&p, &k);
    if (rc) return rc;
    const size_t n = (size_t)T * H * W;
    float* a = (float*)malloc(n * sizeof(float));
    float* b = (float*)malloc(n * sizeof(float));
    if (!a || !b) { free(a); free(b); return ORACLE_ERR_MEMORY; }
    axis_pass_x(v, a, T, H, W, k.x, k.r[2]);
    axis_pass_y(a, b, T, H, W, k.y, k.r[1]);
    axis_pass_t(b, out, T, H, W, k.t, k.r[0]);
    free(a);
    free(b);
    return ORACLE_OK;
}

static void conv_sep(const float* v, float* out, float* tmp, uint32_t T, uint32_t H,
                     uint32_t W, const oracle_kernel* k) {
    axis_pass_x(v, out, T, H, W, k->x, k->r[2]);
    axis_pass_y(out, tmp, T, H, W, k->y, k->r[1]);
    axis_pass_t(tmp, out, T, H, W, k->t, k->r[0]);
}

/* ---- config validation: engine.cpp:21-42 ------------------------------- */

int oracle_validate(const sfseg_params* c) {
    if (!(c->alpha > 0.0)) return ORACLE_ERR_PARAMETER;
    if (c->p < 0.0) return ORACLE_ERR_PARAMETER;
    if (c->iterations < 1) return ORACLE_ERR_PARAMETER;
    if (c->binarize_start < 1) return ORACLE_ERR_PARAMETER;
    if (!(c->sigmoid_slope0 > 0.0)) return ORACLE_ERR_PARAMETER;
    if (!(c->slope_growth >= 1.0)) return ORACLE_ERR_PARAMETER;
    if (!(c->threshold_frac > 0.0 && c->threshold_frac < 1.0)) return ORACLE_ERR_PARAMETER;
    if (!(c->final_threshold > 0.0 && c->final_threshold < 1.0)) return ORACLE_ERR_PARAMETER;
    for (int a = 0; a < 3; ++a)
        if (!(c->sigmas[a] > 0.0)) return ORACLE_ERR_PARAMETER;
    for (int a = 0; a < 3; ++a)
        if (c->radii[a] < 0) return ORACLE_ERR_PARAMETER;
    if (c->temporal_window >= 0 && c->temporal_window < c->radii[0])
        return ORACLE_ERR_PARAMETER;
    if (!c->allow_negative_affinity && c->alpha > 1.0) return ORACLE_ERR_PARAMETER;
    return ORACLE_OK;
}

/* ---- S^p: engine.cpp:52-71 --------------------------------------------- */

void oracle_pow_volume(const float* s, size_t n, double p, float* out) {
    if (p == 0.0) {
        for (size_t i = 0; i < n; ++i) out[i] = 1.0f;
        return;
    }
    if (p == 1.0) {
        memcpy(out, s, n * sizeof(float));
        return;
    }
    for (size_t i = 0; i < n; ++i) out[i] = (float)pow((double)s[i], p);
}

/* ---- one channel: engine.cpp:74-122 ------------------------------------ */

static int step_channel_core(uint32_t T, uint32_t H, uint32_t W, const float* x,
                             const float* sp, const float* f, double alpha,
                             const oracle_kernel* k, float* out, float* w0, float* w1,
                             float* w2, float* tmp) {
    const size_t n = (size_t)T * H * W;
    const float inv_alpha = (float)(1.0 / alpha);
    for (size_t i = 0; i < n; ++i) { /* engine.cpp:92-100 */
        const float sx = sp[i] * x[i];
        const float fi = f[i];
        w0[i] = sx;
        w1[i] = fi * sx;
        w2[i] = fi * fi * sx;
    }
    /* engine.cpp:103-105: conv_a = G*spx, conv_b = G*f2spx, conv_c = G*fspx */
    float* ca = (float*)malloc(n * sizeof(float));
    float* cb = (float*)malloc(n * sizeof(float));
    float* cc = (float*)malloc(n * sizeof(float));
    if (!ca || !cb || !cc) { free(ca); free(cb); free(cc); return ORACLE_ERR_MEMORY; }
    conv_sep(w0, ca, tmp, T, H, W, k);
    conv_sep(w2, cb, tmp, T, H, W, k);
    conv_sep(w1, cc, tmp, T, H, W, k);
    for (size_t i = 0; i < n; ++i) { /* engine.cpp:113-119 */
        const float fi = f[i];
        out[i] = sp[i] * ((inv_alpha - fi * fi) * ca[i] - cb[i] + 2.0f * fi * cc[i]);
    }
    free(ca);
    free(cb);
    free(cc);
    return ORACLE_OK;
}

/* sfseg_step with S^p precomputed (engine.cpp:141-166 minus validate/pow). */
static int step_sp(uint32_t T, uint32_t H, uint32_t W, int32_t C, const float* x,
                   const float* sp, const float* const* F, double alpha,
                   const oracle_kernel* k, float* out) {
    const size_t n = (size_t)T * H * W;
    float* buf = (float*)malloc(5 * n * sizeof(float));
    if (!buf) return ORACLE_ERR_MEMORY;
    float *w0 = buf, *w1 = buf + n, *w2 = buf + 2 * n, *tmp = buf + 3 * n, *term = buf + 4 * n;
    int rc = ORACLE_OK;
    for (int32_t c = 0; c < C && rc == ORACLE_OK; ++c) {
        float* dst = c == 0 ? out : term;
        rc = step_channel_core(T, H, W, x, sp, F[c], alpha, k, dst, w0, w1, w2, tmp);
        if (c > 0) /* engine.cpp:157-162 */
            for (size_t i = 0; i < n; ++i) out[i] += term[i];
    }
    free(buf);
    return rc;
}

int oracle_step(uint32_t T, uint32_t H, uint32_t W, int32_t C, const float* x,
                const float* s, const float* const* F, const sfseg_params* p, float* out) {
    int rc = oracle_validate(p);
    if (rc) return rc;
    if (C < 1) return ORACLE_ERR_PARAMETER; /* engine.cpp:144-145 */
    oracle_kernel k;
    rc = kernel_from(p, &k);
    if (rc) return rc;
    const size_t n = (size_t)T * H * W;
    float* sp = (float*)malloc(n * sizeof(float));
    if (!sp) return ORACLE_ERR_MEMORY;
    oracle_pow_volume(s, n, p->p, sp); /* engine.cpp:148 */
    rc = step_sp(T, H, W, C, x, sp, F, p->alpha, &k, out);
    free(sp);
    return rc;
}

/* ---- normalize_l2: engine.cpp:168-183 ---------------------------------- */

int oracle_normalize_l2(const float* x, size_t n, float* out, double* norm_out) {
    double sumsq = 0.0;
    for (size_t i = 0; i < n; ++i) sumsq += (double)x[i] * (double)x[i];
    const double norm = sqrt(sumsq);
    if (norm_out) *norm_out = norm;
    if (norm == 0.0) return ORACLE_ERR_DEGENERATE;
    const double inv = 1.0 / norm;
    for (size_t i = 0; i < n; ++i) out[i] = (float)((double)x[i] * inv);
    return ORACLE_OK;
}

/* ---- project_binary: engine.cpp:185-205 -------------------------------- */

void oracle_project_binary(const float* x, size_t n, int32_t iter, const sfseg_params* c,
                           float* out) {
    if (iter < c->binarize_start) {
        if (out != x) memcpy(out, x, n * sizeof(float));
        return;
    }
    float maxv = 0.0f;
    for (size_t i = 0; i < n; ++i) maxv = x[i] > maxv ? x[i] : maxv;
    const double theta = c->threshold_frac * (double)maxv;
    const double lambda = c->sigmoid_slope0 * pow(c->slope_growth, iter - c->binarize_start);
    for (size_t i = 0; i < n; ++i) {
        const double z = lambda * ((double)x[i] - theta);
        out[i] = (float)(1.0 / (1.0 + exp(-z)));
    }
}

/* ---- threshold_final: engine.cpp:207-214, volume.cpp:107-114 ------------ */

void oracle_threshold_final(const float* x, size_t n, double frac, uint8_t* mask) {
    float maxv = 0.0f;
    for (size_t i = 0; i < n; ++i) maxv = x[i] > maxv ? x[i] : maxv;
    const float cut = (float)(frac * (double)maxv);
    for (size_t i = 0; i < n; ++i) mask[i] = x[i] > cut ? 1 : 0;
}

/* ---- guard: engine.cpp:228-243 ----------------------------------------- */

void oracle_scale_unit_range(float* f, size_t n) {
    float lo = f[0], hi = f[0];
    for (size_t i = 0; i < n; ++i) {
        lo = f[i] < lo ? f[i] : lo;
        hi = f[i] > hi ? f[i] : hi;
    }
    if (lo >= 0.0f && hi <= 1.0f) return;
    if (hi > lo) {
        const float span = hi - lo;
        for (size_t i = 0; i < n; ++i) f[i] = (f[i] - lo) / span;
    } else {
        const float c = lo < 0.0f ? 0.0f : (lo > 1.0f ? 1.0f : lo);
        for (size_t i = 0; i < n; ++i) f[i] = c;
    }
}

/* ---- validation: volume.cpp:72-93 -------------------------------------- */

static int finite_nonneg(const float* v, size_t n, int need_nonneg) {
    for (size_t i = 0; i < n; ++i) {
        if (!isfinite(v[i])) return ORACLE_ERR_VALIDATION;
        if (need_nonneg && v[i] < 0.0f) return ORACLE_ERR_VALIDATION;
    }
    return ORACLE_OK;
}

/* ---- run: engine.cpp:247-348 (global-step form) ------------------------ */
/*
 * checkpoints: optional array of iteration numbers (ascending, length nck);
 * ck_out receives the iterate x (after normalisation and projection) at each
 * checkpoint, nck * n floats. norms receives the pre-normalisation norm per
 * iteration (p->iterations doubles), may be NULL.
 */
int oracle_run(uint32_t T, uint32_t H, uint32_t W, int32_t C, const float* S,
               const float* const* F, const float* x0, const sfseg_params* p, float* soft,
               uint8_t* mask, double* norms, const int32_t* checkpoints, int32_t nck,
               float* ck_out) {
    int rc = oracle_validate(p);
    if (rc) return rc;
    if (C < 1 || T == 0 || H == 0 || W == 0) return ORACLE_ERR_VALIDATION;
    const size_t n = (size_t)T * H * W;
    rc = finite_nonneg(S, n, 1);
    for (int32_t c = 0; c < C && rc == ORACLE_OK; ++c) rc = finite_nonneg(F[c], n, 0);
    if (rc) return rc;
    if (x0 && finite_nonneg(x0, n, 1)) return ORACLE_ERR_VALIDATION;

    /* engine.cpp:254-259: private copy, guard rescale */
    float* work = (float*)malloc((size_t)C * n * sizeof(float));
    float* sp = (float*)malloc(n * sizeof(float));
    float* x = (float*)malloc(n * sizeof(float));
    float* y = (float*)malloc(n * sizeof(float));
    const float** Fw = (const float**)malloc((size_t)C * sizeof(float*));
    if (!work || !sp || !x || !y || !Fw) {
        free(work); free(sp); free(x); free(y); free(Fw);
        return ORACLE_ERR_MEMORY;
    }
    for (int32_t c = 0; c < C; ++c) {
        memcpy(work + (size_t)c * n, F[c], n * sizeof(float));
        if (!p->allow_negative_affinity) oracle_scale_unit_range(work + (size_t)c * n, n);
        Fw[c] = work + (size_t)c * n;
    }
    memcpy(x, x0 ? x0 : S, n * sizeof(float)); /* engine.cpp:261-270 */
    oracle_kernel k;
    rc = kernel_from(p, &k);
    if (rc == ORACLE_OK) oracle_pow_volume(S, n, p->p, sp); /* engine.cpp:278 */
    int32_t ck = 0;
    for (int32_t iter = 1; iter <= p->iterations && rc == ORACLE_OK; ++iter) {
        rc = step_sp(T, H, W, C, x, sp, Fw, p->alpha, &k, y);
        if (rc) break;
        double norm = 0.0;
        rc = oracle_normalize_l2(y, n, x, &norm); /* engine.cpp:327 */
        if (norms) norms[iter - 1] = norm;
        if (rc) break;
        oracle_project_binary(x, n, iter, p, x); /* engine.cpp:328 */
        if (checkpoints && ck < nck && checkpoints[ck] == iter) {
            memcpy(ck_out + (size_t)ck * n, x, n * sizeof(float));
            ++ck;
        }
    }
    if (rc == ORACLE_OK) {
        if (mask) oracle_threshold_final(x, n, p->final_threshold, mask); /* :344 */
        if (soft) memcpy(soft, x, n * sizeof(float));
    }
    free(work); free(sp); free(x); free(y); free(Fw);
    return rc;
}

/* ---- xoshiro256** restated: rng.hpp:20-75 ------------------------------- */

static uint64_t splitmix64_next(uint64_t* state) {
    *state += 0x9e3779b97f4a7c15ULL;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static uint64_t rotl64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

/* Writes n outputs of next_u64 from a generator seeded with `seed`. */
void oracle_xoshiro_u64(uint64_t seed, uint64_t* out, size_t n) {
    uint64_t s[4], sm = seed;
    for (int i = 0; i < 4; ++i) s[i] = splitmix64_next(&sm);
    for (size_t i = 0; i < n; ++i) {
        const uint64_t result = rotl64(s[1] * 5, 7) * 9;
        const uint64_t t = s[1] << 17;
        s[2] ^= s[0];
        s[3] ^= s[1];
        s[1] ^= s[2];
        s[0] ^= s[3];
        s[2] ^= t;
        s[3] = rotl64(s[3], 45);
        out[i] = result;
    }
}
