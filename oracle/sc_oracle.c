/*
 * sc_oracle.c -- CPU restatement of the one-vector hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * This file is the checker, never the product: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load it.  The product path
 * (paper_2310_10939_b200/) never links or calls anything here.
 *
 * Every routine restates the arithmetic of the reference package `specluster`
 * (/root/reference/pkg/src/specluster) or of the third-party numerics it calls, in
 * the exact floating-point order, so that results are bit-identical:
 *
 *   orc_power_iterate   power_method (spectral.py:87-102) driving either
 *                         rw : lambda x: 0.5*x + 0.5*(A @ (x/d))
 *                         sym: SignlessLaplacianOp.matvec (spectral.py:52-57)
 *                       A @ v is scipy sparsetools csr_matvec: per row, products in
 *                       stored column order, summed left to right from 0, no FMA
 *                       (this file is compiled with -ffp-contract=off).
 *   orc_irwin_hall      x0(u) ~ IW(deg u).  The reference has no
 *                       sampler; the convention is ours:
 *                       uniform j of vertex u = word j%4 of Philox4x64-10 at counter
 *                       (j/4 + 1, u, 0, 0) mapped (raw >> 11) * 2^-53, summed
 *                       sequentially; non-integer degrees add frac(deg) * U_floor(deg).
 *                       numpy.random.Philox(key, counter=[0,u,0,0]).random(m) yields
 *                       the same uniforms (numpy increments the counter first).
 *   orc_kmeanspp        _kmeans_pp_indices + _weighted_index (kmeans.py:116-137)
 *   orc_lloyd_restart   one restart of lloyd (kmeans.py:194-210), with
 *                       _sq_dists_to (:106-113), argmin (:199), _repair_empty (:151-164),
 *                       cluster_means (np.add.at, sequential; :86-93) and kmeans_cost
 *                       (:96-103; numpy einsum "ij,ij->" order: 8192-element buffer
 *                       chunks, two SSE lanes, 4x unrolled reversed -- see
 *                       orc_einsum_sumsq).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>

/* Minimal static row-range parallel-for over pthreads (rows are independent, so the
 * result is bit-identical for every thread count). */
typedef void (*orc_range_fn)(void *ctx, int64_t lo, int64_t hi);
typedef struct { orc_range_fn fn; void *ctx; int64_t lo, hi; } orc_job;
static void *orc_job_run(void *p) { orc_job *j = (orc_job *)p; j->fn(j->ctx, j->lo, j->hi); return NULL; }
static void orc_parallel_for(int64_t n, int32_t nthreads, orc_range_fn fn, void *ctx) {
    if (nthreads <= 1 || n < 4096) { fn(ctx, 0, n); return; }
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    orc_job jobs[256];
    for (int32_t t = 0; t < nthreads; ++t) {
        jobs[t].fn = fn; jobs[t].ctx = ctx;
        jobs[t].lo = n * t / nthreads; jobs[t].hi = n * (t + 1) / nthreads;
        pthread_create(&th[t], NULL, orc_job_run, &jobs[t]);
    }
    for (int32_t t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* ------------------------------------------------------------------------- */
/* Philox4x64-10 (Salmon et al. 2011), the generator behind numpy.random.Philox */

static inline void mulhilo64(uint64_t a, uint64_t b, uint64_t *hi, uint64_t *lo) {
    __uint128_t p = (__uint128_t)a * b;
    *hi = (uint64_t)(p >> 64);
    *lo = (uint64_t)p;
}

void orc_philox4x64_10(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]) {
    uint64_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3];
    uint64_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B97F4A7C15ULL;
            k1 += 0xBB67AE8584CAA73BULL;
        }
        uint64_t h0, l0, h1, l1;
        mulhilo64(0xD2E7470EE14C6C93ULL, x0, &h0, &l0);
        mulhilo64(0xCA5A826395121157ULL, x2, &h1, &l1);
        uint64_t y0 = h1 ^ x1 ^ k0, y2 = h0 ^ x3 ^ k1;
        x0 = y0; x1 = l1; x2 = y2; x3 = l0;
    }
    out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

static inline double u53(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }

/* ------------------------------------------------------------------------- */
/* Irwin-Hall start vector                                                     */

typedef struct { const double *deg; uint64_t key[2]; double *x0; int64_t row0; } ih_ctx;

static void ih_range(void *p, int64_t lo, int64_t hi) {
    ih_ctx *c = (ih_ctx *)p;
    for (int64_t u = lo; u < hi; ++u) {
        double d = c->deg[u];
        double fl = floor(d);
        int64_t m = (int64_t)fl;
        double frac = d - fl;
        int64_t need = m + (frac > 0.0 ? 1 : 0);
        double s = 0.0;
        uint64_t buf[4];
        for (int64_t j = 0; j < need; ++j) {
            if ((j & 3) == 0) {
                uint64_t ctr[4] = {(uint64_t)(j >> 2) + 1u, (uint64_t)(c->row0 + u), 0, 0};
                orc_philox4x64_10(ctr, c->key, buf);
            }
            double un = u53(buf[j & 3]);
            if (j < m) s = s + un;
            else s = s + frac * un;
        }
        c->x0[u] = s;
    }
}

void orc_irwin_hall(int64_t n, const double *deg, uint64_t key0, uint64_t key1, double *x0,
                    int32_t nthreads, int64_t row0) {
    ih_ctx c = {deg, {key0, key1}, x0, row0};
    orc_parallel_for(n, nthreads, ih_range, &c);
}

/* ------------------------------------------------------------------------- */
/* Power iteration                                                             */

typedef struct {
    const int64_t *rp; const int32_t *col; const double *val; const double *deg;
    const double *s; const double *x; const double *z; double *y; double *zo;
    int32_t variant; double half_sgn;
} pi_ctx;

static void pi_scale(void *p, int64_t lo, int64_t hi) {
    pi_ctx *c = (pi_ctx *)p;
    for (int64_t i = lo; i < hi; ++i) c->zo[i] = (c->variant == 1) ? c->s[i] * c->x[i] : c->x[i] / c->deg[i];
}

static void pi_rows(void *p, int64_t lo, int64_t hi) {
    pi_ctx *c = (pi_ctx *)p;
    for (int64_t i = lo; i < hi; ++i) {
        double acc = 0.0;
        for (int64_t j = c->rp[i]; j < c->rp[i + 1]; ++j) {
            double pr = (c->val ? c->val[j] : 1.0) * c->z[c->col[j]];
            acc = acc + pr;
        }
        if (c->variant == 1) acc = c->s[i] * acc;
        c->y[i] = 0.5 * c->x[i] + c->half_sgn * acc;
    }
}

/* variant 0 = lazy random walk  y = 0.5*x + sgn*0.5*(A @ (x/d)),   f = x_T/d
 * variant 1 = signless sym      y = 0.5*x + 0.5*(s*(A @ (s*x))), f = x_T*s, s = 1/sqrt(d)
 * (0.5*x and 0.5*acc are exact, so sgn*0.5 folded into one constant is bit-identical to
 * numpy's 0.5*x + 0.5*(...) and 0.5*x - 0.5*(...).) */
void orc_power_iterate(int64_t n, const int64_t *rp, const int32_t *col, const double *val,
                       const double *deg, const double *x0, int32_t T, int32_t variant,
                       double sgn, double *xT, double *f, int32_t nthreads) {
    double *x = (double *)malloc(sizeof(double) * (size_t)n);
    double *y = (double *)malloc(sizeof(double) * (size_t)n);
    double *z = (double *)malloc(sizeof(double) * (size_t)n);
    double *s = NULL;
    memcpy(x, x0, sizeof(double) * (size_t)n);
    if (variant == 1) {
        s = (double *)malloc(sizeof(double) * (size_t)n);
        for (int64_t i = 0; i < n; ++i) s[i] = 1.0 / sqrt(deg[i]);
    }
    pi_ctx c = {rp, col, val, deg, s, NULL, z, NULL, z, variant, sgn < 0 ? -0.5 : 0.5};
    for (int32_t t = 0; t < T; ++t) {
        c.x = x; c.zo = z;
        orc_parallel_for(n, nthreads, pi_scale, &c);
        c.y = y;
        orc_parallel_for(n, nthreads, pi_rows, &c);
        double *tmp = x; x = y; y = tmp;
    }
    memcpy(xT, x, sizeof(double) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) f[i] = (variant == 1) ? x[i] * s[i] : x[i] / deg[i];
    free(x); free(y); free(z); free(s);
}

/* One rw/sym step for a block of rows given the full gathered vector z (multi-GPU shard
 * oracle): y[i] = 0.5*x[i] + sgn*0.5*sum_j val_j*z[col_j] (sym: scaled by s[i]), then
 * zout[i] = y[i]/deg[i] (sym: y[i]*s[i]).  Same per-row order as orc_power_iterate. */
void orc_rw_rows(int64_t n, const int64_t *rp, const int32_t *col, const double *val,
                 const double *deg, const double *x, const double *z, int32_t variant, double sgn,
                 double *y, double *zout) {
    const double hs = sgn < 0 ? -0.5 : 0.5;
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int64_t j = rp[i]; j < rp[i + 1]; ++j) acc = acc + (val ? val[j] : 1.0) * z[col[j]];
        double s = variant == 1 ? 1.0 / sqrt(deg[i]) : 0.0;
        if (variant == 1) acc = s * acc;
        y[i] = 0.5 * x[i] + hs * acc;
        zout[i] = variant == 1 ? y[i] * s : y[i] / deg[i];
    }
}

/* ------------------------------------------------------------------------- */
/* 1-D k-means replica                                                         */

/* _sq_dists_to for d = 1: ((x*x) - ((2x)*c)) + (c*c), clipped at 0 */
static inline double d2ref(double x, double c) {
    double v = (x * x - (2.0 * x) * c) + c * c;
    return v < 0.0 ? 0.0 : v;
}

/* numpy einsum("ij,ij->", diff, diff) for an (n,1) float64 array (baseline SSE build):
 * the nditer hands the sum-of-products kernel 8192-element buffers; each buffer is summed
 * into two 64-bit lanes, 8 elements per step in the order 6|7, 4|5, 2|3, 0|1, the tail two
 * at a time with zero fill, the lanes added (l0 + l1), and the buffer total added to the
 * running output. */
double orc_einsum_sumsq(int64_t n, const double *v) {
    double out = 0.0;
    for (int64_t c0 = 0; c0 < n; c0 += 8192) {
        int64_t m = (n - c0 < 8192) ? n - c0 : 8192;
        const double *p = v + c0;
        double a0 = 0.0, a1 = 0.0;
        int64_t i = 0;
        for (; m - i >= 8; i += 8) {
            for (int b = 3; b >= 0; --b) {
                a0 = p[i + 2 * b] * p[i + 2 * b] + a0;
                a1 = p[i + 2 * b + 1] * p[i + 2 * b + 1] + a1;
            }
        }
        for (; i < m; i += 2) {
            a0 = p[i] * p[i] + a0;
            double q = (i + 1 < m) ? p[i + 1] : 0.0;
            a1 = q * q + a1;
        }
        out = (a0 + a1) + out;
    }
    return out;
}

/* k-means++ rounds start..k-1 (kmeans.py:121-137).  chosen[0..start-1] are given;
 * u[i-1] is the rng.random() draw of round i.  Returns -1 when all k are chosen, or the
 * round i at which every best_d2 is 0 (the uniform-over-unchosen branch, whose draw the
 * caller replays on the host before resuming at start = i+1). */
int32_t orc_kmeanspp(int64_t n, const double *x, int32_t k, int32_t start, const double *u,
                     int64_t *chosen) {
    double *best = (double *)malloc(sizeof(double) * (size_t)n);
    for (int64_t j = 0; j < n; ++j) best[j] = d2ref(x[j], x[chosen[0]]);
    for (int32_t i = 1; i < start; ++i)
        for (int64_t j = 0; j < n; ++j) {
            double d = d2ref(x[j], x[chosen[i]]);
            if (d < best[j]) best[j] = d;
        }
    int32_t ret = -1;
    for (int32_t i = start; i < k; ++i) {
        int any = 0;
        for (int64_t j = 0; j < n && !any; ++j) any = best[j] > 0.0;
        if (!any) { ret = i; break; }
        double tot = 0.0;
        for (int64_t j = 0; j < n; ++j) tot = tot + best[j];
        double r = u[i - 1] * tot;
        double cum = 0.0;
        int64_t idx = n - 1;
        for (int64_t j = 0; j < n; ++j) {
            cum = cum + best[j];
            if (cum > r) { idx = j; break; }
        }
        chosen[i] = idx;
        double c = x[idx];
        for (int64_t j = 0; j < n; ++j) {
            double d = d2ref(x[j], c);
            if (d < best[j]) best[j] = d;
        }
    }
    free(best);
    return ret;
}

/* One restart of lloyd from the given centers.  labels_out gets the final labels,
 * *cost_out the final cost, return value = iterations run. */
int32_t orc_lloyd_restart(int64_t n, const double *x, int32_t k, const double *centers0,
                          int32_t max_iters, double tol, int64_t *labels_out, double *cost_out) {
    double *cen = (double *)malloc(sizeof(double) * (size_t)k);
    double *sums = (double *)malloc(sizeof(double) * (size_t)k);
    int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
    int64_t *lab = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    double *own = (double *)malloc(sizeof(double) * (size_t)n);
    double *diff = (double *)malloc(sizeof(double) * (size_t)n);
    int32_t *empties = (int32_t *)malloc(sizeof(int32_t) * (size_t)k);
    memcpy(cen, centers0, sizeof(double) * (size_t)k);
    for (int64_t j = 0; j < n; ++j) labels_out[j] = 0;
    double prev = INFINITY;
    int32_t it = 0;
    while (it < max_iters) {
        ++it;
        for (int64_t j = 0; j < n; ++j) {
            int32_t bi = 0;
            double bd = d2ref(x[j], cen[0]);
            for (int32_t c = 1; c < k; ++c) {
                double d = d2ref(x[j], cen[c]);
                if (d < bd) { bd = d; bi = c; }
            }
            lab[j] = bi;
            own[j] = bd;
        }
        /* _repair_empty */
        for (int32_t c = 0; c < k; ++c) cnt[c] = 0;
        for (int64_t j = 0; j < n; ++j) cnt[lab[j]]++;
        int32_t ne = 0;
        for (int32_t c = 0; c < k; ++c) if (cnt[c] == 0) empties[ne++] = c;
        for (int32_t e = 0; e < ne; ++e) {
            int64_t far = 0;
            for (int64_t j = 1; j < n; ++j) if (own[j] > own[far]) far = j;
            cnt[lab[far]]--;
            lab[far] = empties[e];
            cnt[empties[e]] = 1;
            own[far] = 0.0;
        }
        int unchanged = isfinite(prev);
        if (unchanged)
            for (int64_t j = 0; j < n; ++j) if (lab[j] != labels_out[j]) { unchanged = 0; break; }
        memcpy(labels_out, lab, sizeof(int64_t) * (size_t)n);
        /* cluster_means: np.add.at, sequential in index order */
        for (int32_t c = 0; c < k; ++c) { sums[c] = 0.0; cnt[c] = 0; }
        for (int64_t j = 0; j < n; ++j) { sums[lab[j]] = sums[lab[j]] + x[j]; cnt[lab[j]]++; }
        for (int32_t c = 0; c < k; ++c) cen[c] = cnt[c] > 0 ? sums[c] / (double)cnt[c] : sums[c];
        for (int64_t j = 0; j < n; ++j) diff[j] = x[j] - cen[lab[j]];
        double cost = orc_einsum_sumsq(n, diff);
        if (!(cost <= prev * (1.0 + 1e-12) + 1e-12)) { /* kmeans.py:206 assert */
            it = -it;
            prev = cost;
            break;
        }
        int small_gain = isfinite(prev) && (prev - cost <= tol * (prev > 1e-300 ? prev : 1e-300));
        prev = cost;
        if (unchanged || small_gain) break;
    }
    *cost_out = prev;
    free(cen); free(sums); free(cnt); free(lab); free(own); free(diff); free(empties);
    return it; /* iterations run; negative: the cost assertion failed at iteration -it */
}
