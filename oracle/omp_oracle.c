/*
 * oracle/omp_oracle.c -- CPU restatement of the reference's batched OMP kernel.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product
 * path: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load this library, and only as the checker or
 * the timed CPU baseline.
 *
 * What it restates (file:line in /root/reference):
 *   pkg/src/crossdict/_kernels.py:27-42   _dot4  (4 fixed accumulators, tail added last)
 *   pkg/src/crossdict/_kernels.py:45-47   _norm
 *   pkg/src/crossdict/_kernels.py:50-168  omp_batch_kernel (scan, strict '>' select,
 *                                          MGS x2 with RANK_TOL, residual update,
 *                                          dense min-norm fallback, back-substitution)
 *   pkg/src/crossdict/_kernels.py:24      RANK_TOL = 1e-10
 *
 * Arithmetic: IEEE fp64, no FMA contraction (built with -ffp-contract=off),
 * identical operation order to the numba kernel (which is compiled with
 * fastmath=False), so non-fallback outputs are bit-identical to the
 * reference; tests/test_oracle.py pins that against tests/golden/.
 *
 * The one place the reference calls a library is the rank-deficient dense
 * mode, np.linalg.lstsq(rcond=-1) (LAPACK dgelsd, _kernels.py:145).  Here it
 * is restated as a one-sided Jacobi SVD minimum-norm solve.  Coefficients in
 * that mode are "parity unpinned" (the reference tests only check the flag,
 * the support and finiteness: pkg/tests/test_pursuit.py:131-139).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define RANK_TOL 1e-10

/* _kernels.py:27-42 */
static double dot4(const double *a, const double *b, int64_t n) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int64_t m4 = (n / 4) * 4;
    for (int64_t i = 0; i < m4; i += 4) {
        s0 += a[i] * b[i];
        s1 += a[i + 1] * b[i + 1];
        s2 += a[i + 2] * b[i + 2];
        s3 += a[i + 3] * b[i + 3];
    }
    double s = s0 + s1 + s2 + s3;
    for (int64_t i = m4; i < n; i++) s += a[i] * b[i];
    return s;
}

static double norm2(const double *a, int64_t n) { return sqrt(dot4(a, a, n)); }

/*
 * Minimum-norm least squares x = argmin ||A x - y|| with smallest ||x||,
 * A is n x m stored column-major in `a` (overwritten).  One-sided Jacobi SVD
 * (Hestenes); singular values below eps*sigma_max are treated as zero, the
 * rank rule np.linalg.lstsq(rcond=-1) applies (machine precision cut-off).
 * work: m*m doubles for V.
 */
static void lstsq_min_norm(double *a, int64_t n, int64_t m, const double *y,
                           double *x, double *v) {
    for (int64_t i = 0; i < m * m; i++) v[i] = 0.0;
    for (int64_t i = 0; i < m; i++) v[i * m + i] = 1.0;
    const double eps = 1.1102230246251565e-16; /* 2^-53 */
    for (int sweep = 0; sweep < 80; sweep++) {
        int rotated = 0;
        for (int64_t p = 0; p < m - 1; p++) {
            for (int64_t q = p + 1; q < m; q++) {
                double *ap = a + p * n, *aq = a + q * n;
                double alpha = 0.0, beta = 0.0, gamma = 0.0;
                for (int64_t i = 0; i < n; i++) {
                    alpha += ap[i] * ap[i];
                    beta += aq[i] * aq[i];
                    gamma += ap[i] * aq[i];
                }
                if (gamma == 0.0 || fabs(gamma) <= eps * sqrt(alpha * beta)) continue;
                rotated = 1;
                double zeta = (beta - alpha) / (2.0 * gamma);
                double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                double c = 1.0 / sqrt(1.0 + t * t);
                double s = c * t;
                for (int64_t i = 0; i < n; i++) {
                    double xp = ap[i], xq = aq[i];
                    ap[i] = c * xp - s * xq;
                    aq[i] = s * xp + c * xq;
                }
                double *vp = v + p * m, *vq = v + q * m;
                for (int64_t i = 0; i < m; i++) {
                    double xp = vp[i], xq = vq[i];
                    vp[i] = c * xp - s * xq;
                    vq[i] = s * xp + c * xq;
                }
            }
        }
        if (!rotated) break;
    }
    double smax = 0.0;
    for (int64_t j = 0; j < m; j++) {
        double s2 = 0.0;
        for (int64_t i = 0; i < n; i++) s2 += a[j * n + i] * a[j * n + i];
        double s = sqrt(s2);
        if (s > smax) smax = s;
    }
    for (int64_t i = 0; i < m; i++) x[i] = 0.0;
    for (int64_t j = 0; j < m; j++) {
        double s2 = 0.0, uy = 0.0;
        for (int64_t i = 0; i < n; i++) {
            s2 += a[j * n + i] * a[j * n + i];
            uy += a[j * n + i] * y[i];
        }
        double s = sqrt(s2);
        if (!(s > eps * smax) || s == 0.0) continue;
        double f = uy / s2; /* (u_j . y) / sigma_j  with a_j = sigma_j u_j */
        for (int64_t i = 0; i < m; i++) x[i] += v[j * m + i] * f;
    }
}

/* One signal of omp_batch_kernel (_kernels.py:68-168). */
static void omp_one(const double *mat_t, int64_t t, int64_t n, const double *y,
                    int64_t k_max, double tol, const int64_t *allowed_row,
                    int64_t s_allowed, int restricted, int64_t *sel, double *coef,
                    int64_t *count, double *rnorm_out, int64_t *scans_out,
                    uint8_t *flag, double *work) {
    int64_t c = restricted ? s_allowed : t;
    double ynorm = norm2(y, n);
    *count = 0;
    *rnorm_out = ynorm;
    *scans_out = 0;
    *flag = 0;
    if (ynorm <= tol) return;

    /* scratch layout */
    double *r = work;                          /* n */
    double *qmat = r + n;                      /* k_max * n */
    double *rmat = qmat + k_max * n;           /* k_max * k_max */
    double *qty = rmat + k_max * k_max;        /* k_max */
    double *u = qty + k_max;                   /* n */
    double *amat = u + n;                      /* n * k_max (column-major) */
    double *coefs = amat + n * k_max;          /* k_max */
    double *vwork = coefs + k_max;             /* k_max * k_max */
    uint8_t *taken = (uint8_t *)(vwork + k_max * k_max); /* c */

    memcpy(r, y, (size_t)n * sizeof(double));
    for (int64_t i = 0; i < k_max * k_max; i++) rmat[i] = 0.0;
    memset(taken, 0, (size_t)c);
    int64_t scans = 0, kdone = 0;
    double rnorm = ynorm;
    int dense = 0;

    for (int64_t k = 0; k < k_max; k++) {
        scans += c - k;
        double best = -1.0;
        int64_t bestj = -1;
        for (int64_t jl = 0; jl < c; jl++) {
            if (taken[jl]) continue;
            int64_t g = restricted ? allowed_row[jl] : jl;
            double v = dot4(mat_t + g * n, r, n);
            if (v < 0.0) v = -v;
            if (v > best) {
                best = v;
                bestj = jl;
            }
        }
        if (bestj < 0 || best <= 0.0) break;
        taken[bestj] = 1;
        int64_t g = restricted ? allowed_row[bestj] : bestj;
        sel[kdone] = g;
        kdone += 1;

        if (!dense) {
            memcpy(u, mat_t + g * n, (size_t)n * sizeof(double));
            double anorm = norm2(u, n);
            for (int64_t j = 0; j < kdone - 1; j++) {
                double w = dot4(qmat + j * n, u, n);
                for (int64_t i = 0; i < n; i++) u[i] -= w * qmat[j * n + i];
                rmat[j * k_max + (kdone - 1)] = w;
            }
            for (int64_t j = 0; j < kdone - 1; j++) {
                double w2 = dot4(qmat + j * n, u, n);
                for (int64_t i = 0; i < n; i++) u[i] -= w2 * qmat[j * n + i];
                rmat[j * k_max + (kdone - 1)] += w2;
            }
            double d = norm2(u, n);
            double floor_ = anorm > 1e-300 ? anorm : 1e-300;
            if (d <= RANK_TOL * floor_) {
                dense = 1;
                *flag = 1;
            } else {
                rmat[(kdone - 1) * k_max + (kdone - 1)] = d;
                double *qk = qmat + (kdone - 1) * n;
                for (int64_t i = 0; i < n; i++) qk[i] = u[i] / d;
                double z = dot4(qk, r, n);
                qty[kdone - 1] = z;
                for (int64_t i = 0; i < n; i++) r[i] -= z * qk[i];
                rnorm = norm2(r, n);
            }
        }
        if (dense) {
            for (int64_t j = 0; j < kdone; j++)
                memcpy(amat + j * n, mat_t + sel[j] * n, (size_t)n * sizeof(double));
            lstsq_min_norm(amat, n, kdone, y, coefs, vwork);
            for (int64_t i = 0; i < n; i++) {
                double acc = 0.0;
                for (int64_t j = 0; j < kdone; j++) acc += mat_t[sel[j] * n + i] * coefs[j];
                r[i] = y[i] - acc;
            }
            rnorm = norm2(r, n);
            for (int64_t j = 0; j < kdone; j++) coef[j] = coefs[j];
        }
        if (rnorm <= tol) break;
    }
    if (kdone && !dense) {
        for (int64_t i = kdone - 1; i >= 0; i--) {
            double acc = qty[i];
            for (int64_t j = i + 1; j < kdone; j++) acc -= rmat[i * k_max + j] * coef[j];
            coef[i] = acc / rmat[i * k_max + i];
        }
    }
    *count = kdone;
    *rnorm_out = rnorm;
    *scans_out = scans;
}

/*
 * Batched entry point with the reference kernel's argument list
 * (_kernels.py:51).  Outputs must be pre-initialised by the caller exactly as
 * pursuit._run_kernel does (pursuit.py:240-245): sel = -1, coef = 0.
 * nthreads > 1 splits signals into contiguous chunks over pthreads (signals
 * are independent); results do not depend on nthreads.
 */
typedef struct {
    const double *mat_t; int64_t t, n; const double *ys; int64_t p0, p1, k_max;
    const double *eps; const int64_t *allowed; int64_t s_allowed; int restricted;
    int64_t *out_sel; double *out_coef; int64_t *out_count; double *out_rnorm;
    int64_t *out_scans; uint8_t *out_flag; int failed;
} chunk_t;

static void *run_chunk(void *arg) {
    chunk_t *a = (chunk_t *)arg;
    int64_t c = a->restricted ? a->s_allowed : a->t;
    int64_t n = a->n, k_max = a->k_max;
    size_t work_doubles = (size_t)(n + k_max * n + k_max * k_max + k_max + n + n * k_max +
                                   k_max + k_max * k_max) + (size_t)(c / 8 + 2);
    double *work = (double *)malloc(work_doubles * sizeof(double));
    if (!work) { a->failed = 1; return NULL; }
    for (int64_t p = a->p0; p < a->p1; p++) {
        omp_one(a->mat_t, a->t, n, a->ys + p * n, k_max, a->eps[p],
                a->restricted ? a->allowed + p * a->s_allowed : NULL, a->s_allowed,
                a->restricted, a->out_sel + p * k_max, a->out_coef + p * k_max,
                a->out_count + p, a->out_rnorm + p, a->out_scans + p, a->out_flag + p, work);
    }
    free(work);
    return NULL;
}

int oracle_omp_batch(const double *mat_t, int64_t t, int64_t n, const double *ys,
                     int64_t p_all, int64_t k_max, const double *eps,
                     const int64_t *allowed, int64_t s_allowed, int restricted,
                     int64_t *out_sel, double *out_coef, int64_t *out_count,
                     double *out_rnorm, int64_t *out_scans, uint8_t *out_flag,
                     int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if (nthreads > p_all) nthreads = p_all > 0 ? (int)p_all : 1;
    chunk_t chunks[256];
    pthread_t tids[256];
    int64_t per = (p_all + nthreads - 1) / nthreads;
    for (int i = 0; i < nthreads; i++) {
        chunk_t ch = {mat_t, t, n, ys, i * per, (i + 1) * per < p_all ? (i + 1) * per : p_all,
                      k_max, eps, allowed, s_allowed, restricted, out_sel, out_coef,
                      out_count, out_rnorm, out_scans, out_flag, 0};
        if (ch.p0 > ch.p1) ch.p0 = ch.p1;
        chunks[i] = ch;
    }
    for (int i = 1; i < nthreads; i++) pthread_create(&tids[i], NULL, run_chunk, &chunks[i]);
    run_chunk(&chunks[0]);
    for (int i = 1; i < nthreads; i++) pthread_join(tids[i], NULL);
    for (int i = 0; i < nthreads; i++) if (chunks[i].failed) return -1;
    return 0;
}
