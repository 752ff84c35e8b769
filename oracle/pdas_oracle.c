/*
 * pdas_oracle.c -- CPU restatement of the reference kernel core.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the reported CPU baseline -- never as the product
 * path (the product is paper_1502_03543_b200/csrc, CUDA only, no CPU fallback).
 *
 * Restates the arithmetic of /root/reference/pkg/src/adascale/_kernels.pyx
 * (the compiled core, which SURVEY.md §8c names as THE oracle) in plain C.
 * Every function below cites the routine it follows.  Build flags must keep
 * -ffp-contract=off (reference pkg/setup.py:22) so products and sums round
 * separately; see oracle/Makefile.
 *
 * Layout: every matrix is column-contiguous, element (i,j) at j*rows+i
 * (reference linalg.py:1-7).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef int64_t idx_t;

static const double DENOM_EPS_REL = 1e-12; /* _kernels.pyx:21-23 */

static idx_t pow2_ceil(idx_t k) /* _kernels.pyx:26-30 */
{
    idx_t p = 1;
    while (p < k) p <<= 1;
    return p;
}

/* Fixed pairwise tree over products u[i]*v[i] (_kernels.pyx:33-52).
 * Level 0 folds the upper half onto the lower half ("add during load",
 * PAPER.md:127), padding with +0.0 past n; then halves until one value
 * remains.  `work` needs pow2_ceil(n)/2 doubles. */
static double tree_dot(const double *u, idx_t su, const double *v, idx_t sv,
                       idx_t n, double *work)
{
    if (n == 1) return u[0] * v[0];
    idx_t h = pow2_ceil(n) >> 1;
    for (idx_t i = 0; i < h; ++i) {
        double upper = 0.0;
        idx_t j = i + h;
        if (j < n) upper = u[j * su] * v[j * sv];
        double lower = u[i * su] * v[i * sv];
        work[i] = lower + upper;
    }
    for (h >>= 1; h >= 1; h >>= 1)
        for (idx_t i = 0; i < h; ++i) work[i] = work[i] + work[i + h];
    return work[0];
}

static double *work_alloc(idx_t n)
{
    idx_t h = pow2_ceil(n) >> 1;
    if (h < 1) h = 1;
    return (double *)malloc((size_t)h * sizeof(double));
}

/* dot_tree (_kernels.pyx:55-71) */
int or_dot_tree(const double *u, idx_t su, const double *v, idx_t sv, idx_t n, double *out)
{
    double *w = work_alloc(n);
    if (!w) return -1;
    *out = tree_dot(u, su, v, sv, n, w);
    free(w);
    return 0;
}

/* mat_vec (_kernels.pyx:74-88): out[i] = tree_k a[i,k]*x[k] (row stride m). */
int or_mat_vec(const double *a, idx_t m, idx_t n, const double *x, double *out)
{
    double *w = work_alloc(n);
    if (!w) return -1;
    for (idx_t i = 0; i < m; ++i) out[i] = tree_dot(a + i, m, x, 1, n, w);
    free(w);
    return 0;
}

/* mat_t_vec (_kernels.pyx:91-105): out[j] = tree_i a[i,j]*y[i]. */
int or_mat_t_vec(const double *a, idx_t m, idx_t n, const double *y, double *out)
{
    double *w = work_alloc(m);
    if (!w) return -1;
    for (idx_t j = 0; j < n; ++j) out[j] = tree_dot(a + j * m, 1, y, 1, m, w);
    free(w);
    return 0;
}

/* gram / scaled_gram (_kernels.pyx:108-141): upper triangle accumulated with
 * k as the OUTER loop (each g[i,j] sums its k terms in ascending order from
 * +0.0), then mirrored.  With d != NULL the right factor is a[j,k]*d[k],
 * rounded before the product (scaled_gram). */
void or_gram(const double *a, idx_t m, idx_t n, const double *d, double *g)
{
    memset(g, 0, (size_t)(m * m) * sizeof(double));
    for (idx_t k = 0; k < n; ++k) {
        const double *ak = a + k * m;
        for (idx_t j = 0; j < m; ++j) {
            double r = d ? ak[j] * d[k] : ak[j];
            double *gj = g + j * m;
            for (idx_t i = 0; i <= j; ++i) gj[i] = gj[i] + ak[i] * r;
        }
    }
    for (idx_t j = 0; j < m; ++j)
        for (idx_t i = j + 1; i < m; ++i) g[j * m + i] = g[i * m + j];
}

/* cholesky_factor (_kernels.pyx:144-171): left-looking, column by column.
 * Returns the first failing column or -1.  `low` must be zeroed by us. */
idx_t or_cholesky_factor(const double *g, idx_t nn, double eps_rel, double *low)
{
    memset(low, 0, (size_t)(nn * nn) * sizeof(double));
    double dmax = 0.0;
    for (idx_t j = 0; j < nn; ++j)
        if (g[j * nn + j] > dmax) dmax = g[j * nn + j];
    double eps = eps_rel * dmax;
    for (idx_t j = 0; j < nn; ++j) {
        double s = g[j * nn + j];
        for (idx_t k = 0; k < j; ++k) s -= low[k * nn + j] * low[k * nn + j];
        if (!isfinite(s) || s <= eps) return j;
        double piv = sqrt(s);
        low[j * nn + j] = piv;
        for (idx_t i = j + 1; i < nn; ++i) {
            double t = g[j * nn + i];
            for (idx_t k = 0; k < j; ++k) t -= low[k * nn + i] * low[k * nn + j];
            low[j * nn + i] = t / piv;
        }
    }
    return -1;
}

/* cholesky_solve_many (_kernels.pyx:174-193), in place on x (m x k). */
void or_cholesky_solve_many(const double *low, idx_t m, double *x, idx_t k)
{
    for (idx_t c = 0; c < k; ++c) {
        double *xc = x + c * m;
        for (idx_t i = 0; i < m; ++i) {
            double s = xc[i];
            for (idx_t j = 0; j < i; ++j) s -= low[j * m + i] * xc[j];
            xc[i] = s / low[i * m + i];
        }
        for (idx_t i = m - 1; i >= 0; --i) {
            double s = xc[i];
            for (idx_t j = i + 1; j < m; ++j) s -= low[i * m + j] * xc[j];
            xc[i] = s / low[i * m + i];
        }
    }
}

/* build_v (_kernels.pyx:196-202) */
void or_build_v(const double *a, idx_t m, idx_t l0, double dl, double *v)
{
    double f = dl - 1.0;
    for (idx_t i = 0; i < m; ++i) v[i] = a[l0 * m + i] * f;
}

/* sweep_phase1 (_kernels.pyx:205-218) */
int or_sweep_phase1(const double *cols, idx_t m, const double *v, double *inner, idx_t k0, idx_t k1)
{
    double *w = work_alloc(m);
    if (!w) return -1;
    for (idx_t k = k0; k < k1; ++k) inner[k] = tree_dot(v, 1, cols + k * m, 1, m, w);
    free(w);
    return 0;
}

/* sweep_phase2 (_kernels.pyx:221-231) */
void or_sweep_phase2(double *cols, idx_t m, idx_t l0, const double *inner, double denom,
                     idx_t k0, idx_t k1)
{
    const double *piv = cols + l0 * m;
    for (idx_t k = k0; k < k1; ++k) {
        double g = inner[k] / denom;
        double *ck = cols + k * m;
        for (idx_t i = 0; i < m; ++i) ck[i] = ck[i] - g * piv[i];
    }
}

/* solve_sweeps / _cascade (_kernels.pyx:234-291): the full Egidi-Maponi
 * cascade in place; 0 or the 1-based breakdown step.  Column loops are
 * split over `workers` OpenMP threads; column arithmetic is independent of
 * the split, so every worker count gives the same bits. */
int or_solve_sweeps(double *cols, const double *a, const double *d, double *inner, double *v,
                    idx_t m, idx_t n, int workers)
{
    int nt = workers > 1 ? workers : 1;
    idx_t half = pow2_ceil(m) >> 1;
    if (half < 1) half = 1;
    double *work = (double *)malloc((size_t)(nt * half) * sizeof(double));
    if (!work) return -1;
    int fail = 0;
    for (idx_t l0 = 0; l0 < n; ++l0) {
        double dl = d[l0];
        if (dl == 1.0) continue;
        or_build_v(a, m, l0, dl, v);
#pragma omp parallel for num_threads(nt) schedule(static)
        for (idx_t k = l0; k <= n; ++k) {
            int t = 0;
#ifdef _OPENMP
            t = omp_get_thread_num();
#endif
            inner[k] = tree_dot(v, 1, cols + k * m, 1, m, work + (idx_t)t * half);
        }
        double denom = 1.0 + inner[l0];
        if (fabs(denom) <= DENOM_EPS_REL * (1.0 + fabs(inner[l0]))) {
            fail = (int)(l0 + 1);
            break;
        }
        const double *piv = cols + l0 * m;
#pragma omp parallel for num_threads(nt) schedule(static)
        for (idx_t k = l0 + 1; k <= n; ++k) {
            double g = inner[k] / denom;
            double *ck = cols + k * m;
            for (idx_t i = 0; i < m; ++i) ck[i] = ck[i] - g * piv[i];
        }
    }
    free(work);
    return fail;
}

/* Bounded cascade sample for CPU baselines: runs steps [0, steps) only. */
int or_solve_sweeps_prefix(double *cols, const double *a, const double *d, double *inner,
                           double *v, idx_t m, idx_t n, idx_t steps, int workers)
{
    double *dd = (double *)malloc((size_t)n * sizeof(double));
    if (!dd) return -1;
    for (idx_t l = 0; l < n; ++l) dd[l] = l < steps ? d[l] : 1.0;
    int r = or_solve_sweeps(cols, a, dd, inner, v, m, n, workers);
    free(dd);
    return r;
}
