/*
 * TEST INFRASTRUCTURE ONLY -- not part of the product path.
 *
 * CPU restatement of the reference (sembench) hot path, used as the parity
 * checker by tests/, by __graft_entry__.smoke() and as the CPU baseline leg
 * of bench.py ("cpu_baseline.kind" = "port").  Nothing under
 * paper_2005_13425_b200/ may link or call this file.
 *
 * Every routine reproduces the reference's arithmetic ORDER so that results
 * are bit-identical to sembench (pinned by tests/test_oracle_golden.py against
 * fixtures generated from the reference itself, tests/golden/make_golden.py):
 *
 *   oracle_ax_layered   sembench/kernels.py:267-329 (_ax_layered_generic);
 *                       at n = 10 the reference dispatches to :332-410 whose
 *                       sums start from the first product instead of 0.0 --
 *                       identical except for the sign of an all-zero sum.
 *   oracle_ax_reference sembench/kernels.py:159-205 (REFERENCE: three full
 *                       passes through E*n^3 intermediates ur/us/ut, which
 *                       hold the metric-scaled gradients on return)
 *   oracle_ax_scratch   sembench/kernels.py:213-259 (SCRATCH: element staged,
 *                       phase 2 reads D transposed in place of diff_t)
 *   oracle_dssum        sembench/assembly.py:113-120 (np.bincount order:
 *                       ascending local index, accumulator starts at +0.0)
 *   oracle_wdot3        sembench/cg.py:77-92 (65536-point chunks, in order)
 *   oracle_axpy_into    sembench/cg.py:95-98   x += alpha*y  (no FMA)
 *   oracle_scale_add    sembench/cg.py:101-104 p = beta*p + z (no FMA)
 *   oracle_mask         sembench/assembly.py:123-129  f*mask
 *
 * Build: oracle/Makefile (gcc -O2 -fopenmp -ffp-contract=off).  FP
 * contraction is disabled so a*b+c is never fused, matching numba/LLVM
 * without fastmath.  OpenMP only splits disjoint element ranges or disjoint
 * chunks, so results do not depend on the thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define WDOT_CHUNK 65536

static void set_threads(int nthreads)
{
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* One element of the layered operator.  Index conventions follow the field
 * layout [e][k][j][i] (i fastest).  Scratch: col_u[j][i][l] holds the u
 * column of point (i,j) along k, col_w[j][i][kk] the output accumulators,
 * lay_* one k-layer of intermediates. */
static void ax_layered_one(int n, const double *ue, const double *ge,
                           const double *dx, const double *dxt, double *we,
                           double *col_u, double *col_w, double *lay_u,
                           double *lay_r, double *lay_s, double *lay_t)
{
    const int nn = n * n, nnn = n * n * n;
    for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i)
                col_u[(j * n + i) * n + k] = ue[(k * n + j) * n + i];
    memset(col_w, 0, sizeof(double) * (size_t)nnn);

    for (int k = 0; k < n; ++k) {
        for (int ji = 0; ji < nn; ++ji)
            lay_u[ji] = col_u[ji * n + k];
        /* phase 1: three directional derivatives + metric, finalized per layer */
        for (int j = 0; j < n; ++j) {
            for (int i = 0; i < n; ++i) {
                double dr = 0.0, ds = 0.0, dt = 0.0;
                const double *ucol = col_u + (j * n + i) * n;
                for (int l = 0; l < n; ++l) {
                    dr += dx[i * n + l] * lay_u[j * n + l];
                    ds += dx[j * n + l] * lay_u[l * n + i];
                    dt += dx[k * n + l] * ucol[l];
                }
                const size_t p = (size_t)(k * n + j) * n + i;
                const double g1 = ge[0 * nnn + p], g2 = ge[1 * nnn + p];
                const double g3 = ge[2 * nnn + p], g4 = ge[3 * nnn + p];
                const double g5 = ge[4 * nnn + p], g6 = ge[5 * nnn + p];
                lay_r[j * n + i] = g1 * dr + g2 * ds + g3 * dt;
                lay_s[j * n + i] = g2 * dr + g4 * ds + g5 * dt;
                lay_t[j * n + i] = g3 * dr + g5 * ds + g6 * dt;
            }
        }
        /* phase 2: transpose contractions; t-direction scatters down the column */
        for (int j = 0; j < n; ++j) {
            for (int i = 0; i < n; ++i) {
                double ar = 0.0, as = 0.0;
                for (int l = 0; l < n; ++l) {
                    ar += dxt[i * n + l] * lay_r[j * n + l];
                    as += dxt[j * n + l] * lay_s[l * n + i];
                }
                double *wcol = col_w + (j * n + i) * n;
                wcol[k] += ar + as;
                const double tv = lay_t[j * n + i];
                for (int kk = 0; kk < n; ++kk)
                    wcol[kk] += dxt[kk * n + k] * tv;
            }
        }
    }
    for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i)
                we[(k * n + j) * n + i] = col_w[(j * n + i) * n + k];
}

int oracle_ax_layered(const double *u, const double *g, const double *dx,
                      const double *dxt, double *w, int64_t num_elements, int n,
                      int nthreads)
{
    if (n < 2 || n > 16 || num_elements < 0) return 1;
    set_threads(nthreads);
    const int64_t nnn = (int64_t)n * n * n;
    int status = 0;
#pragma omp parallel
    {
        const size_t scratch = (size_t)(2 * nnn + 4 * n * n);
        double *buf = (double *)malloc(sizeof(double) * scratch);
        if (!buf) {
#pragma omp atomic write
            status = 2;
        } else {
            double *col_u = buf, *col_w = buf + nnn;
            double *lay = buf + 2 * nnn;
#pragma omp for schedule(static)
            for (int64_t e = 0; e < num_elements; ++e)
                ax_layered_one(n, u + e * nnn, g + e * 6 * nnn, dx, dxt, w + e * nnn,
                               col_u, col_w, lay, lay + n * n, lay + 2 * n * n,
                               lay + 3 * n * n);
            free(buf);
        }
    }
    return status;
}

/* REFERENCE variant: derivative pass -> geometric pass (in place) ->
 * transpose pass, each over all elements.  Sums start at 0.0 and add the
 * l-th product in ascending l; the transpose pass interleaves r, s, t terms
 * per l (kernels.py:196-203). */
int oracle_ax_reference(const double *u, const double *g, const double *dx,
                        const double *dxt, double *ur, double *us, double *ut, double *w,
                        int64_t num_elements, int n, int nthreads)
{
    if (n < 2 || n > 16 || num_elements < 0) return 1;
    set_threads(nthreads);
    const int64_t nnn = (int64_t)n * n * n;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < num_elements; ++e) {
        const double *ue = u + e * nnn;
        for (int k = 0; k < n; ++k)
            for (int j = 0; j < n; ++j)
                for (int i = 0; i < n; ++i) {
                    double ar = 0.0, as = 0.0, at = 0.0;
                    for (int l = 0; l < n; ++l) {
                        ar += dx[i * n + l] * ue[(k * n + j) * n + l];
                        as += dx[j * n + l] * ue[(k * n + l) * n + i];
                        at += dx[k * n + l] * ue[(l * n + j) * n + i];
                    }
                    const int64_t q = e * nnn + (k * n + j) * n + i;
                    ur[q] = ar;
                    us[q] = as;
                    ut[q] = at;
                }
    }
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < num_elements; ++e)
        for (int64_t p = 0; p < nnn; ++p) {
            const int64_t q = e * nnn + p;
            const double *ge = g + e * 6 * nnn + p;
            const double wr = ur[q], ws = us[q], wt = ut[q];
            const double g1 = ge[0], g2 = ge[nnn], g3 = ge[2 * nnn];
            const double g4 = ge[3 * nnn], g5 = ge[4 * nnn], g6 = ge[5 * nnn];
            ur[q] = g1 * wr + g2 * ws + g3 * wt;
            us[q] = g2 * wr + g4 * ws + g5 * wt;
            ut[q] = g3 * wr + g5 * ws + g6 * wt;
        }
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < num_elements; ++e) {
        const double *re = ur + e * nnn, *se = us + e * nnn, *te = ut + e * nnn;
        for (int k = 0; k < n; ++k)
            for (int j = 0; j < n; ++j)
                for (int i = 0; i < n; ++i) {
                    double acc = 0.0;
                    for (int l = 0; l < n; ++l) {
                        acc += dxt[i * n + l] * re[(k * n + j) * n + l];
                        acc += dxt[j * n + l] * se[(k * n + l) * n + i];
                        acc += dxt[k * n + l] * te[(l * n + j) * n + i];
                    }
                    w[e * nnn + (k * n + j) * n + i] = acc;
                }
    }
    return 0;
}

/* SCRATCH variant: per element, phase 1 with the metric applied per point,
 * then phase 2 with D read transposed (sd[l][i] for diff_t[i][l]). */
int oracle_ax_scratch(const double *u, const double *g, const double *dx, double *w,
                      int64_t num_elements, int n, int nthreads)
{
    if (n < 2 || n > 16 || num_elements < 0) return 1;
    set_threads(nthreads);
    const int64_t nnn = (int64_t)n * n * n;
    int status = 0;
#pragma omp parallel
    {
        double *sr = (double *)malloc(sizeof(double) * 3 * (size_t)nnn);
        if (!sr) {
#pragma omp atomic write
            status = 2;
        } else {
            double *ss = sr + nnn, *st = sr + 2 * nnn;
#pragma omp for schedule(static)
            for (int64_t e = 0; e < num_elements; ++e) {
                const double *ue = u + e * nnn, *ge = g + e * 6 * nnn;
                for (int k = 0; k < n; ++k)
                    for (int j = 0; j < n; ++j)
                        for (int i = 0; i < n; ++i) {
                            double wr = 0.0, ws = 0.0, wt = 0.0;
                            for (int l = 0; l < n; ++l) {
                                wr += dx[i * n + l] * ue[(k * n + j) * n + l];
                                ws += dx[j * n + l] * ue[(k * n + l) * n + i];
                                wt += dx[k * n + l] * ue[(l * n + j) * n + i];
                            }
                            const int p = (k * n + j) * n + i;
                            const double g1 = ge[p], g2 = ge[nnn + p], g3 = ge[2 * nnn + p];
                            const double g4 = ge[3 * nnn + p], g5 = ge[4 * nnn + p];
                            const double g6 = ge[5 * nnn + p];
                            sr[p] = g1 * wr + g2 * ws + g3 * wt;
                            ss[p] = g2 * wr + g4 * ws + g5 * wt;
                            st[p] = g3 * wr + g5 * ws + g6 * wt;
                        }
                for (int k = 0; k < n; ++k)
                    for (int j = 0; j < n; ++j)
                        for (int i = 0; i < n; ++i) {
                            double acc = 0.0;
                            for (int l = 0; l < n; ++l) {
                                acc += dx[l * n + i] * sr[(k * n + j) * n + l];
                                acc += dx[l * n + j] * ss[(k * n + l) * n + i];
                                acc += dx[l * n + k] * st[(l * n + j) * n + i];
                            }
                            w[e * nnn + (k * n + j) * n + i] = acc;
                        }
            }
            free(sr);
        }
    }
    return status;
}

/* np.bincount(gid, weights=f, minlength=num_global)[gid]: every class sums its
 * members in ascending local index order starting from +0.0. */
int oracle_dssum(const double *f, const int64_t *gid, int64_t count,
                 int64_t num_global, double *out)
{
    double *acc = (double *)calloc((size_t)num_global, sizeof(double));
    if (!acc) return 2;
    for (int64_t p = 0; p < count; ++p) acc[gid[p]] += f[p];
    for (int64_t p = 0; p < count; ++p) out[p] = acc[gid[p]];
    free(acc);
    return 0;
}

void oracle_mask(const double *f, const double *m, double *out, int64_t count)
{
    for (int64_t p = 0; p < count; ++p) out[p] = f[p] * m[p];
}

/* Chunked, in-order weighted dot: each chunk is a sequential left fold of
 * (a*b)*w, chunk partials are then folded in chunk order. */
double oracle_wdot3(const double *a, const double *b, const double *wt,
                    int64_t count, int nthreads)
{
    set_threads(nthreads);
    const int64_t nchunks = (count + WDOT_CHUNK - 1) / WDOT_CHUNK;
    double *part = (double *)malloc(sizeof(double) * (size_t)(nchunks > 0 ? nchunks : 1));
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < nchunks; ++c) {
        const int64_t lo = c * WDOT_CHUNK;
        const int64_t hi = lo + WDOT_CHUNK < count ? lo + WDOT_CHUNK : count;
        double s = 0.0;
        for (int64_t p = lo; p < hi; ++p) s += a[p] * b[p] * wt[p];
        part[c] = s;
    }
    double total = 0.0;
    for (int64_t c = 0; c < nchunks; ++c) total += part[c];
    free(part);
    return total;
}

void oracle_axpy_into(double *x, const double *y, double alpha, int64_t count,
                      int nthreads)
{
    set_threads(nthreads);
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < count; ++p) x[p] += alpha * y[p];
}

void oracle_scale_add(double *p, const double *z, double beta, int64_t count,
                      int nthreads)
{
    set_threads(nthreads);
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < count; ++q) p[q] = beta * p[q] + z[q];
}

/* SplitMix64 counter stream of sembench/fields.py:16-54: value i is
 * 2*((mix(seed+i)) >> 11) * 2^-53 - 1. */
static uint64_t splitmix(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void oracle_random_field(uint64_t seed, int64_t count, double *out)
{
    for (int64_t p = 0; p < count; ++p) {
        const double u01 = (double)(splitmix(seed + (uint64_t)p) >> 11) * (1.0 / 9007199254740992.0);
        out[p] = 2.0 * u01 - 1.0;
    }
}
