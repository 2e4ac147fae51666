/* Type-generic body of the C oracle — TEST INFRASTRUCTURE ONLY.
 *
 * Included twice by spaimg_oracle.c with REAL = double / float and SFX = _f64 / _f32.
 * Every per-point expression follows SURVEY.md Appendix A, i.e. the reference
 * numpy expression trees (reference pkg/src/spaimg/stencils.py:136-153,
 * multigrid.py:86-185), one IEEE rounding per operation, no contraction
 * (built with -ffp-contract=off).
 */

#define CAT_(a, b) a##b
#define CAT(a, b) CAT_(a, b)
#define FN(name) CAT(name, SFX)

/* Zero-extended stencil product at one interior point (stencils.py:147-152):
 * acc = 0; acc += c_k * u[i+o_k] in entry order; out = acc * scale. */
static inline REAL FN(point_apply)(int dim, long n, const REAL *u, long i0, long i1, long i2,
                                   int nterms, const int *offs, const REAL *coef, REAL scale) {
    REAL acc = (REAL)0;
    for (int k = 0; k < nterms; ++k) {
        long j0 = i0 + offs[k * dim + 0];
        long j1 = i1 + offs[k * dim + 1];
        long j2 = dim == 3 ? i2 + offs[k * dim + 2] : 0;
        REAL v = (REAL)0;
        if (j0 >= 0 && j0 < n && j1 >= 0 && j1 < n && (dim == 2 || (j2 >= 0 && j2 < n)))
            v = dim == 2 ? u[j0 * n + j1] : u[(j0 * n + j1) * n + j2];
        REAL p = coef[k] * v;
        acc = acc + p;
    }
    return acc * scale;
}

void FN(oracle_apply)(int dim, int N, const REAL *x, REAL *out, int nterms, const int *offs,
                      const REAL *coef, REAL scale) {
    long n = N - 1;
    long n2 = dim == 3 ? n : 1;
#pragma omp parallel for schedule(static)
    for (long i0 = 0; i0 < n; ++i0)
        for (long i1 = 0; i1 < n; ++i1)
            for (long i2 = 0; i2 < n2; ++i2) {
                long idx = dim == 2 ? i0 * n + i1 : (i0 * n + i1) * n + i2;
                out[idx] = FN(point_apply)(dim, n, x, i0, i1, i2, nterms, offs, coef, scale);
            }
}

#ifndef SPAIMG_ORACLE_LAP_OFFS
#define SPAIMG_ORACLE_LAP_OFFS
static const int LAP2_OFFS[5 * 2] = {0, 0, 1, 0, -1, 0, 0, 1, 0, -1};
static const int LAP3_OFFS[7 * 3] = {0, 0, 0, 1, 0, 0, -1, 0, 0, 0, 1, 0, 0, -1, 0, 0, 0, 1, 0, 0, -1};
#endif

/* r = b - A x (multigrid.py:99): A = laplacian(dim) (stencils.py:209-223). */
void FN(oracle_residual)(int dim, int N, const REAL *x, const REAL *b, REAL *r, REAL sA) {
    long n = N - 1;
    long n2 = dim == 3 ? n : 1;
    REAL lc[7];
    int nt = dim == 2 ? 5 : 7;
    lc[0] = (REAL)(dim == 2 ? 4 : 6);
    for (int k = 1; k < nt; ++k) lc[k] = (REAL)-1;
    const int *lo = dim == 2 ? LAP2_OFFS : LAP3_OFFS;
#pragma omp parallel for schedule(static)
    for (long i0 = 0; i0 < n; ++i0)
        for (long i1 = 0; i1 < n; ++i1)
            for (long i2 = 0; i2 < n2; ++i2) {
                long idx = dim == 2 ? i0 * n + i1 : (i0 * n + i1) * n + i2;
                REAL ax = FN(point_apply)(dim, n, x, i0, i1, i2, nt, lo, lc, sA);
                r[idx] = b[idx] - ax;
            }
}

/* v <- v + omega * (M r) (multigrid.py:100): scale applied inside M, then omega. */
static void FN(update)(int dim, int N, const REAL *x, const REAL *r, REAL *out, int nterms,
                       const int *offs, const REAL *coef, REAL sM, REAL omega) {
    long n = N - 1;
    long n2 = dim == 3 ? n : 1;
#pragma omp parallel for schedule(static)
    for (long i0 = 0; i0 < n; ++i0)
        for (long i1 = 0; i1 < n; ++i1)
            for (long i2 = 0; i2 < n2; ++i2) {
                long idx = dim == 2 ? i0 * n + i1 : (i0 * n + i1) * n + i2;
                REAL mr = FN(point_apply)(dim, n, r, i0, i1, i2, nterms, offs, coef, sM);
                REAL t = omega * mr;
                out[idx] = x[idx] + t;
            }
}

static long FN(count)(int dim, int N) {
    long n = N - 1;
    return dim == 2 ? n * n : n * n * n;
}

/* smooth (multigrid.py:86-101); x and out may alias. */
int FN(oracle_smooth)(int dim, int N, const REAL *x, const REAL *b, REAL *out, int nterms,
                      const int *offs, const REAL *coef, REAL sA, REAL sM, REAL omega, int steps) {
    long cnt = FN(count)(dim, N);
    if (out != x) memcpy(out, x, (size_t)cnt * sizeof(REAL));
    if (steps <= 0) return 0;
    REAL *r = (REAL *)malloc((size_t)cnt * sizeof(REAL));
    REAL *t = (REAL *)malloc((size_t)cnt * sizeof(REAL));
    if (!r || !t) { free(r); free(t); return -1; }
    for (int s = 0; s < steps; ++s) {
        FN(oracle_residual)(dim, N, out, b, r, sA);
        FN(update)(dim, N, out, r, t, nterms, offs, coef, sM, omega);
        memcpy(out, t, (size_t)cnt * sizeof(REAL));
    }
    free(r);
    free(t);
    return 0;
}

/* full weighting of one fine line triple (multigrid.py:106): (0.25 a + 0.5 b) + 0.25 c */
static inline REAL FN(fw)(REAL a, REAL b, REAL c) {
    REAL p = (REAL)0.25 * a;
    REAL q = (REAL)0.5 * b;
    REAL s = p + q;
    REAL w = (REAL)0.25 * c;
    return s + w;
}

/* restrict (multigrid.py:104-119): separable, axis 0 first; r is a dense fine array. */
void FN(oracle_restrict)(int dim, int N, const REAL *r, REAL *out) {
    long nf = N - 1, nc = N / 2 - 1;
    if (dim == 2) {
        REAL *t = (REAL *)malloc((size_t)(nc * nf) * sizeof(REAL));
#pragma omp parallel for schedule(static)
        for (long I = 0; I < nc; ++I)
            for (long j = 0; j < nf; ++j)
                t[I * nf + j] = FN(fw)(r[(2 * I) * nf + j], r[(2 * I + 1) * nf + j], r[(2 * I + 2) * nf + j]);
#pragma omp parallel for schedule(static)
        for (long I = 0; I < nc; ++I)
            for (long J = 0; J < nc; ++J)
                out[I * nc + J] = FN(fw)(t[I * nf + 2 * J], t[I * nf + 2 * J + 1], t[I * nf + 2 * J + 2]);
        free(t);
    } else {
        REAL *t = (REAL *)malloc((size_t)(nc * nf * nf) * sizeof(REAL));
        REAL *u = (REAL *)malloc((size_t)(nc * nc * nf) * sizeof(REAL));
#pragma omp parallel for schedule(static)
        for (long I = 0; I < nc; ++I)
            for (long j = 0; j < nf; ++j)
                for (long k = 0; k < nf; ++k)
                    t[(I * nf + j) * nf + k] = FN(fw)(r[((2 * I) * nf + j) * nf + k],
                                                      r[((2 * I + 1) * nf + j) * nf + k],
                                                      r[((2 * I + 2) * nf + j) * nf + k]);
#pragma omp parallel for schedule(static)
        for (long I = 0; I < nc; ++I)
            for (long J = 0; J < nc; ++J)
                for (long k = 0; k < nf; ++k)
                    u[(I * nc + J) * nf + k] = FN(fw)(t[(I * nf + 2 * J) * nf + k],
                                                      t[(I * nf + 2 * J + 1) * nf + k],
                                                      t[(I * nf + 2 * J + 2) * nf + k]);
#pragma omp parallel for schedule(static)
        for (long I = 0; I < nc; ++I)
            for (long J = 0; J < nc; ++J)
                for (long K = 0; K < nc; ++K)
                    out[(I * nc + J) * nc + K] = FN(fw)(u[(I * nc + J) * nf + 2 * K],
                                                        u[(I * nc + J) * nf + 2 * K + 1],
                                                        u[(I * nc + J) * nf + 2 * K + 2]);
        free(t);
        free(u);
    }
}

/* restrict(b - A x) (multigrid.py:176-177) */
int FN(oracle_residual_restrict)(int dim, int N, const REAL *x, const REAL *b, REAL *out, REAL sA) {
    long cnt = FN(count)(dim, N);
    REAL *r = (REAL *)malloc((size_t)cnt * sizeof(REAL));
    if (!r) return -1;
    FN(oracle_residual)(dim, N, x, b, r, sA);
    FN(oracle_restrict)(dim, N, r, out);
    free(r);
    return 0;
}

/* One prolongation line value (multigrid.py:126-129): fine index i of a coarse line a[0..m). */
static inline REAL FN(pl)(const REAL *a, long stride, long m, long i) {
    if (i & 1) return a[(i >> 1) * stride];
    long j = i >> 1; /* even fine index 2j, 0 <= j <= m */
    if (j == 0) return (REAL)0.5 * a[0];
    if (j == m) return (REAL)0.5 * a[(m - 1) * stride];
    REAL s = a[(j - 1) * stride] + a[j * stride];
    return (REAL)0.5 * s;
}

/* x <- x + prolong(e) (multigrid.py:122-144, :184); Nc = coarse mesh count. */
int FN(oracle_prolong_correct)(int dim, int Nc, REAL *x, const REAL *e) {
    long m = Nc - 1, nf = 2 * Nc - 1;
    if (dim == 2) {
        REAL *t = (REAL *)malloc((size_t)(nf * m) * sizeof(REAL));
        if (!t) return -1;
#pragma omp parallel for schedule(static)
        for (long i = 0; i < nf; ++i)
            for (long J = 0; J < m; ++J) t[i * m + J] = FN(pl)(e + J, m, m, i);
#pragma omp parallel for schedule(static)
        for (long i = 0; i < nf; ++i)
            for (long j = 0; j < nf; ++j) {
                REAL p = FN(pl)(t + i * m, 1, m, j);
                x[i * nf + j] = x[i * nf + j] + p;
            }
        free(t);
    } else {
        REAL *t = (REAL *)malloc((size_t)(nf * m * m) * sizeof(REAL));
        REAL *u = (REAL *)malloc((size_t)(nf * nf * m) * sizeof(REAL));
        if (!t || !u) { free(t); free(u); return -1; }
#pragma omp parallel for schedule(static)
        for (long i = 0; i < nf; ++i)
            for (long J = 0; J < m; ++J)
                for (long K = 0; K < m; ++K) t[(i * m + J) * m + K] = FN(pl)(e + J * m + K, m * m, m, i);
#pragma omp parallel for schedule(static)
        for (long i = 0; i < nf; ++i)
            for (long j = 0; j < nf; ++j)
                for (long K = 0; K < m; ++K) u[(i * nf + j) * m + K] = FN(pl)(t + i * m * m + K, m, m, j);
#pragma omp parallel for schedule(static)
        for (long i = 0; i < nf; ++i)
            for (long j = 0; j < nf; ++j)
                for (long k = 0; k < nf; ++k) {
                    REAL p = FN(pl)(u + (i * nf + j) * m, 1, m, k);
                    x[(i * nf + j) * nf + k] = x[(i * nf + j) * nf + k] + p;
                }
        free(t);
        free(u);
    }
    return 0;
}

/* Coarse direct solve (multigrid.py:147-154): LAPACK getrs order as OpenBLAS runs it for a
 * single right-hand side: row interchanges, column-oriented unit-lower
 * forward substitution with fused multiply-add, then column-oriented upper back substitution with
 * a true division by the pivot.  lu is the n x n row-major factor from scipy lu_factor, piv its
 * 0-based interchange vector. */
void FN(oracle_lu_solve)(int n, const REAL *lu, const int *piv, const REAL *b, REAL *x) {
    if (x != b) memcpy(x, b, (size_t)n * sizeof(REAL));
    for (int i = 0; i < n; ++i) {
        int p = piv[i];
        if (p != i) { REAL t = x[i]; x[i] = x[p]; x[p] = t; }
    }
    for (int j = 0; j < n; ++j) {
        REAL yj = x[j];
        for (int i = j + 1; i < n; ++i) x[i] = FMA(-lu[i * n + j], yj, x[i]);
    }
    for (int j = n - 1; j >= 0; --j) {
        x[j] = x[j] / lu[j * n + j];
        REAL yj = x[j];
        for (int i = 0; i < j; ++i) x[i] = FMA(-lu[i * n + j], yj, x[i]);
    }
}

/* ---------------------------------------------------------------------------------------------
 * whole cycle (multigrid.py:157-185) and the solve loop (multigrid.py:206-219)
 * ------------------------------------------------------------------------------------------- */

typedef struct {
    int dim, nterms, nu1, nu2, gamma, coarsest_N;
    const int *offs;
    const REAL *coef;
    REAL omega;
    int lu_n;
    const REAL *lu;
    const int *piv;
} FN(oracle_cfg);

static REAL FN(sc)(int N, int e) { return (REAL)pow(1.0 / (double)N, (double)e); }

static int FN(cycle_rec)(const FN(oracle_cfg) * c, int N, REAL *u, const REAL *b) {
    int dim = c->dim;
    if (N <= c->coarsest_N) {
        FN(oracle_lu_solve)(c->lu_n, c->lu, c->piv, b, u);
        return 0;
    }
    int rc_ = FN(oracle_smooth)(dim, N, u, b, u, c->nterms, c->offs, c->coef, FN(sc)(N, -2), FN(sc)(N, 2),
                                c->omega, c->nu1);
    if (rc_) return rc_;
    int Nc = N / 2;
    long cc = FN(count)(dim, Nc);
    REAL *rc = (REAL *)malloc((size_t)cc * sizeof(REAL));
    REAL *ec = (REAL *)calloc((size_t)cc, sizeof(REAL));
    if (!rc || !ec) { free(rc); free(ec); return -1; }
    FN(oracle_residual_restrict)(dim, N, u, b, rc, FN(sc)(N, -2));
    if (Nc <= c->coarsest_N) {
        FN(oracle_lu_solve)(c->lu_n, c->lu, c->piv, rc, ec);
    } else {
        for (int g = 0; g < c->gamma; ++g) {
            rc_ = FN(cycle_rec)(c, Nc, ec, rc);
            if (rc_) { free(rc); free(ec); return rc_; }
        }
    }
    FN(oracle_prolong_correct)(dim, Nc, u, ec);
    free(rc);
    free(ec);
    return FN(oracle_smooth)(dim, N, u, b, u, c->nterms, c->offs, c->coef, FN(sc)(N, -2), FN(sc)(N, 2),
                             c->omega, c->nu2);
}

/* In-place cycle on u.  lu/piv describe the coarsest-level factorisation (lu_n unknowns). */
int FN(oracle_cycle)(int dim, int N, REAL *u, const REAL *b, int nterms, const int *offs, const REAL *coef,
                     REAL omega, int nu1, int nu2, int gamma, int coarsest_N, int lu_n, const REAL *lu,
                     const int *piv) {
    FN(oracle_cfg) c = {dim, nterms, nu1, nu2, gamma, coarsest_N, offs, coef, omega, lu_n, lu, piv};
    return FN(cycle_rec)(&c, N, u, b);
}

/* ||b - A x||_2 accumulated in double, fixed per-row order then sequential over rows. */
double FN(oracle_residual_norm)(int dim, int N, const REAL *x, const REAL *b) {
    long n = N - 1;
    long rows = dim == 2 ? n : n * n;
    long cnt = FN(count)(dim, N);
    REAL *r = (REAL *)malloc((size_t)cnt * sizeof(REAL));
    double *part = (double *)malloc((size_t)rows * sizeof(double));
    FN(oracle_residual)(dim, N, x, b, r, FN(sc)(N, -2));
#pragma omp parallel for schedule(static)
    for (long q = 0; q < rows; ++q) {
        double s = 0.0;
        for (long k = 0; k < n; ++k) {
            double v = (double)r[q * n + k];
            s += v * v;
        }
        part[q] = s;
    }
    double s = 0.0;
    for (long q = 0; q < rows; ++q) s += part[q];
    free(r);
    free(part);
    return sqrt(s);
}

/* solve loop from the start held in u (multigrid.py:206-219); norms has room for max_iters+1. */
int FN(oracle_solve)(int dim, int N, REAL *u, const REAL *b, int nterms, const int *offs, const REAL *coef,
                     REAL omega, int nu1, int nu2, int gamma, int coarsest_N, int lu_n, const REAL *lu,
                     const int *piv, double tol, int max_iters, double *norms, int *iterations, int *converged) {
    norms[0] = FN(oracle_residual_norm)(dim, N, u, b);
    int k = 0;
    *converged = 0;
    while (k < max_iters) {
        int rc = FN(oracle_cycle)(dim, N, u, b, nterms, offs, coef, omega, nu1, nu2, gamma, coarsest_N, lu_n,
                                  lu, piv);
        if (rc) return rc;
        ++k;
        norms[k] = FN(oracle_residual_norm)(dim, N, u, b);
        if (norms[k] <= tol * norms[0]) { *converged = 1; break; }
    }
    *iterations = k;
    return 0;
}

#undef FN
#undef CAT
#undef CAT_
