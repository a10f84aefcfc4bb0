/*
 * matern_oracle.c -- TEST INFRASTRUCTURE ONLY.  Dense O(N*M) CPU oracle for the
 * exact Matern kernel matrix-vector product of arXiv 2508.01864.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  The product path (libgpmatern.so and
 * paper_2508_01864_b200/) never links, loads or calls it, and shares no code,
 * header, table or constant with it.
 *
 * What it computes is the plain definition, with no decomposition, no sort and
 * no scan (the method is exact, PAPER.md L549 [§2.2.3]):
 *
 *   (K v)_j      = sum_i v_i Ktilde(x_i, x_j)          PAPER.md L241-247 [eq Ky]
 *   (K_zx v)_q   = sum_i v_i Ktilde(x_i, z_q)          PAPER.md L256 [eq kde], L92 [k_z]
 *
 * with the scaled Matern kernel (PAPER.md L1253 [eq scaled_matern]) and the
 * closed-form half-integer profiles (PAPER.md L1273-1275 [eq matern_1_2,
 * matern_3_2, matern_5_2]):
 *
 *   k_{1/2}(r) = exp(-r)
 *   k_{3/2}(r) = (1 + sqrt3 r) exp(-sqrt3 r)
 *   k_{5/2}(r) = (1 + sqrt5 r + 5/3 r^2) exp(-sqrt5 r)
 *
 * (and k_{7/2}, k_{9/2} of L1276-1277) and the two multivariate forms (PAPER.md L414-422 [eq product_kernel,
 * L1_kernel]; §2.3):
 *
 *   L1:      Ktilde(x,x') = s^2 k( sum_k |x_k - x'_k| / l_k )
 *   product: Ktilde(x,x') = s^2 prod_k k( |x_k - x'_k| / l_k )
 *
 * Per-dimension lengthscales l_k are DESIGN.md reading R2 (the paper has one l).
 * Kernel values are evaluated in double (exp in double); sums accumulate in
 * long double (x86-64 80-bit).  Rows are split across OpenMP threads; each row
 * is summed sequentially in source order.
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* k_nu(r) for nu = two_nu/2, r >= 0. Returns NAN for an
 * unsupported nu so a mistake cannot silently produce numbers. */
static double profile(int two_nu, double r)
{
    switch (two_nu) {
    case 1: return exp(-r);
    case 3: { const double s = sqrt(3.0) * r; return (1.0 + s) * exp(-s); }
    case 5: { const double s = sqrt(5.0) * r; return (1.0 + s + (5.0 / 3.0) * r * r) * exp(-s); }
    case 7: {   /* PAPER.md L1276 [eq matern_7_2] */
        const double s = sqrt(7.0) * r;
        return (1.0 + s + (14.0 / 5.0) * r * r + (7.0 * sqrt(7.0) / 15.0) * r * r * r) * exp(-s);
    }
    case 9: {   /* PAPER.md L1277 [eq matern_9_2] */
        const double s = 3.0 * r;
        return (1.0 + 3.0 * r + (27.0 / 7.0) * r * r + (18.0 / 7.0) * r * r * r +
                (27.0 / 35.0) * r * r * r * r) * exp(-s);
    }
    default: return NAN;
    }
}

/* k'_nu(r), the first derivative of the profile (PAPER.md L1320-1324 [eq dmatern12_dl ..
 * dmatern92_dl]). */
static double dprofile(int two_nu, double r)
{
    switch (two_nu) {
    case 1: return -exp(-r);
    case 3: return -(3.0 * r) * exp(-sqrt(3.0) * r);
    case 5: return -((5.0 / 3.0) * r + (5.0 * sqrt(5.0) / 3.0) * r * r) * exp(-sqrt(5.0) * r);
    case 7:   /* PAPER.md L1323 [eq dmatern72_dl] */
        return -((7.0 / 5.0) * r + (7.0 * sqrt(7.0) / 5.0) * r * r + (49.0 / 15.0) * r * r * r) *
               exp(-sqrt(7.0) * r);
    case 9:   /* PAPER.md L1324 [eq dmatern92_dl] */
        return -((9.0 / 7.0) * r + (27.0 / 7.0) * r * r + (162.0 / 35.0) * r * r * r +
                 (81.0 / 35.0) * r * r * r * r) * exp(-3.0 * r);
    default: return NAN;
    }
}

/* Lengthscale derivative of Ktilde(a, b): with every l_k = c l_k0, d Ktilde / d log c at
 * c = 1 (PAPER.md L1314 [eq dkernel_dl] multiplied by l; one l: divide by l for dK/dl):
 *   L1:      -s^2 r k'_nu(r),   r = sum_k |a_k - b_k| / l_k
 *   product: -s^2 sum_k r_k k'_nu(r_k) prod_{j != k} k_nu(r_j),   r_k = |a_k - b_k| / l_k
 * (the product rule; each factor's r_k scales with 1/c). */
double oracle_dkernel_value(int two_nu, int form, int d, const double *ell, double outputscale,
                            const double *a, const double *b)
{
    if (form == 0) {
        double r = 0.0;
        for (int k = 0; k < d; ++k) r += fabs(a[k] - b[k]) / ell[k];
        return -outputscale * outputscale * r * dprofile(two_nu, r);
    }
    double acc = 0.0;
    for (int k = 0; k < d; ++k) {
        const double rk = fabs(a[k] - b[k]) / ell[k];
        double term = -rk * dprofile(two_nu, rk);
        for (int j = 0; j < d; ++j)
            if (j != k) term *= profile(two_nu, fabs(a[j] - b[j]) / ell[j]);
        acc += term;
    }
    return outputscale * outputscale * acc;
}

/* Ktilde(a, b) for one pair of d-dimensional points (form 0 = L1, 1 = product). */
double oracle_kernel_value(int two_nu, int form, int d, const double *ell, double outputscale,
                           const double *a, const double *b)
{
    double val;
    if (form == 0) {
        double r = 0.0;
        for (int k = 0; k < d; ++k) r += fabs(a[k] - b[k]) / ell[k];
        val = profile(two_nu, r);
    } else {
        val = 1.0;
        for (int k = 0; k < d; ++k) val *= profile(two_nu, fabs(a[k] - b[k]) / ell[k]);
    }
    return outputscale * outputscale * val;
}

/*
 * out[k] = sum_{i<n} v[i] * Ktilde(src_i, tgt_{rows[k]}),  k < nrows
 * absrow[k] (optional) = sum_i |Ktilde(src_i, tgt_{rows[k]})|   (row of ||K||_inf)
 * rows == NULL means rows[k] = k, nrows targets.
 * src: n x d row-major, tgt: (any) x d row-major.  nthreads <= 0: OpenMP default.
 */
static void cross_rows(int kind, int two_nu, int form, int d, const double *ell,
                       double outputscale, const double *src, const double *v, int64_t n,
                       const double *tgt, const int64_t *rows, int64_t nrows,
                       double *out, double *absrow, int nthreads)
{
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t k = 0; k < nrows; ++k) {
        const int64_t j = rows ? rows[k] : k;
        const double *z = tgt + (size_t)j * d;
        long double acc = 0.0L, aacc = 0.0L;
        for (int64_t i = 0; i < n; ++i) {
            const double kv = kind == 0
                ? oracle_kernel_value(two_nu, form, d, ell, outputscale, src + (size_t)i * d, z)
                : oracle_dkernel_value(two_nu, form, d, ell, outputscale, src + (size_t)i * d, z);
            acc += (long double)v[i] * (long double)kv;
            aacc += (long double)fabs(kv);
        }
        out[k] = (double)acc;
        if (absrow) absrow[k] = (double)aacc;
    }
}

void oracle_cross_mvm(int two_nu, int form, int d, const double *ell, double outputscale,
                      const double *src, const double *v, int64_t n,
                      const double *tgt, const int64_t *rows, int64_t nrows,
                      double *out, double *absrow, int nthreads)
{
    cross_rows(0, two_nu, form, d, ell, outputscale, src, v, n, tgt, rows, nrows, out, absrow,
               nthreads);
}

/* As oracle_cross_mvm with the lengthscale derivative l dKtilde/dl (L1 form). */
void oracle_cross_dmvm(int two_nu, int form, int d, const double *ell, double outputscale,
                       const double *src, const double *v, int64_t n,
                       const double *tgt, const int64_t *rows, int64_t nrows,
                       double *out, double *absrow, int nthreads)
{
    cross_rows(1, two_nu, form, d, ell, outputscale, src, v, n, tgt, rows, nrows, out, absrow,
               nthreads);
}

/* Dense block Kout[i*n + j] = Ktilde(a_i, b_j), a: m x d, b: n x d (small sizes only). */
void oracle_dense(int two_nu, int form, int d, const double *ell, double outputscale,
                  const double *a, int64_t m, const double *b, int64_t n, double *Kout,
                  int nthreads)
{
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j)
            Kout[(size_t)i * n + j] = oracle_kernel_value(two_nu, form, d, ell, outputscale,
                                                          a + (size_t)i * d, b + (size_t)j * d);
}

/* Dense block of the lengthscale derivative, Kout[i*n + j] = l dKtilde(a_i, b_j)/dl (L1). */
void oracle_dense_d(int two_nu, int form, int d, const double *ell, double outputscale,
                    const double *a, int64_t m, const double *b, int64_t n, double *Kout,
                    int nthreads)
{
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j)
            Kout[(size_t)i * n + j] = oracle_dkernel_value(two_nu, form, d, ell, outputscale,
                                                           a + (size_t)i * d, b + (size_t)j * d);
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
