/*
 * gpmatern.h -- C ABI of the B200-native exact fast Matern kernel MVM
 * (arXiv 2508.01864, "weighted empirical CDF" decomposition) and the GP
 * posterior-mean pipeline built on it.
 *
 * Citations: "P:n" = line n of the paper text, with the section /
 * equation it falls in.  Readings of ambiguous passages are numbered R1..Rn in
 * DESIGN.md.
 *
 * Conventions for every entry point
 *   - Array pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors) unless
 *     the parameter says "(host)".  All doubles are IEEE float64.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Work is enqueued on it; calls that return host values synchronise it.
 *   - Ownership: the caller owns every pointer it passes and may free it after the
 *     call returns (gp_setup copies what it needs).  A plan owns its device memory
 *     until gp_destroy.  A plan is not safe for concurrent use from two streams.
 *   - Errors: a gp_status is returned, never an exception; gp_last_error() gives a
 *     thread-local message for the last non-OK status.  There is no CPU fallback:
 *     without a CUDA device every compute call returns GP_ERR_CUDA.
 */
#ifndef GPMATERN_H
#define GPMATERN_H
#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define GP_API __attribute__((visibility("default")))
#else
#define GP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GP_OK = 0,
    GP_ERR_INVALID_ARG = 1,   /* null pointer, n < 1, d not in {1,2,3}, outputscale/lengthscale/sigma2/rtol <= 0 */
    GP_ERR_UNSUPPORTED = 2,   /* (nu, form, d) outside the supported set (message lists it) */
    GP_ERR_NONFINITE = 3,     /* NaN/Inf coordinate; message names the first bad row */
    GP_ERR_RANGE = 4,         /* reserved: the literal exp(+t) weights of P:600 are never formed (R5) */
    GP_ERR_NOT_CONVERGED = 5, /* CG hit max_iter; last iterate left in alpha, info filled */
    GP_ERR_BREAKDOWN = 6,     /* CG found p^T A p <= 0 (A not SPD, e.g. L1 nu>=3/2, d>=2, R4) */
    GP_ERR_CUDA = 7,          /* CUDA runtime error (message has cudaGetErrorString) */
    GP_ERR_OOM = 8            /* device allocation failed */
} gp_status;

enum { GP_FORM_L1 = 0, GP_FORM_PRODUCT = 1 };                 /* P:414-422 [eq product_kernel, L1_kernel] */
enum { GP_MEAN_NONE = 0, GP_MEAN_AFFINE = 1, GP_MEAN_BASIS = 2 }; /* P:73-82 [eq BetaLin, BetaFunc] */

/* Scaled Matern kernel, P:294 [eq scaled_kernel], P:1253 [eq scaled_matern]:
 *   L1:      K(x,x') = s^2 k_nu( sum_k |x_k - x'_k| / l_k )        (§2.3)
 *   product: K(x,x') = s^2 prod_k k_nu( |x_k - x'_k| / l_k )
 * with k_nu the half-integer closed forms of P:1273-1275.  Supported:
 *   two_nu in {1,3,5,7,9} (nu = 7/2, 9/2: P:1276-1277); d in {1,2,3}; forms L1 and
 *   PRODUCT for every d and nu (PRODUCT, d = 2: (p+1)^2 mixed moments per channel; d = 3:
 *   (p+1)^2 re-weighted passes of the (p+1)-moment scan per level, P:487-509 [Prop 2] with both
 *   split factors separated -- exact, about (p+1)^2 times the cost of the L1 apply)
 *   (for d == 1 or two_nu == 1 the two forms coincide, and form is ignored).
 * Per-dimension lengthscales are reading R2 (the paper uses one l). */
typedef struct {
    int two_nu;            /* 1, 3, 5, 7, 9 (nu = two_nu / 2) */
    int form;              /* GP_FORM_* */
    double outputscale;    /* s > 0, K(x,x) = s^2 */
    double lengthscale[3]; /* l_k > 0 for k < d */
} gp_kernel;

typedef struct {
    int iters;             /* CG iterations performed (max over right-hand sides) */
    double relres_max;     /* max over columns of the TRUE ||b - A x|| / ||b|| at exit */
    int failed_column;     /* column that broke down / did not converge, else -1 */
    int restarts;          /* residual-replacement restarts taken */
} gp_cg_info;

/* Device-memory hook: alloc(bytes, stream, ctx) returns a device pointer (or NULL), free(ptr,
 * stream, ctx) releases it (stream is always NULL: the library synchronises the device
 * before a release). */
typedef void *(*gp_alloc_fn)(size_t bytes, void *stream, void *ctx);
typedef void (*gp_free_fn)(void *ptr, void *stream, void *ctx);

typedef struct gp_plan_s *gp_plan;    /* opaque: the stored sort / D&C structure of x */
typedef struct gp_cross_s *gp_cross;  /* opaque: structure of the union x U z for K_zx */
typedef struct gp_precond_s *gp_precond;  /* opaque: pivoted-Cholesky preconditioner */

/* Result of gp_lml (log-marginal likelihood estimate and its gradient). */
typedef struct {
  double lml;             /* -1/2 quad - 1/2 logdet - N/2 log(2 pi) */
  double quad;            /* r^T A^-1 r */
  double logdet;          /* estimate of log det A (+ log det P when preconditioned) */
  double logdet_precond;  /* log det P, 0 without preconditioner */
  double grad[3];         /* dL/d outputscale, dL/d log(c) (all lengthscales scaled by c;
                             = l dL/dl for one l; every kernel has gp_kmvm_dlengthscale),
                             dL/d sigma */
  int cg_iters;           /* iterations of the A^-1 r solve */
  int lanczos_iters;      /* Lanczos steps per probe (max over probes) */
} gp_lml_result;

/* gp_setup -- build the stored structure of P:191 [§1], P:338 [§2.1], P:539 [§2.2.3]:
 * scale coordinates t_k = sqrt(2 nu) x_k / l_k, radix-sort each dimension, and for
 * d >= 2 the divide-and-conquer level orders (Bentley).
 *   x   : n x d row-major (device).  n >= 1.
 *   k   : kernel (host).
 *   out : receives the plan (host).
 * Errors: INVALID_ARG, UNSUPPORTED, NONFINITE (first bad row), OOM, CUDA.
 * Synchronises `stream` once (finiteness check). */
/* gp_set_allocator -- route every device allocation of the library (plan structure,
 * scratch, solver buffers) through alloc/free, e.g. the PyTorch caching allocator
 * (SURVEY §8(b)).  Process-wide; buffers keep the hook they were allocated with.  Both NULL:
 * back to cudaMalloc / cudaFree (the default).  Errors: INVALID_ARG if only one is NULL. */
GP_API gp_status gp_set_allocator(gp_alloc_fn alloc, gp_free_fn free, void *ctx);

GP_API gp_status gp_setup(const double *x, int64_t n, int d, const gp_kernel *k, void *stream,
                   gp_plan *out);

/* gp_kmvm -- out = K v (no nugget; the diagonal s^2 is included), P:241-247 [eq Ky],
 * computed exactly by the ECDF decomposition, P:314-325 [eq fast_exact_decomposition_1d],
 * P:459-509 [Props 1-2].
 *   v   : n x nrhs, column-major with leading dimension n (device).
 *   out : n x nrhs, same layout (device); must not alias v.
 * Asynchronous on `stream`; no host synchronisation. */
GP_API gp_status gp_kmvm(gp_plan p, const double *v, int nrhs, double *out, void *stream);

/* gp_kmvm_host -- gp_kmvm with HOST buffers (pinned or pageable): copies v to the
 * device, applies, copies out back and synchronises `stream`.  Used for the
 * end-to-end measurement.  v, out: n x nrhs column-major (host).  With nrhs > 1 and both
 * buffers pinned the columns are pipelined through three device slots: the host->device
 * copy of column c+1, the apply of column c (on `stream`) and the device->host copy of
 * column c-1 overlap (two internal copy streams). */
GP_API gp_status gp_kmvm_host(gp_plan p, const double *v, int nrhs, double *out, void *stream);

/* gp_kmvm_rank -- out = K v with v and out in the plan's STORED order (x1-rank order:
 * element r belongs to the point of rank r).  This is the operator used inside CG
 * (P:155-174 [§1]): with the data presorted, an MVM needs no permutation at all
 * (P:336-338 [§2.1] "when the data comes pre-sorted ... O(N)").  Layout as gp_kmvm. */
GP_API gp_status gp_kmvm_rank(gp_plan p, const double *v_rank, int nrhs, double *out_rank,
                              void *stream);

/* gp_kmvm_dlengthscale -- out = (l dK/dl) v, the lengthscale-gradient MVM of the plan's
 * kernel (PAPER.md L1301-1327 [§ Derivative of Matern covariance functions],
 * eq dkernel_dl): with every lengthscale l_k scaled by a common factor c,
 *   out_j = d/dc [sum_i Ktilde_c(x_i, x_j) v_i] at c = 1
 *         = s^2 sum_i g(r_ij) v_i,   g(r) = -r k_nu'(r),  r = sum_k |x_ik - x_jk| / l_k.
 * For one lengthscale l, dK/dl v = out / l; the outputscale gradient is dK/ds v = (2/s) K v
 * (eq dkernel_dvarsigma) and needs no extra MVM.  Computed by the same decomposition with
 * one more moment (g(s) = (s, s^2, (s^2 + s^3)/3) e^{-s} for nu = 1/2, 3/2, 5/2 in scaled
 * distance s = sqrt(2 nu) r): exact like gp_kmvm, no nugget, zero diagonal.
 * Supported: every kernel gp_setup accepts -- d = 1 (any n), the L1 form for d = 2, 3, and the
 * product form for d = 2 and d = 3 at every nu (product rule sum_k g(r_k) prod_{j != k} k(r_j):
 * d = 2, nu <= 7/2 with (p+2)^2 mixed moments per channel; d = 2 at nu = 9/2 and d = 3 by the
 * separated sub-passes of the scan in two runs, about (p+2)^2 times the L1 apply at d = 3).
 * v_order: 0 = user order (layout as
 * gp_kmvm), 1 = the plan's stored order (as gp_kmvm_rank). */
GP_API gp_status gp_kmvm_dlengthscale(gp_plan p, const double *v, int nrhs, double *out,
                                      int v_order, void *stream);

/* gp_permute -- move n x nrhs column-major vectors between user order and the plan's
 * stored order: to_rank != 0: dst[r] = src[perm[r]]; to_rank == 0: dst[perm[r]] = src[r].
 * src and dst must not alias. */
GP_API gp_status gp_permute(gp_plan p, const double *src, int nrhs, double *dst, int to_rank,
                            void *stream);

/* gp_kzx_setup -- structure for the rectangular product K_zx v (P:92 [k_z],
 * P:256 [eq kde]): the same machinery on the union x U z with data points as
 * sources and queries as targets (reading R7).  z: m x d row-major (device), m >= 1. */
GP_API gp_status gp_kzx_setup(gp_plan p, const double *z, int64_t m, void *stream, gp_cross *out);

/* gp_kzx -- out = K_zx v: out_q = sum_i v_i K(x_i, z_q).
 *   v   : n x nrhs column-major (device), out: m x nrhs column-major (device). */
GP_API gp_status gp_kzx(gp_cross c, const double *v, int nrhs, double *out, void *stream);
GP_API void gp_kzx_destroy(gp_cross c);

/* gp_kmvm_partial -- one shard's share of a d >= 2 apply (the multi-GPU
 * decomposition of the D&C).  Shard `shard` of `nshards` computes the pairs of
 * its tiles of the within-tile level kernels and its items of the carried-pass apply (the
 * carried-pass aggregates run whole on every shard); every pair belongs to exactly one
 * shard, so sum over shards of out_rank = K v_rank (the self term is added by shard 0).
 *   v_rank  : n x nrhs column-major, rank order (device; every shard needs all of v:
 *             gather it first, e.g. ncclAllGather);
 *   out_rank: n x nrhs column-major, rank order (device): this shard's partial product
 *             (sum the shards with e.g. ncclAllReduce / ncclReduceScatter, then gp_permute).
 * Errors: INVALID_ARG (bad shard / nshards), UNSUPPORTED for d = 1 (one launch with a
 * chunk exchange: shard d = 1 by right-hand sides). */
GP_API gp_status gp_kmvm_partial(gp_plan p, const double *v_rank, int nrhs, double *out_rank,
                                 int shard, int nshards, void *stream);

/* gp_shard_ranges -- host only (no device needed): the work split of gp_kmvm_partial for a
 * plan of n points in dimension d: ranges[0..1] = tiles [lo, hi) of the tile kernels,
 * ranges[2..3] = items [lo, hi) of the carried-pass apply.  INVALID_ARG for d = 1. */
GP_API gp_status gp_shard_ranges(int64_t n, int d, int shard, int nshards, int64_t *ranges);

/* gp_cg_solve -- conjugate gradients (P:155-174 [§1]; P:980-1034 [App A, Alg 2] with
 * no preconditioner, zero initial guess) on A = K + sigma2 I for the right-hand sides
 * [y, H] (multi-RHS), then the GLS fixed effects of P:808-812:
 *   beta = (H^T A^-1 H)^-1 H^T A^-1 y,   alpha = A^-1 y - (A^-1 H) beta,
 * so that the posterior mean is mu(z) = h(z)^T beta + K_zx alpha (P:86 [eq gp_mean]).
 *   sigma2    : nugget sigma^2 > 0.
 *   y         : n (device), user order.
 *   mean_kind : GP_MEAN_NONE (beta empty, alpha = A^-1 y), GP_MEAN_AFFINE (H = [1, x]
 *               from the raw coordinates, P:73 [eq BetaLin]), GP_MEAN_BASIS
 *               (H = user basis, n x L column-major device, P:79 [eq BetaFunc]).
 *   rtol      : per-column relative residual target ||b - A x||_2 / ||b||_2 (R8).
 *   max_iter  : iteration cap.
 *   alpha     : n (device) output.
 *   beta      : (host) output of length 1+d (AFFINE) or L (BASIS); may be NULL.
 *   info      : (host) may be NULL.
 * Errors: BREAKDOWN (p^T A p <= 0: column + iteration in the message),
 * NOT_CONVERGED (alpha holds the last iterate).  Synchronises `stream`. */
GP_API gp_status gp_cg_solve(gp_plan p, double sigma2, const double *y, int mean_kind,
                      const double *H, int L, double rtol, int max_iter, double *alpha,
                      double *beta, gp_cg_info *info, void *stream);

/* gp_cg_solve_pc -- gp_cg_solve preconditioned by pc (P = L L^T + sigma2 I,
 * applied by the Woodbury formula; pc = NULL is gp_cg_solve).  Same arguments, semantics
 * and stopping rule (true residual, restarts from it when the recursion drifted). */
GP_API gp_status gp_cg_solve_pc(gp_plan p, gp_precond pc, double sigma2, const double *y,
                                int mean_kind, const double *H, int L, double rtol,
                                int max_iter, double *alpha, double *beta, gp_cg_info *info,
                                void *stream);

/* gp_cg_solve_ex -- gp_cg_solve_pc with the solve's by-products (SURVEY §8(a) a10, §8(c) c1
 * item 4):
 *   beta_ols : (host) NULL or 1+d (AFFINE) / L (BASIS) entries: the OLS estimate
 *              (H^T H)^-1 H^T y that Algorithm 1 starts from (P:829 [Alg 1, first line]);
 *   X        : (device) NULL or n x (1 + nh) column-major, user order: the CG solutions
 *              [A^-1 y, A^-1 H_1, ..., A^-1 H_nh] (nh = 0, 1+d or L), from which beta and
 *              alpha are formed.
 * Unpreconditioned iterations run the fused iteration: the apply returns
 * q = K p + sigma2 p with the p^T q partials, two vector kernels re-sum the partials in a
 * fixed order, and blocks of 8 iterations are replayed as one CUDA graph (run directly
 * when `stream` is itself being captured).  Other arguments and errors as gp_cg_solve. */
GP_API gp_status gp_cg_solve_ex(gp_plan p, gp_precond pc, double sigma2, const double *y,
                                int mean_kind, const double *H, int L, double rtol,
                                int max_iter, double *alpha, double *beta, double *beta_ols,
                                double *X, gp_cg_info *info, void *stream);

/* ---- the likelihood machinery of PAPER.md App A ---------------------- */

/* gp_precond_create -- rank-k pivoted Cholesky K ~ L L^T of the plan's kernel matrix
 * (Harbrecht et al.): k greedy steps, pivot = largest remaining diagonal (ties:
 * smallest x1-rank), one kernel column per step.  1 <= rank <= min(n, 1024).  L is held on
 * the device (n x rank, 8 n rank bytes).  Errors: INVALID_ARG if rank exceeds the numerical
 * rank of K (a non-positive pivot). */
GP_API gp_status gp_precond_create(gp_plan p, int rank, void *stream, gp_precond *out);

/* gp_precond_factor -- copies of the factor: pivots (host int64[rank], user indices, in
 * pivot order) and/or L (device, n x rank column-major, user order); either may be NULL. */
GP_API gp_status gp_precond_factor(gp_precond pc, int64_t *pivots, double *L, void *stream);

/* gp_precond_solve -- z = P^-1 r, P = L L^T + sigma2 I, by the Woodbury formula
 * (P:1080-1083): z = r / sigma2 - L C^-1 L^T r / sigma2^2, C = I + L^T L / sigma2 (C^-1
 * formed once per sigma2 from a host Cholesky of C; nb <= 8 columns stream L twice, more
 * go through cuBLAS GEMMs).  r, z: n x nb column-major (device, user order), may not
 * alias.  Synchronises `stream`. */
GP_API gp_status gp_precond_solve(gp_precond pc, double sigma2, const double *r, int nb,
                                  double *z, void *stream);

/* gp_precond_logdet -- log det P = N log sigma2 + log det(I + L^T L / sigma2) (Sylvester,
 * P:1087-1095); host result. */
GP_API gp_status gp_precond_logdet(gp_precond pc, double sigma2, double *logdet, void *stream);
/* gp_precond_destroy -- frees the preconditioner; if its plan's gp_destroy already ran
 * (deferred, see gp_destroy), the plan is freed with its last preconditioner. */
GP_API void gp_precond_destroy(gp_precond pc);

/* gp_mbcg -- Algorithm 2: CG on A = K + sigma2 I with nb right-hand sides B,
 * zero initial guess, preconditioner pc (NULL: identity), per-column stop at
 *   ||b_c - A x_c||_2 <= rtol ||b_c||_2 (on the recursive residual; rtol = 0: exactly
 *   max_iter iterations -- the Lanczos mode used for log-determinants).
 *   B, X          : n x nb column-major (device, user order).
 *   alpha_hist,
 *   beta_hist     : (host, may be NULL) max_iter x nb, entry [it * nb + c]: the CG
 *                   coefficients alpha_{it+1}, beta_{it+1} of column c; the Lanczos
 *                   tridiagonal of column c has diagonal 1/alpha_j + beta_{j-1}/alpha_{j-1}
 *                   and off-diagonal sqrt(beta_j)/alpha_j.
 *   iters_done    : (host, may be NULL) number of alpha's recorded per column.
 * Errors: BREAKDOWN (p^T A p <= 0).  Synchronises `stream`. */
GP_API gp_status gp_mbcg(gp_plan p, gp_precond pc, double sigma2, const double *B, int nb,
                         int max_iter, double rtol, double *X, double *alpha_hist,
                         double *beta_hist, int *iters_done, void *stream);

/* gp_lml -- log-marginal likelihood and its gradient (eq gp_log_likelihood; eq
 * gp_log_likelihood_derivative) for the centred response r (the fixed effects
 * removed first), as the paper estimates them (App A):
 *   r^T A^-1 r by CG to cg_rtol; log det A by N/l sum_i e1^T log(T_i) e1 over l probes and
 *   `lanczos_iters` Lanczos steps each, + log det P with a preconditioner;
 *   tr(A^-1 dA/dth) by Hutchinson from the probes' CG solutions.
 *   G : n x nprobe (device, user order) standard normal draws; W: rank x nprobe (device)
 *       standard normal draws, required iff pc != NULL: the probes are z = L w + sigma g
 *       ~ N(0, P) (reading R12), z = g without a preconditioner.
 * The caller supplies the random numbers (the library draws none).  Synchronises `stream`.
 * Errors: BREAKDOWN (CG breakdown or a non-positive Lanczos eigenvalue),
 * NOT_CONVERGED (the r solve). */
GP_API gp_status gp_lml(gp_plan p, gp_precond pc, double sigma2, const double *r,
                        const double *G, const double *W, int nprobe, int lanczos_iters,
                        double cg_rtol, gp_lml_result *out, void *stream);

/* Options / result of gp_fit (Algorithm 1).  Zero-initialise the options struct and set
 * what you need: zero fields take the defaults in brackets. */
typedef struct {
  double lr;            /* ADAM step on log(outputscale), log(c) [0.05] */
  int max_steps;        /* gradient steps per descent [50] */
  int max_outer;        /* GLS rounds after the OLS descent [3] */
  double grad_tol;      /* end a descent at ||grad_theta L|| / N <= grad_tol [1e-4] */
  double beta_tol;      /* end at ||beta_GLS - beta_old|| <= beta_tol [1e-3] */
  int lanczos_iters;    /* Lanczos steps per probe [25] */
  int precond_rank;     /* pivoted-Cholesky rank of every solve, 0 = none [0] */
  double cg_rtol;       /* relative residual of every CG solve [1e-8] */
} gp_fit_opts;

typedef struct {
  gp_kernel kernel;     /* fitted outputscale and lengthscales (l_k = c * l0_k) */
  double sigma;         /* fitted noise standard deviation */
  double beta[4];       /* GLS fixed effects for h(x) = [1, x] */
  int steps;            /* gradient steps taken */
  int outer;            /* GLS rounds taken */
  double lml;           /* stochastic LML at the last gradient evaluation */
  double grad_norm;     /* last ||grad_theta L|| / N */
} gp_fit_result;

/* gp_fit -- Algorithm 1: OLS fixed effects, then gradient descents on
 * theta = (log outputscale, log c) (c scales every lengthscale; GradDescStep = one ADAM
 * ascent step on the gp_lml estimate) with the closed-form sigma update
 *   sigma^2 = 1/N y^T (K(s / sigma_prev, l) + I)^-1 y
 * after each step; then rounds of GLS beta, a running average beta_AVG and a
 * descent on y - H beta_AVG, until successive beta_GLS differ by <= beta_tol (reading R13
 * in DESIGN.md: log-parameters, ADAM defaults, gradient norm per observation).
 *   x  : n x d row-major (device); k0: initial kernel (form, nu fixed); sigma0 > 0.
 *   y  : n (device, user order).  G: n x nprobe standard normals (device, user order),
 *   W  : precond_rank x nprobe standard normals (device) iff opts->precond_rank > 0.
 * The probes are the same at every step (common random numbers).  One plan setup per
 * gradient step (the lengthscale changes).  Synchronises `stream`. */
GP_API gp_status gp_fit(const double *x, int64_t n, int d, const gp_kernel *k0, double sigma0,
                        const double *y, const double *G, const double *W, int nprobe,
                        const gp_fit_opts *opts, gp_fit_result *out, void *stream);

/* gp_predict -- posterior mean mu(z_q) = h(z_q)^T beta + sum_i K(z_q, x_i) alpha_i
 * (P:86 [eq gp_mean], P:149 [eq gp_mean_2]).
 *   z      : m x d row-major (device); alpha: n (device, user order);
 *   beta   : (host) 1+d coefficients for the affine mean h(z) = [1, z], or NULL for
 *            out = K_zx alpha exactly;
 *   Hz     : for a basis mean, the m x L column-major basis at z (device) and
 *            beta of length L; pass NULL and L = 0 for the affine mean.
 *   out    : m (device).  The union structure x U z is built on the first call and cached
 *            on the plan: a later call with the same z pointer, the same m and bitwise-equal
 *            contents (compared on the device, one pass over z) reuses it (SURVEY §8(b)
 *            convention 4); any other z replaces the cache.  Synchronises `stream`. */
GP_API gp_status gp_predict(gp_plan p, const double *z, int64_t m, const double *alpha,
                     const double *beta, const double *Hz, int L, double *out, void *stream);

/* gp_plan_query -- introspection for tests and the bench (host value in *value):
 *   0 n, 1 d, 2 levels L, 3 bytes of device structure, 4 kernel launches per
 *   single-RHS gp_kmvm, 5 algorithmic HBM bytes per single-RHS gp_kmvm,
 *   6 d=1 apply path in use (1 = single-launch cooperative k_d1_lpc, 3 = three-launch
 *     reduce-then-scan),
 *   7 d=1 thread-block shape of path 1 (see gp_plan_set_option). */
GP_API gp_status gp_plan_query(gp_plan p, int what, int64_t *value);

/* gp_plan_set_option -- tuning / testing knobs (d = 1 only; ignored otherwise):
 *   option 0: force the d=1 apply path (0 auto, 1 single-chunk k_d1_lpc if it fits, 3 the
 *             three-launch reduce-then-scan path -- the automatic choice above the
 *             single-chunk capacity; 2 is rejected: the multi-sub-tile kernel is gone);
 *   option 1: thread-block shape of path 1 (threads x points per thread): 0 = 512x15
 *             (default), 1 = 384x19, 2 = 256x27;
 *   option 2: programmatic dependent launch of the d=1 kernel (1 default, 0 off);
 *   option 3: L2 prefetch of v before the user-order gathers (1 default, 0 off). */
GP_API gp_status gp_plan_set_option(gp_plan p, int option, int64_t value);

/* gp_destroy -- frees the plan and its device memory.  Preconditioners point into their
 * plan: while any built on p is alive the free is deferred to the last gp_precond_destroy
 * (p must not be used after gp_destroy either way). */
GP_API void gp_destroy(gp_plan p);
GP_API const char *gp_last_error(void);
/* Library version string, e.g. "gpmatern 0.1 sm_100a". */
GP_API const char *gp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GPMATERN_H */
