// lml.cu -- SURVEY §8(f) f3: the likelihood machinery of PAPER.md App A on top of the
// fast K.v apply.
//   * Precond: rank-k pivoted Cholesky K ~ L L^T (greedy pivot on the largest
//     remaining diagonal, ties -> smallest rank), P = L L^T + sigma^2 I applied by the
//     Woodbury formula, log det P by Sylvester's theorem.
//     L is n x k column-major in the plan's rank order; the Woodbury solve streams L twice
//     (k_wlt: L^T R, k_wly: R/s2 - L Y/s2^2) for up to 8 columns; C^-1 W, the Gram matrix
//     L^T L, the pivot GEMV and the solves with more columns go through cuBLAS.
//   * mbcg_rank: Algorithm 2 -- CG with several right-hand sides and the
//     preconditioner solve, zero initial guess, recording alpha_j, beta_j per iteration
//     (the Lanczos tridiagonals T_j); per-column stop (reading R8).
//   * slq: eqn approximationLogDet, e1^T log(T) e1 from an implicit-shift QL
//     eigen-decomposition of the small tridiagonal (first eigenvector components only).
//   * lml: eq gp_log_likelihood / _derivative with Hutchinson traces
//      -- probes z ~ N(0, P) (reading R12).
// All n-vectors live in rank order; every reduction is a fixed-order two-stage tree.
#include <cublas_v2.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "algebra.cuh"
#include "internal.h"

namespace gpm {

namespace {

constexpr int LB = 256;
constexpr int LG = 296;   // reduction partials per column

__device__ __forceinline__ double lblock_sum(double v, double* sh) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (warp == 0) {
    t = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
    for (int off = 16; off > 0; off >>= 1) t += __shfl_down_sync(0xffffffffu, t, off);
  }
  __syncthreads();
  return t;
}

inline int lgrid(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)); }

// ---- kernel matrix column K[:, p] (rank order) for the pivoted Cholesky
// profile k(s) = sum_q a_q s^q e^{-s}, s = scaled distance; os2 = outputscale^2
__device__ __forceinline__ double prof(int P, double s) {
  const double e = exp(-s);
  double poly = 0.0;
  for (int q = P; q >= 0; --q) poly = fma(poly, s, mcoef(P, q));
  return e * poly;
}


// col[r] = os2 k(x_r, x_p)  (the GEMV correction is applied by cuBLAS afterwards)
__global__ void k_kcol(const double* __restrict__ t, int64_t n, int d, int P, int prod, double os2,
                       const int* __restrict__ piv, int i, double* __restrict__ col) {
  const int p = piv[i];
  double tp[3];
  for (int k = 0; k < d; ++k) tp[k] = t[(size_t)k * n + p];
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    double v;
    if (!prod) {
      double s = 0.0;
      for (int k = 0; k < d; ++k) s += fabs(t[(size_t)k * n + r] - tp[k]);
      v = prof(P, s);
    } else {
      v = 1.0;
      for (int k = 0; k < d; ++k) v *= prof(P, fabs(t[(size_t)k * n + r] - tp[k]));
    }
    col[r] = os2 * v;
  }
}

// L[:, i] = col / sqrt(dp); diag -= L[:, i]^2 ; dp = pivot's remaining diagonal (pivd[i])

// k_pcupd followed by k_argmax1's stage 1 on the updated diagonal, in one pass (launched
// <<<LG, LB>>> like k_argmax1: the same grid-stride partition, so the same partials)
__global__ void k_pcupd_am(double* __restrict__ col, double* __restrict__ diag, int64_t n,
                           const int* __restrict__ piv, const double* __restrict__ pivd, int i,
                           double* __restrict__ pv, int* __restrict__ pi) {
  __shared__ double sv[LB];
  __shared__ int si[LB];
  const double inv = 1.0 / sqrt(pivd[i]);
  const int p = piv[i];
  double bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const double l = col[r] * inv;
    col[r] = l;
    const double v = r == p ? 0.0 : diag[r] - l * l;
    diag[r] = v;
    if (v > bv) { bv = v; bi = (int)r; }
  }
  sv[threadIdx.x] = bv;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double v2 = sv[threadIdx.x + o];
      const int i2 = si[threadIdx.x + o];
      if (v2 > sv[threadIdx.x] || (v2 == sv[threadIdx.x] && i2 < si[threadIdx.x])) {
        sv[threadIdx.x] = v2;
        si[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { pv[blockIdx.x] = sv[0]; pi[blockIdx.x] = si[0]; }
}

// argmax of diag (ties -> smallest index): stage 1 per block, stage 2 one block
__global__ void k_argmax1(const double* __restrict__ diag, int64_t n, double* __restrict__ pv,
                          int* __restrict__ pi) {
  __shared__ double sv[LB];
  __shared__ int si[LB];
  double bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const double v = diag[r];
    if (v > bv) { bv = v; bi = (int)r; }
  }
  sv[threadIdx.x] = bv;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double v2 = sv[threadIdx.x + o];
      const int i2 = si[threadIdx.x + o];
      if (v2 > sv[threadIdx.x] || (v2 == sv[threadIdx.x] && i2 < si[threadIdx.x])) {
        sv[threadIdx.x] = v2;
        si[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { pv[blockIdx.x] = sv[0]; pi[blockIdx.x] = si[0]; }
}
// stage 2 also gathers the pivot's row of L (Lp[j] = L[j n + p], j < i; was k_pivrow)
__global__ void k_argmax2(const double* __restrict__ pv, const int* __restrict__ pi, int nb,
                          int* __restrict__ piv, double* __restrict__ pivd, int i,
                          const double* __restrict__ L, int64_t n, double* __restrict__ Lp) {
  __shared__ double sv[LB];
  __shared__ int si[LB];
  double bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    const double v = pv[b];
    if (v > bv || (v == bv && pi[b] < bi)) { bv = v; bi = pi[b]; }
  }
  sv[threadIdx.x] = bv;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double v2 = sv[threadIdx.x + o];
      const int i2 = si[threadIdx.x + o];
      if (v2 > sv[threadIdx.x] || (v2 == sv[threadIdx.x] && i2 < si[threadIdx.x])) {
        sv[threadIdx.x] = v2;
        si[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { piv[i] = si[0]; pivd[i] = sv[0]; }
  const int p = si[0];
  for (int j = threadIdx.x; j < i; j += blockDim.x) Lp[j] = L[(size_t)j * n + p];
}

// ---- CG kernels (columns in blockIdx.y; vectors n x nb column-major)
__global__ void k_dotp(const double* __restrict__ A, const double* __restrict__ B, int64_t n,
                       double* __restrict__ part) {
  __shared__ double sh[32];
  const int c = blockIdx.y;
  const double* a = A + (size_t)c * n;
  const double* b = B + (size_t)c * n;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    acc = fma(a[i], b[i], acc);
  const double t = lblock_sum(acc, sh);
  if (threadIdx.x == 0) part[(size_t)c * gridDim.x + blockIdx.x] = t;
}
__global__ void k_sum(const double* __restrict__ part, int nb, double* __restrict__ out) {
  __shared__ double sh[32];
  const int c = blockIdx.x;
  double acc = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) acc += part[(size_t)c * nb + b];
  const double t = lblock_sum(acc, sh);
  if (threadIdx.x == 0) out[c] = t;
}
// Q += s2 P; part = P.Q
__global__ void k_mq(const double* __restrict__ P, double* __restrict__ Q, int64_t n, double s2,
                     double* __restrict__ part) {
  __shared__ double sh[32];
  const int c = blockIdx.y;
  const double* p = P + (size_t)c * n;
  double* q = Q + (size_t)c * n;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double pv = p[i];
    const double qv = fma(s2, pv, q[i]);
    q[i] = qv;
    acc = fma(pv, qv, acc);
  }
  const double t = lblock_sum(acc, sh);
  if (threadIdx.x == 0) part[(size_t)c * gridDim.x + blockIdx.x] = t;
}
// alpha_c = zr_c / pq_c ; history ; breakdown
__global__ void k_malpha(const double* __restrict__ part, int nb, const double* __restrict__ zr,
                         double* __restrict__ alpha, int* __restrict__ status,
                         double* __restrict__ ahist, int it, int ncol) {
  __shared__ double sh[32];
  const int c = blockIdx.x;
  double acc = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) acc += part[(size_t)c * nb + b];
  const double pq = lblock_sum(acc, sh);
  if (threadIdx.x == 0) {
    double a = 0.0;
    if (status[c] == 0) {
      if (!(pq > 0.0) || !isfinite(pq)) status[c] = 2;
      else a = zr[c] / pq;
      if (ahist && status[c] == 0) ahist[(size_t)it * ncol + c] = a;
    }
    alpha[c] = a;
  }
}
// X += a P ; R -= a Q ; part = R.R
__global__ void k_mupd(double* __restrict__ X, double* __restrict__ R, const double* __restrict__ P,
                       const double* __restrict__ Q, const double* __restrict__ alpha, int64_t n,
                       double* __restrict__ part) {
  __shared__ double sh[32];
  const int c = blockIdx.y;
  const double a = alpha[c];
  double* x = X + (size_t)c * n;
  double* r = R + (size_t)c * n;
  const double* p = P + (size_t)c * n;
  const double* q = Q + (size_t)c * n;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = fma(a, p[i], x[i]);
    const double rv = fma(-a, q[i], r[i]);
    r[i] = rv;
    acc = fma(rv, rv, acc);
  }
  const double t = lblock_sum(acc, sh);
  if (threadIdx.x == 0) part[(size_t)c * gridDim.x + blockIdx.x] = t;
}
// beta_c = zr_new / zr ; convergence on ||R||^2 <= tol2_c ; history
__global__ void k_mbeta(const double* __restrict__ part_rr, int nb,
                        const double* __restrict__ part_zr, int nb2,
                        double* __restrict__ zr, const double* __restrict__ tol2,
                        double* __restrict__ beta, int* __restrict__ status,
                        int* __restrict__ iters, double* __restrict__ bhist, int it, int ncol) {
  __shared__ double sh[32];
  const int c = blockIdx.x;
  double a1 = 0.0, a2 = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) a1 += part_rr[(size_t)c * nb + b];
  for (int b = threadIdx.x; b < nb2; b += blockDim.x) a2 += part_zr[(size_t)c * nb2 + b];
  const double rr = lblock_sum(a1, sh);
  const double zn = lblock_sum(a2, sh);
  if (threadIdx.x == 0) {
    double bt = 0.0;
    if (status[c] == 0) {
      iters[c] = it + 1;
      bt = zn / zr[c];
      zr[c] = zn;
      if (bhist) bhist[(size_t)it * ncol + c] = bt;
      if (rr <= tol2[c]) status[c] = 1;
    }
    beta[c] = bt;
  }
}
// P = Z + beta P (active columns)
__global__ void k_mpupd(double* __restrict__ P, const double* __restrict__ Z,
                        const double* __restrict__ beta, const int* __restrict__ status, int64_t n) {
  const int c = blockIdx.y;
  if (status[c] != 0) return;
  const double b = beta[c];
  double* p = P + (size_t)c * n;
  const double* z = Z + (size_t)c * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = fma(b, p[i], z[i]);
}
__global__ void k_fill(double* __restrict__ x, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] = v;
}
// out = a*X + b*Y (elementwise, n*nb)
__global__ void k_lin(const double* __restrict__ X, const double* __restrict__ Y, double a,
                      double b, int64_t nk, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nk;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a * X[i] + (Y ? b * Y[i] : 0.0);
}

// symmetric k x k Cholesky (lower, in place, row-major); false if not SPD
bool chol(std::vector<double>& A, int k) {
  for (int j = 0; j < k; ++j) {
    double s = A[j * k + j];
    for (int q = 0; q < j; ++q) s -= A[j * k + q] * A[j * k + q];
    if (!(s > 0.0)) return false;
    const double d = std::sqrt(s);
    A[j * k + j] = d;
    for (int i = j + 1; i < k; ++i) {
      double t = A[i * k + j];
      for (int q = 0; q < j; ++q) t -= A[i * k + q] * A[j * k + q];
      A[i * k + j] = t / d;
    }
  }
  return true;
}

const char* cublas_msg(cublasStatus_t st) {
  switch (st) {
    case CUBLAS_STATUS_NOT_INITIALIZED: return "cuBLAS not initialised";
    case CUBLAS_STATUS_ALLOC_FAILED: return "cuBLAS allocation failed";
    case CUBLAS_STATUS_INVALID_VALUE: return "cuBLAS invalid value";
    case CUBLAS_STATUS_EXECUTION_FAILED: return "cuBLAS execution failed";
    default: return "cuBLAS error";
  }
}
#define GPM_CUBLAS(x)                                                  \
  do {                                                                 \
    cublasStatus_t st_ = (x);                                          \
    if (st_ != CUBLAS_STATUS_SUCCESS) return fail(GP_ERR_CUDA, cublas_msg(st_)); \
  } while (0)

}  // namespace

// ---------------------------------------------------------------------------
// Preconditioner
gp_status precond_build(Precond& pc, Plan& pl, int k, cudaStream_t s) {
  const int64_t n = pl.n;
  pc.pl = &pl;
  pc.k = k;
  pc.n = n;
  GPM_CUBLAS(cublasCreate(&pc.h));
  GPM_CUBLAS(cublasSetStream(pc.h, s));
  GPM_CUBLAS(cublasSetPointerMode(pc.h, CUBLAS_POINTER_MODE_HOST));
  GPM_TRY(pc.L.alloc(sizeof(double) * (size_t)n * k));
  DevBuf diag, pv, pi, piv, pivd, Lp, G;
  struct Guard {   // scratch released on every exit path
    DevBuf* b[7];
    ~Guard() { for (auto* x : b) x->release(); }
  } guard{{&diag, &pv, &pi, &piv, &pivd, &Lp, &G}};
  GPM_TRY(diag.alloc(8 * n));
  GPM_TRY(pv.alloc(8 * LG));
  GPM_TRY(pi.alloc(4 * LG));
  GPM_TRY(piv.alloc(4 * (size_t)k));
  GPM_TRY(pivd.alloc(8 * (size_t)k));
  GPM_TRY(Lp.alloc(8 * (size_t)k + 8));
  // diag K = outputscale^2 at every point (stationary kernel)
  k_fill<<<lgrid(n), 256, 0, s>>>(diag.as<double>(), n, pl.os2);
  double* L = pc.L.as<double>();
  const int prod = pl.form == GP_FORM_PRODUCT ? 1 : 0;
  for (int i = 0; i < k; ++i) {
    // step i's argmax partials: k_argmax1 at i = 0, else step i-1's k_pcupd_am
    if (i == 0) k_argmax1<<<LG, LB, 0, s>>>(diag.as<double>(), n, pv.as<double>(), pi.as<int>());
    k_argmax2<<<1, LB, 0, s>>>(pv.as<double>(), pi.as<int>(), LG, piv.as<int>(),
                               pivd.as<double>(), i, L, n, Lp.as<double>());
    double* col = L + (size_t)i * n;
    k_kcol<<<lgrid(n), 256, 0, s>>>(pl.t.as<double>(), n, pl.d, pl.P, prod, pl.os2,
                                    piv.as<int>(), i, col);
    if (i > 0) {
      const double m1 = -1.0, one = 1.0;
      GPM_CUBLAS(cublasDgemv(pc.h, CUBLAS_OP_N, (int)n, i, &m1, L, (int)n, Lp.as<double>(), 1,
                             &one, col, 1));
    }
    k_pcupd_am<<<LG, LB, 0, s>>>(col, diag.as<double>(), n, piv.as<int>(), pivd.as<double>(),
                                 i, pv.as<double>(), pi.as<int>());
    GPM_CUDA(cudaGetLastError());
  }
  pc.piv.resize(k);
  std::vector<double> hpd(k);
  GPM_CUDA(cudaMemcpyAsync(pc.piv.data(), piv.ptr, 4 * (size_t)k, cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaMemcpyAsync(hpd.data(), pivd.ptr, 8 * (size_t)k, cudaMemcpyDeviceToHost, s));
  // Gram matrix G = L^T L (k x k, symmetric)
  GPM_TRY(G.alloc(8 * (size_t)k * k));
  const double one = 1.0, zero = 0.0;
  GPM_CUBLAS(cublasDgemm(pc.h, CUBLAS_OP_T, CUBLAS_OP_N, k, k, (int)n, &one, L, (int)n, L,
                         (int)n, &zero, G.as<double>(), k));
  pc.G.resize((size_t)k * k);
  GPM_CUDA(cudaMemcpyAsync(pc.G.data(), G.ptr, 8 * (size_t)k * k, cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < k; ++i)
    if (!(hpd[i] > 0.0))
      return fail(GP_ERR_INVALID_ARG, "pivoted Cholesky: rank " + std::to_string(k) +
                                          " exceeds the numerical rank of K (pivot " +
                                          std::to_string(i) + ")");
  GPM_TRY(pc.Cinv.alloc(8 * (size_t)k * k));
  return GP_OK;
}

// C = I + G / s2 ; Cinv (device) and log det C for this sigma^2
static gp_status precond_sigma(Precond& pc, double s2, cudaStream_t s) {
  if (pc.s2 == s2) return GP_OK;
  const int k = pc.k;
  std::vector<double> C((size_t)k * k);
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j)
      C[(size_t)i * k + j] = 0.5 * (pc.G[(size_t)i * k + j] + pc.G[(size_t)j * k + i]) / s2 +
                             (i == j ? 1.0 : 0.0);
  if (!chol(C, k)) return fail(GP_ERR_INVALID_ARG, "Woodbury capacitance matrix not SPD");
  double ld = 0.0;
  for (int i = 0; i < k; ++i) ld += 2.0 * std::log(C[(size_t)i * k + i]);
  // C^-1 from the Cholesky factor C = F F^T (F lower, row-major in C, i.e. U = F^T upper
  // in cuBLAS's column-major view): X = U^-1 by one triangular solve on the identity, then
  // C^-1 = U^-1 U^-T = X X^T (device, O(k^3) flops off the host)
  DevBuf Fd, Xd;
  struct Guard {
    DevBuf* b[2];
    ~Guard() { for (auto* x : b) x->release(); }
  } guard{{&Fd, &Xd}};
  GPM_TRY(Fd.alloc(8 * (size_t)k * k));
  GPM_TRY(Xd.alloc(8 * (size_t)k * k));
  std::vector<double> I((size_t)k * k, 0.0);
  for (int i = 0; i < k; ++i) I[(size_t)i * k + i] = 1.0;
  GPM_CUDA(cudaMemcpyAsync(Fd.ptr, C.data(), 8 * (size_t)k * k, cudaMemcpyHostToDevice, s));
  GPM_CUDA(cudaMemcpyAsync(Xd.ptr, I.data(), 8 * (size_t)k * k, cudaMemcpyHostToDevice, s));
  GPM_CUBLAS(cublasSetStream(pc.h, s));
  const double one = 1.0, zero = 0.0;
  GPM_CUBLAS(cublasDtrsm(pc.h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N,
                         CUBLAS_DIAG_NON_UNIT, k, k, &one, Fd.as<double>(), k, Xd.as<double>(), k));
  GPM_CUBLAS(cublasDgemm(pc.h, CUBLAS_OP_N, CUBLAS_OP_T, k, k, k, &one, Xd.as<double>(), k,
                         Xd.as<double>(), k, &zero, pc.Cinv.as<double>(), k));
  GPM_CUDA(cudaStreamSynchronize(s));
  pc.s2 = s2;
  pc.logdetC = ld;
  return GP_OK;
}

double precond_logdet_val(const Precond& pc) {
  return (double)pc.n * std::log(pc.s2) + pc.logdetC;
}

gp_status precond_logdet(Precond& pc, double s2, double* out, cudaStream_t s) {
  GPM_TRY(precond_sigma(pc, s2, s));
  *out = precond_logdet_val(pc);
  return GP_OK;
}

// ---- Woodbury solve for a few columns (nb <= 8): the two passes over L (n x k, the
// dominant traffic: 8 n k bytes each) as streaming kernels instead of the library's
// tall-skinny GEMMs.  Both are HBM-bound: L is read once per pass, coalesced along n.
template <int NB>
__host__ __device__ constexpr int wb_rows() { return NB >= 8 ? 128 : 256; }   // k_wlt: rows of L per CTA
constexpr int WB_THREADS = 256;

// k_wlt: partial[(c k + j) nblk + b] = sum_{i in row block b} L[j n + i] R[c n + i].
// Each lane keeps its rows' R values in registers for the whole CTA; a warp takes 32 / NB
// columns at a time (32 partial dot products per lane) and reduces them with one
// reduce-scatter butterfly (31 shuffles instead of 5 per value), leaving lane l with value l.
constexpr int WT_THREADS = 128;   // k_wlt: 4 warps per CTA, 3 CTAs per SM
template <int NB>
__global__ void __launch_bounds__(WT_THREADS, 3) k_wlt(const double* __restrict__ L,
                                                    const double* __restrict__ R, int64_t n,
                                                    int k, int nb, double* __restrict__ part) {
  constexpr int WB_ROWS = wb_rows<NB>();
  constexpr int RPL = WB_ROWS / 32;   // rows per lane
  constexpr int G = 32 / NB;          // columns per warp step
  const int64_t i0 = (int64_t)blockIdx.x * WB_ROWS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nblk = gridDim.x;
  double rr[NB][RPL];
#pragma unroll
  for (int c = 0; c < NB; ++c)
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
      const int64_t i = i0 + lane + 32 * t;
      rr[c][t] = (c < nb && i < n) ? __ldg(R + (int64_t)c * n + i) : 0.0;
    }
  for (int j0 = warp * G; j0 < k; j0 += (WT_THREADS / 32) * G) {
    double vals[32];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int j = j0 + g;
      const double* Lj = L + (int64_t)j * n + i0 + lane;
      double l[RPL];
#pragma unroll
      for (int t = 0; t < RPL; ++t)
        l[t] = (j < k && i0 + lane + 32 * t < n) ? __ldcs(Lj + 32 * t) : 0.0;
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t < RPL; ++t) acc = fma(l[t], rr[c][t], acc);
        vals[g * NB + c] = acc;
      }
    }
    // reduce-scatter: after the step with offset s, a lane holds the half of the values
    // selected by its bit s; at the end vals[0] is the warp total of value `lane`
#pragma unroll
    for (int sft = 16; sft >= 1; sft >>= 1) {
      const bool up = (lane & sft) != 0;
#pragma unroll
      for (int i = 0; i < sft; ++i) {
        const double send = up ? vals[i] : vals[i + sft];
        const double keep = up ? vals[i + sft] : vals[i];
        vals[i] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
      }
    }
    const int j = j0 + lane / NB, c = lane % NB;
    if (j < k && j < j0 + G) part[((int64_t)c * k + j) * nblk + blockIdx.x] = vals[0];
  }
}

// k_wred: W[o] = sum_b part[o nblk + b], o = c k + j (fixed order: lane-strided, then a
// warp tree; one warp per output, coalesced along b)
__global__ void k_wred(const double* __restrict__ part, int nblk, int kn,
                       double* __restrict__ W) {
  const int o = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (o >= kn) return;
  double s = 0.0;
  const double* po = part + (int64_t)o * nblk;
  for (int b = lane; b < nblk; b += 32) s += po[b];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
  if (lane == 0) W[o] = s;
}

// k_wly: Z[c n + i] = b R[c n + i] + a sum_j L[j n + i] Y[c k + j]  (Z may alias R)
template <int NB>
__global__ void __launch_bounds__(WB_THREADS) k_wly(const double* __restrict__ L,
                                                    const double* R, int64_t n, int k, int nb,
                                                    const double* __restrict__ Y, double a,
                                                    double b, double* Z, double* zr_part) {
  extern __shared__ double Ys[];   // [k][NB]
  __shared__ double wsum[NB][WB_THREADS / 32];
  for (int t = threadIdx.x; t < k * NB; t += WB_THREADS) {
    const int j = t / NB, c = t % NB;
    Ys[t] = c < nb ? __ldg(Y + (int64_t)c * k + j) : 0.0;
  }
  __syncthreads();
  const int64_t i0 = (int64_t)blockIdx.x * WB_THREADS + threadIdx.x;
  const bool live = i0 < n;
  const int64_t i = live ? i0 : n - 1;   // dead lanes recompute the last row, write nothing
  double acc[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) acc[c] = 0.0;
  const double* Li = L + i;
  int j = 0;
  for (; j + 8 <= k; j += 8) {
    double l[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) l[u] = __ldcs(Li + (int64_t)(j + u) * n);
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < NB; ++c) acc[c] = fma(l[u], Ys[(j + u) * NB + c], acc[c]);
  }
  for (; j < k; ++j) {
    const double l = __ldcs(Li + (int64_t)j * n);
#pragma unroll
    for (int c = 0; c < NB; ++c) acc[c] = fma(l, Ys[j * NB + c], acc[c]);
  }
  double zr[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    zr[c] = 0.0;
    if (c < nb && live) {
      const double rv = R[(int64_t)c * n + i];
      const double zv = fma(b, rv, a * acc[c]);
      Z[(int64_t)c * n + i] = zv;
      zr[c] = zv * rv;
    }
  }
  if (zr_part) {   // fixed-order block sums of z.r per column (Alg 2's z^T r)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int c = 0; c < NB; ++c) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) zr[c] += __shfl_down_sync(0xffffffffu, zr[c], off);
      if (lane == 0) wsum[c][warp] = zr[c];
    }
    __syncthreads();
    if (threadIdx.x < nb) {
      double t = 0.0;
      for (int w = 0; w < WB_THREADS / 32; ++w) t += wsum[threadIdx.x][w];
      zr_part[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = t;
    }
  }
}

template <int NB>
static gp_status wood_stream(Precond& pc, const double* R, int nb, double* Z, double a, double b,
                             cudaStream_t s, double* zr_part, int* zr_nblk) {
  const int k = pc.k;
  const int64_t n = pc.n;
  const int nblk = (int)((n + wb_rows<NB>() - 1) / wb_rows<NB>());
  const size_t pb = 8 * (size_t)nblk * NB * k;
  if (pc.Wp.bytes < pb) GPM_TRY(pc.Wp.alloc(pb));
  k_wlt<NB><<<nblk, WT_THREADS, 0, s>>>(pc.L.as<double>(), R, n, k, nb, pc.Wp.as<double>());
  GPM_CUDA(cudaGetLastError());
  const int kn = k * nb;   // W is k x nb column-major
  k_wred<<<(kn + 7) / 8, 256, 0, s>>>(pc.Wp.as<double>(), nblk, kn, pc.W.as<double>());
  GPM_CUDA(cudaGetLastError());
  const double one = 1.0, zero = 0.0;
  GPM_CUBLAS(cublasSetStream(pc.h, s));
  GPM_CUBLAS(cublasDgemm(pc.h, CUBLAS_OP_N, CUBLAS_OP_N, k, nb, k, &one, pc.Cinv.as<double>(), k,
                         pc.W.as<double>(), k, &zero, pc.Y.as<double>(), k));
  const size_t ysm = 8 * (size_t)k * NB;
  // opt in once per instantiation to the largest Y any rank can need (k <= 1024): the
  // static wsum[][] adds to the dynamic size, so a 48 KB test on ysm alone is not enough
  static bool attr_set = false;
  if (!attr_set) {
    GPM_CUDA(cudaFuncSetAttribute(k_wly<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(8 * 1024 * NB)));
    attr_set = true;
  }
  k_wly<NB><<<(int)((n + WB_THREADS - 1) / WB_THREADS), WB_THREADS, ysm, s>>>(
      pc.L.as<double>(), R, n, k, nb, pc.Y.as<double>(), a, b, Z, zr_part);
  GPM_CUDA(cudaGetLastError());
  if (zr_nblk) *zr_nblk = zr_part ? (int)((n + WB_THREADS - 1) / WB_THREADS) : 0;
  return GP_OK;
}

// Z = P^-1 R = R/s2 - L Cinv L^T R / s2^2   (rank order, nb columns)
gp_status precond_apply(Precond& pc, double s2, const double* R, int nb, double* Z,
                        cudaStream_t s, double* zr_part, int* zr_nblk) {
  if (zr_nblk) *zr_nblk = 0;
  GPM_TRY(precond_sigma(pc, s2, s));
  const int k = pc.k;
  const int n = (int)pc.n;
  if (pc.W.bytes < 8 * (size_t)k * nb) GPM_TRY(pc.W.alloc(8 * (size_t)k * nb));
  if (pc.Y.bytes < 8 * (size_t)k * nb) GPM_TRY(pc.Y.alloc(8 * (size_t)k * nb));
  const double one = 1.0, zero = 0.0, a = -1.0 / (s2 * s2), b = 1.0 / s2;
  if (!getenv("GPM_WOODBURY_CUBLAS") && k * 8 * 8 <= 200 * 1024) {
    if (nb == 1) return wood_stream<1>(pc, R, nb, Z, a, b, s, zr_part, zr_nblk);
    if (nb == 2) return wood_stream<2>(pc, R, nb, Z, a, b, s, zr_part, zr_nblk);
    if (nb <= 4) return wood_stream<4>(pc, R, nb, Z, a, b, s, zr_part, zr_nblk);
    if (nb <= 8) return wood_stream<8>(pc, R, nb, Z, a, b, s, zr_part, zr_nblk);
  }
  GPM_CUBLAS(cublasSetStream(pc.h, s));
  GPM_CUBLAS(cublasDgemm(pc.h, CUBLAS_OP_T, CUBLAS_OP_N, k, nb, n, &one, pc.L.as<double>(), n, R,
                         n, &zero, pc.W.as<double>(), k));
  GPM_CUBLAS(cublasDgemm(pc.h, CUBLAS_OP_N, CUBLAS_OP_N, k, nb, k, &one, pc.Cinv.as<double>(), k,
                         pc.W.as<double>(), k, &zero, pc.Y.as<double>(), k));
  if (Z != R) GPM_CUDA(cudaMemcpyAsync(Z, R, 8 * (size_t)n * nb, cudaMemcpyDeviceToDevice, s));
  GPM_CUBLAS(cublasDgemm(pc.h, CUBLAS_OP_N, CUBLAS_OP_N, n, nb, k, &a, pc.L.as<double>(), n,
                         pc.Y.as<double>(), k, &b, Z, n));
  return GP_OK;
}

// z = L w + sigma g  (a sample of N(0, P) from standard normals g (n) and w (k))
gp_status precond_sample(Precond& pc, double s2, const double* G, const double* W, int nb,
                         double* Z, cudaStream_t s) {
  const int k = pc.k;
  const int n = (int)pc.n;
  GPM_CUBLAS(cublasSetStream(pc.h, s));
  const double one = 1.0, sg = std::sqrt(s2);
  k_lin<<<lgrid((int64_t)n * nb), 256, 0, s>>>(G, nullptr, sg, 0.0, (int64_t)n * nb, Z);
  GPM_CUDA(cudaGetLastError());
  GPM_CUBLAS(cublasDgemm(pc.h, CUBLAS_OP_N, CUBLAS_OP_N, n, nb, k, &one, pc.L.as<double>(), n, W,
                         k, &one, Z, n));
  return GP_OK;
}

void precond_free(Precond& pc) {
  pc.L.release();
  pc.Cinv.release();
  pc.W.release();
  pc.Y.release();
  pc.Wp.release();
  if (pc.h) cublasDestroy(pc.h);
  pc.h = nullptr;
}

// ---------------------------------------------------------------------------
// Algorithm 2 in rank order.  B, X: n x nb.  tol2[c]: absolute stop level for ||r_c||^2
// (0: run max_iter iterations).  ahist/bhist: device, max_iter x nb (may be null).
gp_status mbcg_rank(Plan& pl, Precond* pc, double s2, const double* B, int nb, int max_iter,
                    const std::vector<double>& tol2, double* X, double* ahist, double* bhist,
                    std::vector<int>& iters, std::vector<int>& status, double* P0,
                    cudaStream_t s) {
  const int64_t n = pl.n;
  const size_t nk = (size_t)n * nb;
  DevBuf bR, bP, bQ, bZ, bpart, bsc;
  struct Guard {
    DevBuf* b[6];
    ~Guard() { for (auto* x : b) x->release(); }
  } guard{{&bR, &bP, &bQ, &bZ, &bpart, &bsc}};
  GPM_TRY(bR.alloc(8 * nk));
  GPM_TRY(bP.alloc(8 * nk));
  GPM_TRY(bQ.alloc(8 * nk));
  if (pc) GPM_TRY(bZ.alloc(8 * nk));
  // part: LG partials per column; part2: z.r partials (LG from k_dotp, or one per k_wly CTA)
  GPM_TRY(bpart.alloc(8 * (size_t)nb * (LG + std::max(LG, precond_zr_blocks(n)))));
  GPM_TRY(bsc.alloc(8 * 4 * (size_t)nb + 4 * 2 * (size_t)nb + 64));
  double* R = bR.as<double>();
  double* Pm = bP.as<double>();
  double* Q = bQ.as<double>();
  double* Z = pc ? bZ.as<double>() : R;
  double* part = bpart.as<double>();
  double* part2 = part + (size_t)LG * nb;
  double* zr = bsc.as<double>();
  double* t2 = zr + nb;
  double* al = t2 + nb;
  double* be = al + nb;
  int* st = reinterpret_cast<int*>(be + nb);
  int* itc = st + nb;

  GPM_CUDA(cudaMemsetAsync(X, 0, 8 * nk, s));
  GPM_CUDA(cudaMemcpyAsync(R, B, 8 * nk, cudaMemcpyDeviceToDevice, s));
  if (pc) GPM_TRY(precond_apply(*pc, s2, R, nb, Z, s));
  GPM_CUDA(cudaMemcpyAsync(Pm, Z, 8 * nk, cudaMemcpyDeviceToDevice, s));
  if (P0) GPM_CUDA(cudaMemcpyAsync(P0, Z, 8 * nk, cudaMemcpyDeviceToDevice, s));   // P^-1 b
  k_dotp<<<dim3(LG, nb), LB, 0, s>>>(Z, R, n, part);
  k_sum<<<nb, LB, 0, s>>>(part, LG, zr);
  k_dotp<<<dim3(LG, nb), LB, 0, s>>>(R, R, n, part);
  DevBuf brr;
  GPM_TRY(brr.alloc(8 * (size_t)nb));
  k_sum<<<nb, LB, 0, s>>>(part, LG, brr.as<double>());
  GPM_CUDA(cudaGetLastError());
  std::vector<double> hrr(nb), hzr(nb);
  GPM_CUDA(cudaMemcpyAsync(hrr.data(), brr.ptr, 8 * (size_t)nb, cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaMemcpyAsync(hzr.data(), zr, 8 * (size_t)nb, cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  brr.release();
  status.assign(nb, 0);
  iters.assign(nb, 0);
  for (int c = 0; c < nb; ++c)
    if (hrr[c] == 0.0 || hrr[c] <= tol2[c]) status[c] = 1;   // x = 0 already meets the level
  GPM_CUDA(cudaMemcpyAsync(t2, tol2.data(), 8 * (size_t)nb, cudaMemcpyHostToDevice, s));
  GPM_CUDA(cudaMemcpyAsync(st, status.data(), 4 * (size_t)nb, cudaMemcpyHostToDevice, s));
  GPM_CUDA(cudaMemsetAsync(itc, 0, 4 * (size_t)nb, s));

  std::vector<char> active(nb);
  int it = 0;
  bool any = false;
  for (int c = 0; c < nb; ++c) { active[c] = status[c] == 0; any |= active[c] != 0; }
  while (any && it < max_iter) {
    for (int step = 0; step < 8 && it < max_iter; ++step, ++it) {
      // T = A Pbar (active columns; maximal runs through one multi-RHS apply)
      for (int c = 0; c < nb;) {
        if (!active[c]) { ++c; continue; }
        int e = c;
        while (e < nb && active[e]) ++e;
        GPM_TRY(apply_rank(pl, Pm + (size_t)c * n, Q + (size_t)c * n, e - c, s));
        c = e;
      }
      k_mq<<<dim3(LG, nb), LB, 0, s>>>(Pm, Q, n, s2, part);
      k_malpha<<<nb, LB, 0, s>>>(part, LG, zr, al, st, ahist, it, nb);
      k_mupd<<<dim3(LG, nb), LB, 0, s>>>(X, R, Pm, Q, al, n, part);
      int nzr = LG;
      if (pc) {   // z.r comes out of the Woodbury kernel when it streams (else k_dotp)
        GPM_TRY(precond_apply(*pc, s2, R, nb, Z, s, part2, &nzr));
        if (nzr == 0) {
          k_dotp<<<dim3(LG, nb), LB, 0, s>>>(Z, R, n, part2);
          nzr = LG;
        }
      }
      k_mbeta<<<nb, LB, 0, s>>>(part, LG, pc ? part2 : part, nzr, zr, t2, be, st, itc, bhist,
                                it, nb);
      k_mpupd<<<dim3(LG, nb), LB, 0, s>>>(Pm, Z, be, st, n);
    }
    GPM_CUDA(cudaGetLastError());
    GPM_CUDA(cudaMemcpyAsync(status.data(), st, 4 * (size_t)nb, cudaMemcpyDeviceToHost, s));
    GPM_CUDA(cudaStreamSynchronize(s));
    any = false;
    for (int c = 0; c < nb; ++c) {
      active[c] = status[c] == 0;
      any |= active[c] != 0;
      if (status[c] == 2) any = false;
    }
    bool broke = false;
    for (int c = 0; c < nb; ++c) broke |= status[c] == 2;
    if (broke) break;
  }
  GPM_CUDA(cudaMemcpyAsync(iters.data(), itc, 4 * (size_t)nb, cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  return GP_OK;
}

// ---------------------------------------------------------------------------
// e1^T f(T) e1 for the symmetric tridiagonal T (diag d[0..m-1], off e[0..m-2]) with
// f = log: implicit-shift QL (Wilkinson shift), eigenvalues in d, first eigenvector
// components in z.  Returns false on non-convergence or a non-positive eigenvalue.
static bool tridiag_log_e1(std::vector<double> d, std::vector<double> e, double* out) {
  const int m = (int)d.size();
  e.resize(m, 0.0);
  std::vector<double> z(m, 0.0);
  z[0] = 1.0;
  for (int l = 0; l < m; ++l) {
    int iter = 0;
    while (true) {
      int mm = l;
      for (; mm < m - 1; ++mm) {
        const double dd = std::fabs(d[mm]) + std::fabs(d[mm + 1]);
        if (std::fabs(e[mm]) <= 1e-16 * dd) break;
      }
      if (mm == l) break;
      if (++iter > 200) return false;
      double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
      double r = std::hypot(g, 1.0);
      g = d[mm] - d[l] + e[l] / (g + std::copysign(r, g));
      double sn = 1.0, cs = 1.0, p = 0.0;
      int i = mm - 1;
      bool early = false;
      for (; i >= l; --i) {
        double f = sn * e[i];
        const double b = cs * e[i];
        r = std::hypot(f, g);
        e[i + 1] = r;
        if (r == 0.0) {
          d[i + 1] -= p;
          e[mm] = 0.0;
          early = true;
          break;
        }
        sn = f / r;
        cs = g / r;
        g = d[i + 1] - p;
        r = (d[i] - g) * sn + 2.0 * cs * b;
        p = sn * r;
        d[i + 1] = g + p;
        g = cs * r - b;
        // rotate the first row of the eigenvector matrix (columns i, i+1)
        f = z[i + 1];
        z[i + 1] = sn * z[i] + cs * f;
        z[i] = cs * z[i] - sn * f;
      }
      if (early) continue;
      d[l] -= p;
      e[l] = g;
      e[mm] = 0.0;
    }
  }
  double acc = 0.0;
  for (int j = 0; j < m; ++j) {
    if (!(d[j] > 0.0) || !std::isfinite(d[j])) return false;
    acc += z[j] * z[j] * std::log(d[j]);
  }
  *out = acc;
  return true;
}

// Lanczos tridiagonal of column c from the CG coefficients (Alg 2)
gp_status slq_column(const double* ah, const double* bh, int nb, int c, int m, double* q) {
  if (m < 1) return fail(GP_ERR_BREAKDOWN, "Lanczos quadrature: no iteration recorded");
  std::vector<double> d(m), e(std::max(m - 1, 0));
  for (int j = 0; j < m; ++j) {
    const double a = ah[(size_t)j * nb + c];
    d[j] = 1.0 / a + (j > 0 ? bh[(size_t)(j - 1) * nb + c] / ah[(size_t)(j - 1) * nb + c] : 0.0);
    if (j + 1 < m) e[j] = std::sqrt(bh[(size_t)j * nb + c]) / a;
  }
  if (!tridiag_log_e1(d, e, q))
    return fail(GP_ERR_BREAKDOWN, "Lanczos tridiagonal has a non-positive or unresolved "
                                  "eigenvalue (loss of orthogonality, P:713)");
  return GP_OK;
}

// ---------------------------------------------------------------------------
// gp_lml: value and gradient of the log-marginal likelihood (App A).
gp_status lml_eval(Plan& pl, Precond* pc, double s2, const double* r_user, const double* G_user,
                   const double* W, int nprobe, int m, double cg_rtol, gp_lml_result* out,
                   cudaStream_t s) {
  const int64_t n = pl.n;
  const int l = nprobe;
  const int nc = 1 + l;                    // column 0: the response, 1..l: the probes
  DevBuf bB, bX, bP0, bK, bD, bpart, bdots, bah, bbh;
  struct Guard {
    DevBuf* b[9];
    ~Guard() { for (auto* x : b) x->release(); }
  } guard{{&bB, &bX, &bP0, &bK, &bD, &bpart, &bdots, &bah, &bbh}};
  GPM_TRY(bB.alloc(8 * (size_t)n * nc));
  GPM_TRY(bX.alloc(8 * (size_t)n * nc));
  GPM_TRY(bP0.alloc(8 * (size_t)n * nc));
  GPM_TRY(bK.alloc(8 * (size_t)n * nc));
  GPM_TRY(bD.alloc(8 * (size_t)n * nc));
  GPM_TRY(bpart.alloc(8 * (size_t)LG * nc));
  GPM_TRY(bdots.alloc(8 * (size_t)nc * 4));
  GPM_TRY(bah.alloc(8 * (size_t)m * l));
  GPM_TRY(bbh.alloc(8 * (size_t)m * l));
  double* B = bB.as<double>();
  double* X = bX.as<double>();
  double* P0 = bP0.as<double>();
  double* KP = bK.as<double>();
  double* DP = bD.as<double>();
  double* dots = bdots.as<double>();
  // rank-order right-hand sides
  GPM_TRY(permute_vec(pl, r_user, B, true, s));
  for (int c = 0; c < l; ++c)
    GPM_TRY(permute_vec(pl, G_user + (size_t)c * n, P0 + (size_t)c * n, true, s));
  if (pc) {
    GPM_TRY(precond_sample(*pc, s2, P0, W, l, B + n, s));   // z = L w + sigma g ~ N(0, P)
  } else {
    GPM_CUDA(cudaMemcpyAsync(B + n, P0, 8 * (size_t)n * l, cudaMemcpyDeviceToDevice, s));
  }
  // (1) a = A^-1 r to cg_rtol
  std::vector<int> it1, st1, itl, stl;
  {
    k_dotp<<<dim3(LG, 1), LB, 0, s>>>(B, B, n, bpart.as<double>());
    k_sum<<<1, LB, 0, s>>>(bpart.as<double>(), LG, dots);
    double rr = 0.0;
    GPM_CUDA(cudaMemcpyAsync(&rr, dots, 8, cudaMemcpyDeviceToHost, s));
    GPM_CUDA(cudaStreamSynchronize(s));
    std::vector<double> t2(1, cg_rtol * cg_rtol * rr);
    const int cap = (int)std::min<int64_t>(std::max<int64_t>(1000, 20 * n), 200000);
    GPM_TRY(mbcg_rank(pl, pc, s2, B, 1, cap, t2, X, nullptr, nullptr, it1, st1, nullptr, s));
    if (st1[0] == 2) return fail(GP_ERR_BREAKDOWN, "CG breakdown in the r solve");
    if (st1[0] != 1) return fail(GP_ERR_NOT_CONVERGED, "CG for A^-1 r did not reach cg_rtol");
  }
  // (2) probes: m Lanczos steps (rtol 0); P0 = P^-1 z
  {
    std::vector<double> t2(l, 0.0);
    GPM_TRY(mbcg_rank(pl, pc, s2, B + n, l, m, t2, X + n, bah.as<double>(), bbh.as<double>(),
                      itl, stl, P0 + n, s));
    for (int c = 0; c < l; ++c)
      if (stl[c] == 2) return fail(GP_ERR_BREAKDOWN, "CG breakdown on probe " + std::to_string(c));
  }
  if (!pc) GPM_CUDA(cudaMemcpyAsync(P0 + n, B + n, 8 * (size_t)n * l, cudaMemcpyDeviceToDevice, s));
  GPM_CUDA(cudaMemcpyAsync(P0, X, 8 * (size_t)n, cudaMemcpyDeviceToDevice, s));   // col 0: a
  // (3) K [a, P^-1 z] and l dK/dl [a, P^-1 z]
  GPM_TRY(apply_rank(pl, P0, KP, nc, s, 0));
  const bool has_dl = true;   // every (nu, form, d) has a lengthscale-gradient MVM (round 2)
  if (has_dl) GPM_TRY(apply_rank(pl, P0, DP, nc, s, 1));
  // (4) dots: col 0: a.Ka, a.dKa, a.a, r.a ; probe c: x_c.K p_c, x_c.dK p_c, x_c.p_c
  //     (x_c = A^-1 z_c from Lanczos, p_c = P^-1 z_c)
  std::vector<double> hk(nc), hd(nc, 0.0), hp(nc), hq(1);
  auto dotcols = [&](const double* Aa, const double* Bb, std::vector<double>& h) -> gp_status {
    k_dotp<<<dim3(LG, nc), LB, 0, s>>>(Aa, Bb, n, bpart.as<double>());
    k_sum<<<nc, LB, 0, s>>>(bpart.as<double>(), LG, dots);
    GPM_CUDA(cudaGetLastError());
    GPM_CUDA(cudaMemcpyAsync(h.data(), dots, 8 * (size_t)nc, cudaMemcpyDeviceToHost, s));
    GPM_CUDA(cudaStreamSynchronize(s));
    return GP_OK;
  };
  GPM_TRY(dotcols(X, KP, hk));
  if (has_dl) GPM_TRY(dotcols(X, DP, hd));
  GPM_TRY(dotcols(X, P0, hp));
  {
    k_dotp<<<dim3(LG, 1), LB, 0, s>>>(B, X, n, bpart.as<double>());
    k_sum<<<1, LB, 0, s>>>(bpart.as<double>(), LG, dots);
    GPM_CUDA(cudaMemcpyAsync(hq.data(), dots, 8, cudaMemcpyDeviceToHost, s));
    GPM_CUDA(cudaStreamSynchronize(s));
  }
  // (5) log det by Lanczos quadrature
  std::vector<double> ah((size_t)m * l), bh((size_t)m * l);
  GPM_CUDA(cudaMemcpyAsync(ah.data(), bah.ptr, 8 * (size_t)m * l, cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaMemcpyAsync(bh.data(), bbh.ptr, 8 * (size_t)m * l, cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  double acc = 0.0;
  int mmax = 0;
  for (int c = 0; c < l; ++c) {
    double q = 0.0;
    GPM_TRY(slq_column(ah.data(), bh.data(), l, c, itl[c], &q));
    acc += q;
    mmax = std::max(mmax, itl[c]);
  }
  double ldP = 0.0;
  if (pc) GPM_TRY(precond_logdet(*pc, s2, &ldP, s));
  const double N = (double)n;
  const double logdet = N / l * acc + ldP;
  // (6) assemble; Hutchinson: tr(A^-1 M) ~ 1/l sum_c x_c^T M p_c
  double trK = 0.0, trD = 0.0, trI = 0.0;
  for (int c = 1; c <= l; ++c) { trK += hk[c]; trD += hd[c]; trI += hp[c]; }
  trK /= l; trD /= l; trI /= l;
  const double os = std::sqrt(pl.os2), sg = std::sqrt(s2);
  out->quad = hq[0];
  out->logdet = logdet;
  out->logdet_precond = ldP;
  out->lml = -0.5 * hq[0] - 0.5 * logdet - 0.5 * N * std::log(2.0 * M_PI);
  out->grad[0] = (hk[0] - trK) / os;                       // 1/2 (2/s) (a'Ka - tr(A^-1 K))
  out->grad[1] = has_dl ? 0.5 * (hd[0] - trD) : NAN;
  out->grad[2] = sg * (hp[0] - trI);                        // 1/2 (2 sigma) (a'a - tr A^-1)
  out->cg_iters = it1[0];
  out->lanczos_iters = mmax;
  return GP_OK;
}

}  // namespace gpm

// ---------------------------------------------------------------------------
// gp_fit: Algorithm 1 with GradDescStep = one ADAM ascent step on
// theta = (log s, log c) (reading R13).
namespace gpm {

namespace {

// y - H beta for H = [1, x] (host)
std::vector<double> centre(const std::vector<double>& y, const std::vector<double>& x, int d,
                           const std::vector<double>& beta) {
  const size_t n = y.size();
  std::vector<double> r(n);
  for (size_t i = 0; i < n; ++i) {
    double m = beta[0];
    for (int k = 0; k < d; ++k) m += beta[1 + k] * x[i * d + k];
    r[i] = y[i] - m;
  }
  return r;
}

bool solve_small(std::vector<double> G, std::vector<double> g, int k, std::vector<double>& x) {
  for (int c = 0; c < k; ++c) {
    int piv = c;
    for (int r = c + 1; r < k; ++r)
      if (std::fabs(G[r * k + c]) > std::fabs(G[piv * k + c])) piv = r;
    if (G[piv * k + c] == 0.0) return false;
    if (piv != c) {
      for (int j = 0; j < k; ++j) std::swap(G[c * k + j], G[piv * k + j]);
      std::swap(g[c], g[piv]);
    }
    for (int r = c + 1; r < k; ++r) {
      const double f = G[r * k + c] / G[c * k + c];
      for (int j = c; j < k; ++j) G[r * k + j] -= f * G[c * k + j];
      g[r] -= f * g[c];
    }
  }
  x.assign(k, 0.0);
  for (int c = k - 1; c >= 0; --c) {
    double s = g[c];
    for (int j = c + 1; j < k; ++j) s -= G[c * k + j] * x[j];
    x[c] = s / G[c * k + c];
  }
  return true;
}

struct FitState {
  const double* x;
  int64_t n;
  int d;
  gp_kernel k0;
  double s, c, sigma;           // outputscale, lengthscale scale, noise sd
  double m[2] = {0, 0}, v[2] = {0, 0};
  int t = 0;
  Plan pl;
  bool built = false;
  Precond pc;
  bool has_pc = false;
};

gp_kernel cur_kernel(const FitState& F) {
  gp_kernel k = F.k0;
  k.outputscale = F.s;
  for (int j = 0; j < 3; ++j) k.lengthscale[j] = F.k0.lengthscale[j] * F.c;
  return k;
}

gp_status rebuild(FitState& F, int rank, cudaStream_t s) {
  if (F.has_pc) { precond_free(F.pc); F.pc = Precond(); F.has_pc = false; }
  if (F.built) { plan_free(F.pl); F.pl = Plan(); F.built = false; }
  GPM_TRY(plan_build(F.pl, F.x, F.n, F.d, cur_kernel(F), s));
  F.built = true;
  if (rank > 0) {
    GPM_TRY(precond_build(F.pc, F.pl, rank, s));
    F.has_pc = true;
  }
  return GP_OK;
}

}  // namespace

gp_status fit_alg1(const double* x, int64_t n, int d, const gp_kernel& k0, double sigma0,
                   const double* y, const double* G, const double* W, int nprobe,
                   const gp_fit_opts& o, gp_fit_result* out, cudaStream_t s) {
  FitState F;
  F.x = x; F.n = n; F.d = d; F.k0 = k0;
  F.s = k0.outputscale; F.c = 1.0; F.sigma = sigma0;
  struct Cleanup {
    FitState* f;
    ~Cleanup() {
      if (f->has_pc) precond_free(f->pc);
      if (f->built) plan_free(f->pl);
    }
  } cleanup{&F};
  // host copies: x (n x d) and y for OLS / centring
  std::vector<double> hx((size_t)n * d), hy((size_t)n);
  GPM_CUDA(cudaMemcpyAsync(hx.data(), x, 8 * hx.size(), cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaMemcpyAsync(hy.data(), y, 8 * hy.size(), cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  const int nh = 1 + d;
  std::vector<double> beta_ols;
  {
    std::vector<long double> G2(nh * nh, 0.0L), g2(nh, 0.0L);
    for (int64_t i = 0; i < n; ++i) {
      double h[4] = {1.0, 0, 0, 0};
      for (int k = 0; k < d; ++k) h[1 + k] = hx[(size_t)i * d + k];
      for (int a = 0; a < nh; ++a) {
        g2[a] += (long double)h[a] * hy[i];
        for (int b = 0; b < nh; ++b) G2[a * nh + b] += (long double)h[a] * h[b];
      }
    }
    std::vector<double> Gd(nh * nh), gd(nh);
    for (int a = 0; a < nh * nh; ++a) Gd[a] = (double)G2[a];
    for (int a = 0; a < nh; ++a) gd[a] = (double)g2[a];
    if (!solve_small(Gd, gd, nh, beta_ols))
      return fail(GP_ERR_INVALID_ARG, "OLS: H^T H is singular");
  }
  DevBuf byc, ba;
  GPM_TRY(byc.alloc(8 * (size_t)n));
  GPM_TRY(ba.alloc(8 * (size_t)n));
  GPM_TRY(rebuild(F, o.precond_rank, s));
  int steps = 0;
  double last_lml = 0.0, last_norm = 0.0;

  auto descent = [&](const std::vector<double>& yc_host, int cap) -> gp_status {
    GPM_CUDA(cudaMemcpyAsync(byc.ptr, yc_host.data(), 8 * (size_t)n, cudaMemcpyHostToDevice, s));
    int local = 0;
    while (true) {
      // GradDescStep: gradient of the LML at (s, c, sigma), ADAM ascent on (log s, log c)
      gp_lml_result r{};
      GPM_TRY(lml_eval(F.pl, F.has_pc ? &F.pc : nullptr, F.sigma * F.sigma, byc.as<double>(), G,
                       W, nprobe, o.lanczos_iters, o.cg_rtol, &r, s));
      if (!std::isfinite(r.grad[1]))
        return fail(GP_ERR_UNSUPPORTED, "gp_fit needs the lengthscale gradient of this kernel");
      last_lml = r.lml;
      const double g[2] = {r.grad[0] * F.s, r.grad[1]};
      ++F.t;
      double th[2] = {std::log(F.s), std::log(F.c)};
      for (int q = 0; q < 2; ++q) {
        F.m[q] = 0.9 * F.m[q] + 0.1 * g[q];
        F.v[q] = 0.999 * F.v[q] + 0.001 * g[q] * g[q];
        const double mh = F.m[q] / (1.0 - std::pow(0.9, F.t));
        const double vh = F.v[q] / (1.0 - std::pow(0.999, F.t));
        th[q] += o.lr * mh / (std::sqrt(vh) + 1e-8);
      }
      F.s = std::exp(th[0]);
      F.c = std::exp(th[1]);
      last_norm = std::sqrt(g[0] * g[0] + g[1] * g[1]) / (double)n;
      ++steps;
      ++local;
      // sigma update at the new (s, l): 1/N y^T (K(s/sigma_prev) + I)^-1 y
      //   = sigma_prev^2 / N  y^T (K(s) + sigma_prev^2 I)^-1 y
      GPM_TRY(rebuild(F, o.precond_rank, s));
      {
        std::vector<double> t2(1);
        double yy = 0.0;
        for (double v : yc_host) yy += v * v;
        t2[0] = o.cg_rtol * o.cg_rtol * yy;
        std::vector<double> hr(n);
        DevBuf rb;
        GPM_TRY(rb.alloc(8 * (size_t)n));
        GPM_TRY(permute_vec(F.pl, byc.as<double>(), rb.as<double>(), true, s));
        std::vector<int> it, st;
        const int capcg = (int)std::min<int64_t>(std::max<int64_t>(1000, 20 * n), 200000);
        GPM_TRY(mbcg_rank(F.pl, F.has_pc ? &F.pc : nullptr, F.sigma * F.sigma, rb.as<double>(), 1,
                          capcg, t2, ba.as<double>(), nullptr, nullptr, it, st, nullptr, s));
        if (st[0] != 1) return fail(GP_ERR_NOT_CONVERGED, "gp_fit: sigma-update CG failed");
        std::vector<double> ha(n), hrr(n);
        GPM_CUDA(cudaMemcpyAsync(ha.data(), ba.ptr, 8 * (size_t)n, cudaMemcpyDeviceToHost, s));
        GPM_CUDA(cudaMemcpyAsync(hrr.data(), rb.ptr, 8 * (size_t)n, cudaMemcpyDeviceToHost, s));
        GPM_CUDA(cudaStreamSynchronize(s));
        long double q = 0.0L;
        for (int64_t i = 0; i < n; ++i) q += (long double)hrr[i] * ha[i];
        F.sigma = std::sqrt(F.sigma * F.sigma * (double)q / (double)n);
      }
      if (last_norm <= o.grad_tol || local >= cap) return GP_OK;
    }
  };

  GPM_TRY(descent(centre(hy, hx, d, beta_ols), o.max_steps));
  std::vector<double> beta_avg(nh, 0.0), beta_old = beta_ols, beta_gls = beta_ols;
  int outer = 0;
  while (outer < o.max_outer) {
    // beta_GLS at the current parameters
    DevBuf al;
    GPM_TRY(al.alloc(8 * (size_t)n));
    double bb[4] = {0, 0, 0, 0};
    gp_cg_info info{};
    GPM_TRY(cg_solve(F.pl, F.sigma * F.sigma, y, GP_MEAN_AFFINE, nullptr, 0, o.cg_rtol,
                     (int)std::min<int64_t>(std::max<int64_t>(1000, 20 * n), 200000), al.as<double>(),
                     bb, &info, s, F.has_pc ? &F.pc : nullptr));
    for (int a = 0; a < nh; ++a) beta_gls[a] = bb[a];
    ++outer;
    for (int a = 0; a < nh; ++a)
      beta_avg[a] = (double)(outer - 1) / outer * beta_avg[a] + beta_gls[a] / outer;
    GPM_TRY(descent(centre(hy, hx, d, beta_avg), o.max_steps));
    double ch = 0.0;
    for (int a = 0; a < nh; ++a) ch += (beta_gls[a] - beta_old[a]) * (beta_gls[a] - beta_old[a]);
    beta_old = beta_gls;
    if (std::sqrt(ch) <= o.beta_tol) break;
  }
  out->kernel = cur_kernel(F);
  out->sigma = F.sigma;
  for (int a = 0; a < 4; ++a) out->beta[a] = a < nh ? beta_gls[a] : 0.0;
  out->steps = steps;
  out->outer = outer;
  out->lml = last_lml;
  out->grad_norm = last_norm;
  return GP_OK;
}

}  // namespace gpm
