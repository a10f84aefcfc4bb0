// solve.cu -- a9/a10: multi-RHS conjugate gradients on A = K + sigma^2 I and the GLS
// fixed-effects correction.
//   CG: P:155-174 [§1] ("the core computational step in each conjugate-gradient
//   iteration is the multiplication of K with a vector"), P:980-1034 [App A, Alg 2]
//   with s_P = identity (no preconditioner, reading R8) and a zero initial guess.
//   Per column j: alpha_j = r_j^T r_j / p_j^T A p_j, x += alpha p, r -= alpha A p,
//   beta_j = r'^T r' / r^T r, p = r' + beta p  (Alg 2 loop body).
//   Stop per column at ||r_j|| <= rtol ||b_j|| (reading R8: per-column relative 2-norm,
//   not Alg 2's aggregated ||R||^2 < tol); the TRUE residual b - A x is re-evaluated at
//   exit and CG restarts from it if recursion drift left it above rtol.
//   Breakdown p^T A p <= 0 (A not SPD, reading R4) is reported, never hidden.
//   GLS: beta = (H^T A^-1 H)^-1 H^T A^-1 y; alpha = A^-1 y - (A^-1 H) beta.
// All vectors live in x1-rank order so no permutation is applied inside the loop;
// every reduction is a fixed-order two-stage tree (deterministic, no atomics).
#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.h"

namespace gpm {

namespace {

constexpr int CG_BLOCK = 256;
constexpr int CG_GRID = 296;   // 2 x 148 SMs; reduction partials per column

__device__ __forceinline__ double block_sum(double v, double* sh) {
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
  return t;  // valid in thread 0
}

// q_c += sigma2 p_c ; partial[c][block] = sum p_c . q_c     (grid.y = column)
__global__ void k_pq(const double* __restrict__ P, double* __restrict__ Q, int64_t n,
                     double sigma2, double* __restrict__ part) {
  __shared__ double sh[32];
  const int c = blockIdx.y;
  const double* p = P + (size_t)c * n;
  double* q = Q + (size_t)c * n;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double pv = p[i];
    const double qv = fma(sigma2, pv, q[i]);
    q[i] = qv;
    acc = fma(pv, qv, acc);
  }
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) part[(size_t)c * gridDim.x + blockIdx.x] = t;
}

// alpha_c = rr_c / pq_c (status 0 only); breakdown detection
__global__ void k_alpha(const double* __restrict__ part, int nb, const double* __restrict__ rr,
                        double* __restrict__ alpha, int* __restrict__ status,
                        int* __restrict__ bd_iter, int iter) {
  __shared__ double sh[32];
  const int c = blockIdx.x;
  double acc = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) acc += part[(size_t)c * nb + b];
  const double pq = block_sum(acc, sh);
  if (threadIdx.x == 0) {
    double a = 0.0;
    if (status[c] == 0) {
      if (!(pq > 0.0) || !isfinite(pq)) {
        status[c] = 2;
        bd_iter[c] = iter;
      } else {
        a = rr[c] / pq;
      }
    }
    alpha[c] = a;
  }
}

// x += alpha p ; r -= alpha q ; partial rr
__global__ void k_update(double* __restrict__ X, double* __restrict__ R,
                         const double* __restrict__ P, const double* __restrict__ Q,
                         const double* __restrict__ alpha, int64_t n, double* __restrict__ part) {
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
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) part[(size_t)c * gridDim.x + blockIdx.x] = t;
}

// beta_c = rr_new / rr ; convergence test against tol2_c = (rtol ||b_c||)^2
__global__ void k_beta(const double* __restrict__ part, int nb, double* __restrict__ rr,
                       const double* __restrict__ tol2, double* __restrict__ beta,
                       int* __restrict__ status) {
  __shared__ double sh[32];
  const int c = blockIdx.x;
  double acc = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) acc += part[(size_t)c * nb + b];
  const double rn = block_sum(acc, sh);
  if (threadIdx.x == 0) {
    double bt = 0.0;
    if (status[c] == 0) {
      bt = rn / rr[c];
      rr[c] = rn;
      if (rn <= tol2[c]) status[c] = 1;
    }
    beta[c] = bt;
  }
}

// p = r + beta p   (active columns)
__global__ void k_pupd(double* __restrict__ P, const double* __restrict__ R,
                       const double* __restrict__ beta, const int* __restrict__ status,
                       int64_t n) {
  const int c = blockIdx.y;
  if (status[c] != 0) return;
  const double b = beta[c];
  double* p = P + (size_t)c * n;
  const double* r = R + (size_t)c * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = fma(b, p[i], r[i]);
}

// ---- fused CG iteration.  The apply's epilogue already returns
// q = K p + s2 p with per-block partials of p . q; every block of the two kernels below
// re-sums the partials it needs in a fixed order (no separate reduction launches, the
// results are identical in every block, hence deterministic).
__device__ __forceinline__ double sum_fixed(const double* __restrict__ part, int nb, double* sh) {
  double acc = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) acc += part[b];
  return block_sum(acc, sh);   // valid in thread 0
}

// alpha = r.r / p.q (old r.r from the previous iteration's partials); x += alpha p,
// r -= alpha q, partials of the new r.r.  Breakdown p.q <= 0 -> alpha = 0, status 2.
__global__ void k_cg_xr(double* __restrict__ X, double* __restrict__ R,
                        const double* __restrict__ P, const double* __restrict__ Q,
                        const double* __restrict__ part_pq, int nb_pq,
                        const double* __restrict__ rr_old, double* __restrict__ rr_new,
                        int* __restrict__ status, int* __restrict__ bd_iter, int it,
                        int64_t n) {
  __shared__ double sh[32];
  __shared__ double s_alpha;
  const int c = blockIdx.y;
  const double pq = sum_fixed(part_pq + (size_t)c * nb_pq, nb_pq, sh);
  const double ro = sum_fixed(rr_old + (size_t)c * gridDim.x, gridDim.x, sh);
  if (threadIdx.x == 0) {
    double a = 0.0;
    if (status[c] == 0) {
      if (!(pq > 0.0) || !isfinite(pq)) {
        if (blockIdx.x == 0) {
          status[c] = 2;
          bd_iter[c] = it;
        }
      } else {
        a = ro / pq;
      }
    }
    s_alpha = a;
  }
  __syncthreads();
  const double a = s_alpha;
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
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) rr_new[(size_t)c * gridDim.x + blockIdx.x] = t;
}

// beta = new r.r / old r.r; p = r + beta p (active columns); convergence at
// r.r <= tol2 (status 1, block 0); rr_out[c] = new r.r for the host
// pts != nullptr (d >= 2): columns c0 <= c < c1 are the next apply's one run of active columns;
// the new p also goes into the u field of its packed point records (32 B per point, column
// c - c0), so that apply needs no pack launch (apply_rank prepacked).
__global__ void k_cg_p(double* __restrict__ P, const double* __restrict__ R,
                       const double* __restrict__ rr_new, const double* __restrict__ rr_old,
                       const double* __restrict__ tol2, int* __restrict__ status,
                       double* __restrict__ rr_out, int64_t n, double* __restrict__ pts, int c0,
                       int c1) {
  __shared__ double sh[32];
  __shared__ double s_beta;
  __shared__ int s_act;
  const int c = blockIdx.y;
  const double rn = sum_fixed(rr_new + (size_t)c * gridDim.x, gridDim.x, sh);
  const double ro = sum_fixed(rr_old + (size_t)c * gridDim.x, gridDim.x, sh);
  if (threadIdx.x == 0) {
    const int st = status[c];
    s_act = st == 0;
    s_beta = st == 0 ? rn / ro : 0.0;
    if (blockIdx.x == 0 && st == 0) {
      rr_out[c] = rn;
      if (rn <= tol2[c]) status[c] = 1;
    }
  }
  __syncthreads();
  if (!s_act) return;
  const double b = s_beta;
  double* p = P + (size_t)c * n;
  const double* r = R + (size_t)c * n;
  double* pu = (pts && c >= c0 && c < c1) ? pts + (size_t)(c - c0) * n * 4 + 3 : nullptr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double pn = fma(b, p[i], r[i]);
    p[i] = pn;
    if (pu) pu[4 * i] = pn;
  }
}

// X columns back to user order: Xu[c][perm[r]] = X[c][r]
__global__ void k_cols_to_user(const int* __restrict__ perm, const double* __restrict__ X,
                               int64_t n, double* __restrict__ Xu) {
  const int c = blockIdx.y;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    Xu[(size_t)c * n + perm[r]] = X[(size_t)c * n + r];
}

// partial sums of squares of columns (grid.y = column)
__global__ void k_sumsq(const double* __restrict__ V, int64_t n, double* __restrict__ part) {
  __shared__ double sh[32];
  const int c = blockIdx.y;
  const double* v = V + (size_t)c * n;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    acc = fma(v[i], v[i], acc);
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) part[(size_t)c * gridDim.x + blockIdx.x] = t;
}

__global__ void k_finish_sum(const double* __restrict__ part, int nb, double* __restrict__ out) {
  __shared__ double sh[32];
  const int c = blockIdx.x;
  double acc = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) acc += part[(size_t)c * nb + b];
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) out[c] = t;
}

// R = B - (Q + sigma2 X)   (Q = K X)
__global__ void k_resid(const double* __restrict__ B, const double* __restrict__ Q,
                        const double* __restrict__ X, double sigma2, int64_t nk,
                        double* __restrict__ R) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nk;
       i += (int64_t)gridDim.x * blockDim.x)
    R[i] = B[i] - fma(sigma2, X[i], Q[i]);
}

// X += D
__global__ void k_add(double* __restrict__ X, const double* __restrict__ D, int64_t nk) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nk;
       i += (int64_t)gridDim.x * blockDim.x)
    X[i] += D[i];
}

// B columns in rank order: col 0 = y[perm], cols 1.. = H (affine from x_raw, or basis)
__global__ void k_build_rhs(const int* __restrict__ perm, const double* __restrict__ y,
                            const double* __restrict__ xraw, int d, const double* __restrict__ H,
                            int nh, int mean_kind, int64_t n, double* __restrict__ B) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int i = perm[r];
    B[r] = y[i];
    if (mean_kind == GP_MEAN_AFFINE) {
      B[n + r] = 1.0;
      for (int k = 0; k < d; ++k) B[(size_t)(2 + k) * n + r] = xraw[(size_t)i * d + k];
    } else if (mean_kind == GP_MEAN_BASIS) {
      for (int c = 0; c < nh; ++c) B[(size_t)(1 + c) * n + r] = H[(size_t)c * n + i];
    }
  }
}

// GLS partials: G[a][b] = sum_r H_a X_{1+b}, g[a] = sum_r H_a X_0   (grid.y = a*(nh+1)+b)
__global__ void k_gls_part(const double* __restrict__ B, const double* __restrict__ X, int nh,
                           int64_t n, double* __restrict__ part) {
  __shared__ double sh[32];
  const int ab = blockIdx.y;
  const int a = ab / (nh + 1), b = ab % (nh + 1);
  const double* h = B + (size_t)(1 + a) * n;
  const double* x = X + (size_t)(b == nh ? 0 : 1 + b) * n;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    acc = fma(h[i], x[i], acc);
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) part[(size_t)ab * gridDim.x + blockIdx.x] = t;
}

// alpha[perm[r]] = X0[r] - sum_a X_{1+a}[r] beta_a
__global__ void k_alpha_out(const int* __restrict__ perm, const double* __restrict__ X, int nh,
                            double b0, double b1, double b2, double b3, const double* __restrict__ bdev,
                            int64_t n, double* __restrict__ alpha) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    double v = X[r];
    for (int a = 0; a < nh; ++a) {
      const double ba = a == 0 ? b0 : a == 1 ? b1 : a == 2 ? b2 : a == 3 ? b3 : bdev[a];
      v -= X[(size_t)(1 + a) * n + r] * ba;
    }
    alpha[perm[r]] = v;
  }
}

// out[q] += h(z_q)^T beta  (affine: h = [1, z]; basis: Hz m x L col-major)
__global__ void k_mean_epi(const double* __restrict__ z, int64_t m, int d,
                           const double* __restrict__ Hz, int Lb, const double* __restrict__ bdev,
                           double* __restrict__ out) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m;
       q += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    if (Hz) {
      for (int a = 0; a < Lb; ++a) v += Hz[(size_t)a * m + q] * bdev[a];
    } else {
      v = bdev[0];
      for (int k = 0; k < d; ++k) v += z[(size_t)q * d + k] * bdev[1 + k];
    }
    out[q] += v;
  }
}

inline int g1(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)); }

// small dense SPD solve (Gaussian elimination with partial pivoting), host
bool small_solve(std::vector<double> G, std::vector<double> g, int k, std::vector<double>& x) {
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

}  // namespace

// Q[:, c] = K P[:, c] for the active columns: maximal runs of consecutive active columns
// go through one multi-RHS apply.
static gp_status apply_active(Plan& pl, const double* P, double* Q, const std::vector<char>& act,
                              int k, cudaStream_t s) {
  const size_t n = (size_t)pl.n;
  for (int c = 0; c < k;) {
    if (!act[c]) { ++c; continue; }
    int e = c;
    while (e < k && act[e]) ++e;
    GPM_TRY(apply_rank(pl, P + c * n, Q + c * n, e - c, s));
    c = e;
  }
  return GP_OK;
}

gp_status launch_affine_epilogue(const double* z, int64_t m, int d, const double* beta_host,
                                 const double* Hz, int Lb, double* out, cudaStream_t s,
                                 DevBuf& bd) {
  const int nb = Hz ? Lb : 1 + d;
  if (bd.bytes < sizeof(double) * nb) GPM_TRY(bd.alloc(sizeof(double) * 16));
  GPM_CUDA(cudaMemcpyAsync(bd.ptr, beta_host, sizeof(double) * nb, cudaMemcpyHostToDevice, s));
  k_mean_epi<<<g1(m), 256, 0, s>>>(z, m, d, Hz, Lb, bd.as<double>(), out);
  GPM_CUDA(cudaGetLastError());
  return GP_OK;   // the host beta is copied: the caller synchronises before returning
}

namespace {
__global__ void k_differs(const double* __restrict__ a, const double* __restrict__ b, int64_t m,
                          int* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    if (__double_as_longlong(a[i]) != __double_as_longlong(b[i])) *flag = 1;
}
}  // namespace

// 1 when the m doubles at a and b differ bitwise (synchronises s; flag: 4 device bytes)
gp_status device_differs(const double* a, const double* b, int64_t m, int* flag, cudaStream_t s,
                         bool* out) {
  GPM_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
  k_differs<<<g1(m), 256, 0, s>>>(a, b, m, flag);
  GPM_CUDA(cudaGetLastError());
  int h = 0;
  GPM_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  *out = h != 0;
  return GP_OK;
}

// The CG iterations of one 8-iteration block, enqueued on s: per iteration the apply with
// the fused epilogue (q = K p + s2 p and the p.q partials), k_cg_xr, k_cg_p.  Captured once
// per solve as a CUDA graph and replayed (when s is not itself being captured).
struct CgBufs {
  double *B, *X, *R, *P, *Q, *ppq, *prr, *tol2, *rr;
  int *status, *bd_iter;
  int k, nb_pq;
};
static gp_status cg_block(Plan& pl, const CgBufs& b, double sigma2, int it0, int iters,
                          const std::vector<char>& act, cudaStream_t s) {
  const int64_t n = pl.n;
  // d >= 2 with one run of at most LV_MAXB active columns: k_cg_p writes the new p straight
  // into the packed point records of the next apply (no pack launch after the block's first
  // iteration, which packs t and p itself)
  int nruns = 0, r0 = 0, r1 = 0;
  for (int c = 0; c < b.k;) {
    if (!act[c]) { ++c; continue; }
    int e = c;
    while (e < b.k && act[e]) ++e;
    if (nruns++ == 0) { r0 = c; r1 = e; }
    c = e;
  }
  const bool fuse_pack = pl.d >= 2 && nruns == 1 && r1 - r0 <= LV_MAXB && !getenv("GPM_CG_NOPACKFUSE");
  for (int j = 0; j < iters; ++j) {
    const int it = it0 + j;
    double* rr_new = b.prr + (size_t)(it & 1) * b.k * CG_GRID;
    double* rr_old = b.prr + (size_t)((it + 1) & 1) * b.k * CG_GRID;
    // the apply on the runs of active columns (converged ones keep alpha = 0)
    for (int c = 0; c < b.k;) {
      if (!act[c]) { ++c; continue; }
      int e = c;
      while (e < b.k && act[e]) ++e;
      GPM_TRY(apply_rank(pl, b.P + (size_t)c * n, b.Q + (size_t)c * n, e - c, s, 0, sigma2,
                         b.ppq + (size_t)c * b.nb_pq, fuse_pack && j > 0));
      c = e;
    }
    k_cg_xr<<<dim3(CG_GRID, b.k), CG_BLOCK, 0, s>>>(b.X, b.R, b.P, b.Q, b.ppq, b.nb_pq, rr_old,
                                                     rr_new, b.status, b.bd_iter, it, n);
    k_cg_p<<<dim3(CG_GRID, b.k), CG_BLOCK, 0, s>>>(b.P, b.R, rr_new, rr_old, b.tol2, b.status,
                                                    b.rr, n,
                                                    fuse_pack && j + 1 < iters ? pl.pts.as<double>() : nullptr,
                                                    r0, r1);
  }
  GPM_CUDA(cudaGetLastError());
  return GP_OK;
}

gp_status cg_solve(Plan& pl, double sigma2, const double* y, int mean_kind, const double* H,
                   int Lb, double rtol, int max_iter, double* alpha, double* beta,
                   gp_cg_info* info, cudaStream_t s, Precond* pc, double* beta_ols,
                   double* Xout) {
  const int64_t n = pl.n;
  const int nh = mean_kind == GP_MEAN_AFFINE ? 1 + pl.d : mean_kind == GP_MEAN_BASIS ? Lb : 0;
  const int k = 1 + nh;
  const size_t nk = (size_t)n * k;
  const int nb_pq = getenv("GPM_CG_UNFUSED") ? 0 : cg_nblk(pl);   // apply's CG-epilogue blocks (0: unfused)
  // scratch cached on the plan (grow-only): no per-call frees, no device-wide syncs
  const size_t nsc = 8 * (5 * nk + (size_t)std::max(nb_pq, 1) * k + 2 * (size_t)CG_GRID * k +
                          (size_t)CG_GRID * std::max(k, (nh + 1) * std::max(nh, 1)) + 2 * k + 64) +
                     4 * (2 * (size_t)k + 16);
  if (pl.cg_scratch.bytes < nsc) GPM_TRY(pl.cg_scratch.alloc(nsc));
  CgBufs b;
  b.k = k;
  b.nb_pq = nb_pq;
  b.B = pl.cg_scratch.as<double>();
  b.X = b.B + nk;
  b.R = b.X + nk;
  b.P = b.R + nk;
  b.Q = b.P + nk;
  b.ppq = b.Q + nk;
  b.prr = b.ppq + (size_t)std::max(nb_pq, 1) * k;
  double* part = b.prr + 2 * (size_t)CG_GRID * k;   // general reductions (k_sumsq, GLS)
  b.tol2 = part + (size_t)CG_GRID * std::max(k, (nh + 1) * std::max(nh, 1));
  b.rr = b.tol2 + k;
  double* bn2 = b.rr + k;
  b.status = reinterpret_cast<int*>(bn2 + k);
  b.bd_iter = b.status + k;
  double* B = b.B;
  double* X = b.X;
  double* R = b.R;
  double* Pm = b.P;
  double* Q = b.Q;

  k_build_rhs<<<g1(n), 256, 0, s>>>(pl.perm.as<int>(), y, pl.x_raw.as<double>(), pl.d, H, nh,
                                     mean_kind, n, B);
  GPM_CUDA(cudaMemsetAsync(X, 0, 8 * nk, s));
  GPM_CUDA(cudaMemcpyAsync(R, B, 8 * nk, cudaMemcpyDeviceToDevice, s));
  GPM_CUDA(cudaMemcpyAsync(Pm, B, 8 * nk, cudaMemcpyDeviceToDevice, s));
  // ||b_c||^2 partials, kept as the "previous r.r" of iteration 0 (rr parity 1)
  double* rr1 = b.prr + (size_t)k * CG_GRID;
  k_sumsq<<<dim3(CG_GRID, k), CG_BLOCK, 0, s>>>(B, n, rr1);
  k_finish_sum<<<k, CG_BLOCK, 0, s>>>(rr1, CG_GRID, bn2);
  GPM_CUDA(cudaGetLastError());
  std::vector<double> hb2(k), hrr(k), htol2(k);
  std::vector<int> hst(k), hbd(k);
  GPM_CUDA(cudaMemcpyAsync(hb2.data(), bn2, 8 * k, cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  for (int c = 0; c < k; ++c) {
    htol2[c] = rtol * rtol * hb2[c];
    hst[c] = hb2[c] == 0.0 ? 1 : 0;   // zero right-hand side: x = 0 is exact
  }
  GPM_CUDA(cudaMemcpyAsync(b.tol2, htol2.data(), 8 * k, cudaMemcpyHostToDevice, s));
  GPM_CUDA(cudaMemcpyAsync(b.rr, hb2.data(), 8 * k, cudaMemcpyHostToDevice, s));
  GPM_CUDA(cudaMemcpyAsync(b.status, hst.data(), 4 * k, cudaMemcpyHostToDevice, s));
  double* rr = b.rr;
  double* tol2 = b.tol2;
  double* al = part;   // unfused path scalars (alpha, beta) live in the reduction area
  double* be = part + k;
  int* status = b.status;
  int* bd_iter = b.bd_iter;

  const int check_every = 8;
  int it = 0, restarts = 0;
  gp_status result = GP_OK;
  std::vector<double> relres(k, 0.0);
  if (pc) {
    // preconditioned (Alg 2 with s_P = Woodbury): solve, then the true
    // residual; restart on it (solve A D = R, X += D) while the recursion drifted
    std::vector<double> t2(k);
    for (int c = 0; c < k; ++c) t2[c] = htol2[c];
    std::vector<int> iters, st;
    DevBuf bD;
    GPM_TRY(bD.alloc(8 * nk));
    const double* rhs = B;
    double* sol = X;
    while (true) {
      GPM_TRY(mbcg_rank(pl, pc, sigma2, rhs, k, std::max(1, max_iter - it), t2, sol, nullptr,
                        nullptr, iters, st, nullptr, s));
      int mx = 0;
      for (int c = 0; c < k; ++c) mx = std::max(mx, iters[c]);
      it += mx;
      if (sol != X) {   // X += D
        k_add<<<g1((int64_t)nk), 256, 0, s>>>(X, sol, (int64_t)nk);
        GPM_CUDA(cudaGetLastError());
      }
      bool broke = false;
      for (int c = 0; c < k; ++c) { hst[c] = st[c]; broke |= st[c] == 2; }
      GPM_TRY(apply_rank(pl, X, Q, k, s));
      k_resid<<<g1((int64_t)nk), 256, 0, s>>>(B, Q, X, sigma2, (int64_t)nk, R);
      k_sumsq<<<dim3(CG_GRID, k), CG_BLOCK, 0, s>>>(R, n, part);
      k_finish_sum<<<k, CG_BLOCK, 0, s>>>(part, CG_GRID, rr);
      GPM_CUDA(cudaGetLastError());
      GPM_CUDA(cudaMemcpyAsync(hrr.data(), rr, 8 * k, cudaMemcpyDeviceToHost, s));
      GPM_CUDA(cudaStreamSynchronize(s));
      bool need = false;
      int bad = -1;
      for (int c = 0; c < k; ++c) {
        relres[c] = hb2[c] > 0 ? std::sqrt(hrr[c] / hb2[c]) : 0.0;
        if (relres[c] > rtol || st[c] == 2) { need = true; if (bad < 0) bad = c; }
      }
      if (broke) {
        result = fail(GP_ERR_BREAKDOWN, "preconditioned CG breakdown (p^T A p <= 0) in column " +
                                            std::to_string(bad) +
                                            ": K + sigma^2 I is not positive definite");
        break;
      }
      if (!need) break;
      if (it >= max_iter || restarts >= 5) {
        result = fail(GP_ERR_NOT_CONVERGED, "preconditioned CG did not reach rtol in " +
                                                std::to_string(it) + " iterations (column " +
                                                std::to_string(bad) + ", relres " +
                                                std::to_string(relres[bad]) + ")");
        break;
      }
      ++restarts;
      rhs = R;                  // solve A D = R_true, same absolute levels
      sol = bD.as<double>();
      GPM_CUDA(cudaMemcpyAsync(Pm, R, 8 * nk, cudaMemcpyDeviceToDevice, s));   // (keep R)
      rhs = Pm;
    }
  }
  // unpreconditioned: the fused iteration in 8-iteration blocks, one CUDA graph replayed
  // per block when possible (a stream that is itself capturing runs the block directly)
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  GPM_CUDA(cudaStreamIsCapturing(s, &cap));
  const bool fused = nb_pq > 0;
  const bool use_graph = fused && cap == cudaStreamCaptureStatusNone && !getenv("GPM_CG_NOGRAPH");
  cudaGraphExec_t gexec = nullptr;
  std::vector<char> gmask;   // the active-column mask gexec was captured with
  cudaStream_t cs = nullptr;
  struct GraphGuard {
    cudaGraphExec_t* g;
    cudaStream_t* s;
    ~GraphGuard() {
      if (*g) cudaGraphExecDestroy(*g);
      if (*s) cudaStreamDestroy(*s);
    }
  } gguard{&gexec, &cs};
  while (!pc) {
    bool any = false;
    for (int c = 0; c < k; ++c) any |= hst[c] == 0;
    while (any && it < max_iter) {
      std::vector<char> act(k, 0);
      for (int c = 0; c < k; ++c) act[c] = hst[c] == 0;
      if (fused) {
        if (use_graph && it > 0) {   // the first block ran directly (it sizes the scratch)
          if (gexec && gmask != act) {   // another active set: capture again
            GPM_CUDA(cudaGraphExecDestroy(gexec));
            gexec = nullptr;
          }
          if (!gexec) {   // capture the 8-iteration block (the iteration parity repeats)
            if (!cs) GPM_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
            cudaGraph_t g = nullptr;
            GPM_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
            gp_status bst = cg_block(pl, b, sigma2, 0, check_every, act, cs);
            cudaError_t ce = cudaStreamEndCapture(cs, &g);
            if (bst != GP_OK) {
              if (g) cudaGraphDestroy(g);
              return bst;
            }
            GPM_CUDA(ce);
            cudaError_t ie = cudaGraphInstantiate(&gexec, g, 0);
            cudaGraphDestroy(g);
            GPM_CUDA(ie);
            gmask = act;
          }
          GPM_CUDA(cudaGraphLaunch(gexec, s));
        } else {
          GPM_TRY(cg_block(pl, b, sigma2, 0, check_every, act, s));
        }
        it += check_every;   // breakdown iterations are recorded relative to the block
      } else {
        for (int step = 0; step < check_every && it < max_iter; ++step, ++it) {
          GPM_TRY(apply_active(pl, Pm, Q, act, k, s));
          k_pq<<<dim3(CG_GRID, k), CG_BLOCK, 0, s>>>(Pm, Q, n, sigma2, part);
          k_alpha<<<k, CG_BLOCK, 0, s>>>(part, CG_GRID, rr, al, status, bd_iter, it);
          k_update<<<dim3(CG_GRID, k), CG_BLOCK, 0, s>>>(X, R, Pm, Q, al, n, part);
          k_beta<<<k, CG_BLOCK, 0, s>>>(part, CG_GRID, rr, tol2, be, status);
          k_pupd<<<dim3(CG_GRID, k), CG_BLOCK, 0, s>>>(Pm, R, be, status, n);
        }
        GPM_CUDA(cudaGetLastError());
      }
      GPM_CUDA(cudaMemcpyAsync(hst.data(), status, 4 * k, cudaMemcpyDeviceToHost, s));
      GPM_CUDA(cudaStreamSynchronize(s));
      any = false;
      for (int c = 0; c < k; ++c) any |= hst[c] == 0;
      for (int c = 0; c < k; ++c)
        if (hst[c] == 2) any = false;   // stop on breakdown
    }
    // true residual R = B - (K X + sigma2 X)
    GPM_TRY(apply_rank(pl, X, Q, k, s));
    k_resid<<<g1((int64_t)nk), 256, 0, s>>>(B, Q, X, sigma2, (int64_t)nk, R);
    k_sumsq<<<dim3(CG_GRID, k), CG_BLOCK, 0, s>>>(R, n, part);
    k_finish_sum<<<k, CG_BLOCK, 0, s>>>(part, CG_GRID, rr);
    GPM_CUDA(cudaGetLastError());
    GPM_CUDA(cudaMemcpyAsync(hrr.data(), rr, 8 * k, cudaMemcpyDeviceToHost, s));
    GPM_CUDA(cudaMemcpyAsync(hbd.data(), bd_iter, 4 * k, cudaMemcpyDeviceToHost, s));
    GPM_CUDA(cudaStreamSynchronize(s));
    bool need_restart = false, broke = false;
    int bad_col = -1;
    for (int c = 0; c < k; ++c) {
      relres[c] = hb2[c] > 0 ? std::sqrt(hrr[c] / hb2[c]) : 0.0;
      if (hst[c] == 2) { broke = true; if (bad_col < 0) bad_col = c; }
      else if (relres[c] > rtol) { need_restart = true; if (bad_col < 0) bad_col = c; }
    }
    if (broke) {
      result = fail(GP_ERR_BREAKDOWN, "CG breakdown (p^T A p <= 0) in column " +
                                          std::to_string(bad_col) + " near iteration " +
                                          std::to_string(fused ? it - check_every + hbd[bad_col]
                                                               : hbd[bad_col]) +
                                          ": K + sigma^2 I is not positive definite");
      break;
    }
    if (!need_restart) break;
    if (it >= max_iter || restarts >= 5) {
      result = fail(GP_ERR_NOT_CONVERGED, "CG did not reach rtol in " + std::to_string(it) +
                                              " iterations (column " + std::to_string(bad_col) +
                                              ", relres " + std::to_string(relres[bad_col]) + ")");
      break;
    }
    // residual replacement: restart from the true residual (its r.r becomes the "previous
    // r.r" of the next block: rr parity 1)
    ++restarts;
    for (int c = 0; c < k; ++c) hst[c] = relres[c] > rtol ? 0 : 1;
    GPM_CUDA(cudaMemcpyAsync(Pm, R, 8 * nk, cudaMemcpyDeviceToDevice, s));
    GPM_CUDA(cudaMemcpyAsync(status, hst.data(), 4 * k, cudaMemcpyHostToDevice, s));
    if (fused) {
      k_sumsq<<<dim3(CG_GRID, k), CG_BLOCK, 0, s>>>(R, n, rr1);
      GPM_CUDA(cudaGetLastError());
    }
  }
  if (info) {
    info->iters = it;
    info->restarts = restarts;
    info->relres_max = 0.0;
    info->failed_column = -1;
    for (int c = 0; c < k; ++c) info->relres_max = std::max(info->relres_max, relres[c]);
    if (result != GP_OK) {
      for (int c = 0; c < k; ++c)
        if (hst[c] == 2 || relres[c] > rtol) { info->failed_column = c; break; }
    }
  }
  if (result == GP_ERR_BREAKDOWN) return result;

  // GLS (a10) and alpha in user order; OLS (P:829 [Alg 1, first line]) on request
  std::vector<double> hbeta(std::max(nh, 1), 0.0);
  auto normal_eqs = [&](const double* Xs, std::vector<double>& sol) -> gp_status {
    // G[a][b] = sum_r H_a Xs_{1+b}, g[a] = sum_r H_a Xs_0; solve G beta = g
    const int nab = nh * (nh + 1);
    k_gls_part<<<dim3(CG_GRID, nab), CG_BLOCK, 0, s>>>(B, Xs, nh, n, part);
    k_finish_sum<<<nab, CG_BLOCK, 0, s>>>(part, CG_GRID, Q);   // Q: free after the solve
    std::vector<double> hg(nab);
    GPM_CUDA(cudaMemcpyAsync(hg.data(), Q, 8 * nab, cudaMemcpyDeviceToHost, s));
    GPM_CUDA(cudaStreamSynchronize(s));
    std::vector<double> G(nh * nh), g(nh);
    for (int a = 0; a < nh; ++a) {
      for (int b2 = 0; b2 < nh; ++b2) G[a * nh + b2] = hg[a * (nh + 1) + b2];
      g[a] = hg[a * (nh + 1) + nh];
    }
    for (int a = 0; a < nh; ++a)   // symmetrise (symmetric in exact arithmetic)
      for (int b2 = a + 1; b2 < nh; ++b2) {
        const double m = 0.5 * (G[a * nh + b2] + G[b2 * nh + a]);
        G[a * nh + b2] = G[b2 * nh + a] = m;
      }
    if (!small_solve(G, g, nh, sol))
      return fail(GP_ERR_INVALID_ARG, "normal equations are singular (rank-deficient H)");
    return GP_OK;
  };
  if (nh > 0) {
    std::vector<double> sol;
    GPM_TRY(normal_eqs(X, sol));   // H^T A^-1 H beta = H^T A^-1 y
    hbeta = sol;
    if (beta) for (int a = 0; a < nh; ++a) beta[a] = sol[a];
    if (beta_ols) {               // H^T H beta = H^T y (the columns of B)
      GPM_TRY(normal_eqs(B, sol));
      for (int a = 0; a < nh; ++a) beta_ols[a] = sol[a];
    }
  }
  if (Xout) {
    k_cols_to_user<<<dim3(g1(n), k), 256, 0, s>>>(pl.perm.as<int>(), X, n, Xout);
    GPM_CUDA(cudaGetLastError());
  }
  double* bbd = part;   // beta on the device (after the reductions above consumed part)
  GPM_CUDA(cudaMemcpyAsync(bbd, hbeta.data(), 8 * std::max(nh, 1), cudaMemcpyHostToDevice, s));
  auto bv = [&](int a) { return a < nh ? hbeta[a] : 0.0; };
  k_alpha_out<<<g1(n), 256, 0, s>>>(pl.perm.as<int>(), X, nh, bv(0), bv(1), bv(2), bv(3), bbd, n,
                                     alpha);
  GPM_CUDA(cudaGetLastError());
  GPM_CUDA(cudaStreamSynchronize(s));
  return result;
}

}  // namespace gpm
