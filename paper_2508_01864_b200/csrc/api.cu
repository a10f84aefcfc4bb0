// api.cu -- the C ABI of include/gpmatern.h.  Argument validation, error strings and
// plan lifetime; every compute step is a kernel in setup.cu / apply*.cu / solve.cu.
#include <cmath>
#include <cstring>
#include <new>
#include <string>
#include <vector>
#include <algorithm>

#include "internal.h"

namespace gpm {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }
gp_status fail(gp_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

static gp_status check_kernel(const gp_kernel* k, int d) {
  if (!k) return fail(GP_ERR_INVALID_ARG, "kernel is NULL");
  if (d < 1 || d > 3) return fail(GP_ERR_INVALID_ARG, "d must be 1, 2 or 3");
  if (!(k->outputscale > 0) || !std::isfinite(k->outputscale))
    return fail(GP_ERR_INVALID_ARG, "outputscale must be > 0");
  for (int j = 0; j < d; ++j)
    if (!(k->lengthscale[j] > 0) || !std::isfinite(k->lengthscale[j]))
      return fail(GP_ERR_INVALID_ARG, "lengthscale[" + std::to_string(j) + "] must be > 0");
  static const char* kSupp =
      "supported: two_nu in {1,3,5,7,9}, d in {1,2,3}, forms L1 and PRODUCT";
  if (k->two_nu != 1 && k->two_nu != 3 && k->two_nu != 5 && k->two_nu != 7 && k->two_nu != 9)
    return fail(GP_ERR_UNSUPPORTED,
                "two_nu=" + std::to_string(k->two_nu) + " unsupported; " + kSupp);
  if (k->form != GP_FORM_L1 && k->form != GP_FORM_PRODUCT)
    return fail(GP_ERR_INVALID_ARG, "form must be GP_FORM_L1 or GP_FORM_PRODUCT");
  return GP_OK;
}

static gp_status check_device() {
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    (void)cudaGetLastError();
    return fail(GP_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e) +
                                 " (there is no CPU fallback)");
  }
  return GP_OK;
}

}  // namespace gpm

using namespace gpm;

extern "C" {

const char* gp_last_error(void) { return g_err.c_str(); }

gp_status gp_set_allocator(gp_alloc_fn alloc, gp_free_fn free_fn, void* ctx) {
  if ((alloc == nullptr) != (free_fn == nullptr))
    return fail(GP_ERR_INVALID_ARG, "alloc and free must both be set or both be NULL");
  set_allocator(alloc, free_fn, ctx);
  return GP_OK;
}
const char* gp_version(void) { return "gpmatern 0.1 sm_100a"; }

gp_status gp_setup(const double* x, int64_t n, int d, const gp_kernel* k, void* stream,
                   gp_plan* out) {
  if (!out) return fail(GP_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (!x) return fail(GP_ERR_INVALID_ARG, "x is NULL");
  if (n < 1) return fail(GP_ERR_INVALID_ARG, "n must be >= 1");
  if (n >= (int64_t(1) << 30)) return fail(GP_ERR_UNSUPPORTED, "n >= 2^30 not supported");
  GPM_TRY(check_kernel(k, d));
  GPM_TRY(check_device());
  gp_plan p = new (std::nothrow) gp_plan_s();
  if (!p) return fail(GP_ERR_OOM, "host allocation failed");
  gp_status st = plan_build(p->pl, x, n, d, *k, static_cast<cudaStream_t>(stream));
  if (st != GP_OK) {
    plan_free(p->pl);
    delete p;
    return st;
  }
  *out = p;
  return GP_OK;
}

gp_status gp_kmvm(gp_plan p, const double* v, int nrhs, double* out, void* stream) {
  if (!p || !v || !out) return fail(GP_ERR_INVALID_ARG, "NULL argument");
  if (nrhs < 1) return fail(GP_ERR_INVALID_ARG, "nrhs must be >= 1");
  if (v == out) return fail(GP_ERR_INVALID_ARG, "out must not alias v");
  return apply_user(p->pl, v, out, nrhs, static_cast<cudaStream_t>(stream));
}

gp_status gp_kmvm_rank(gp_plan p, const double* v, int nrhs, double* out, void* stream) {
  if (!p || !v || !out) return fail(GP_ERR_INVALID_ARG, "NULL argument");
  if (nrhs < 1) return fail(GP_ERR_INVALID_ARG, "nrhs must be >= 1");
  if (v == out) return fail(GP_ERR_INVALID_ARG, "out must not alias v");
  return apply_rank(p->pl, v, out, nrhs, static_cast<cudaStream_t>(stream));
}

gp_status gp_kmvm_dlengthscale(gp_plan p, const double* v, int nrhs, double* out, int v_order,
                               void* stream) {
  if (!p || !v || !out) return fail(GP_ERR_INVALID_ARG, "NULL argument");
  if (nrhs < 1) return fail(GP_ERR_INVALID_ARG, "nrhs must be >= 1");
  if (v == out) return fail(GP_ERR_INVALID_ARG, "out must not alias v");
  if (v_order != 0 && v_order != 1) return fail(GP_ERR_INVALID_ARG, "v_order must be 0 or 1");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return v_order == 0 ? apply_user(p->pl, v, out, nrhs, s, 1)
                      : apply_rank(p->pl, v, out, nrhs, s, 1);
}

gp_status gp_permute(gp_plan p, const double* src, int nrhs, double* dst, int to_rank,
                     void* stream) {
  if (!p || !src || !dst) return fail(GP_ERR_INVALID_ARG, "NULL argument");
  if (nrhs < 1) return fail(GP_ERR_INVALID_ARG, "nrhs must be >= 1");
  if (src == dst) return fail(GP_ERR_INVALID_ARG, "dst must not alias src");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int c = 0; c < nrhs; ++c)
    GPM_TRY(permute_vec(p->pl, src + (size_t)c * p->pl.n, dst + (size_t)c * p->pl.n,
                        to_rank != 0, s));
  return GP_OK;
}

static bool is_pinned(const void* ptr) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// nrhs > 1 with pinned host buffers: columns flow through three device stage slots with
// the host->device copy of column c+1, the apply of column c and the device->host copy of
// column c-1 in flight together (copy streams + events; the apply stays on `s`).
static gp_status kmvm_host_pipelined(gp_plan p, const double* v, int nrhs, double* out,
                                     cudaStream_t s) {
  Plan& pl = p->pl;
  const size_t n = (size_t)pl.n;
  const size_t col = sizeof(double) * n;
  if (!pl.hs_in) {
    GPM_CUDA(cudaStreamCreateWithFlags(&pl.hs_in, cudaStreamNonBlocking));
    GPM_CUDA(cudaStreamCreateWithFlags(&pl.hs_out, cudaStreamNonBlocking));
    for (int b = 0; b < 9; ++b) GPM_CUDA(cudaEventCreateWithFlags(&pl.hev[b], cudaEventDisableTiming));
  }
  if (pl.stage_in.bytes < 3 * col) GPM_TRY(pl.stage_in.alloc(3 * col));
  if (pl.stage_out.bytes < 3 * col) GPM_TRY(pl.stage_out.alloc(3 * col));
  cudaEvent_t* e_in = pl.hev;
  cudaEvent_t* e_cmp = pl.hev + 3;
  cudaEvent_t* e_out = pl.hev + 6;
  GPM_CUDA(cudaEventRecord(e_cmp[0], s));   // copies start after prior work on s
  GPM_CUDA(cudaStreamWaitEvent(pl.hs_in, e_cmp[0], 0));
  for (int c = 0; c < nrhs; ++c) {
    const int b = c % 3;
    double* vb = pl.stage_in.as<double>() + b * n;
    double* ob = pl.stage_out.as<double>() + b * n;
    if (c >= 3) GPM_CUDA(cudaStreamWaitEvent(pl.hs_in, e_cmp[b], 0));   // slot consumed
    GPM_CUDA(cudaMemcpyAsync(vb, v + c * n, col, cudaMemcpyHostToDevice, pl.hs_in));
    GPM_CUDA(cudaEventRecord(e_in[b], pl.hs_in));
    GPM_CUDA(cudaStreamWaitEvent(s, e_in[b], 0));
    if (c >= 3) GPM_CUDA(cudaStreamWaitEvent(s, e_out[b], 0));          // slot drained
    GPM_TRY(apply_user(pl, vb, ob, 1, s));
    GPM_CUDA(cudaEventRecord(e_cmp[b], s));
    GPM_CUDA(cudaStreamWaitEvent(pl.hs_out, e_cmp[b], 0));
    GPM_CUDA(cudaMemcpyAsync(out + c * n, ob, col, cudaMemcpyDeviceToHost, pl.hs_out));
    GPM_CUDA(cudaEventRecord(e_out[b], pl.hs_out));
  }
  GPM_CUDA(cudaStreamSynchronize(pl.hs_out));
  GPM_CUDA(cudaStreamSynchronize(s));
  return GP_OK;
}

gp_status gp_kmvm_partial(gp_plan p, const double* v_rank, int nrhs, double* out_rank, int shard,
                          int nshards, void* stream) {
  if (!p || !v_rank || !out_rank) return fail(GP_ERR_INVALID_ARG, "NULL argument");
  if (nrhs < 1) return fail(GP_ERR_INVALID_ARG, "nrhs must be >= 1");
  if (nshards < 1 || shard < 0 || shard >= nshards)
    return fail(GP_ERR_INVALID_ARG, "need 0 <= shard < nshards");
  Plan& pl = p->pl;
  if (pl.d < 2)
    return fail(GP_ERR_UNSUPPORTED,
                "gp_kmvm_partial: d >= 2 only (the d = 1 apply is one launch; shard d = 1 by columns)");
  pl.shard = shard;
  pl.nshards = nshards;
  gp_status st = apply_rank(pl, v_rank, out_rank, nrhs, static_cast<cudaStream_t>(stream));
  pl.shard = 0;
  pl.nshards = 1;
  return st;
}

gp_status gp_shard_ranges(int64_t n, int d, int shard, int nshards, int64_t* ranges) {
  if (!ranges) return fail(GP_ERR_INVALID_ARG, "NULL argument");
  if (n < 1 || d < 2 || d > 3 || nshards < 1 || shard < 0 || shard >= nshards)
    return fail(GP_ERR_INVALID_ARG, "need n >= 1, d in {2, 3}, 0 <= shard < nshards");
  shard_ranges(n, d, shard, nshards, ranges);
  return GP_OK;
}

gp_status gp_kmvm_host(gp_plan p, const double* v, int nrhs, double* out, void* stream) {
  if (!p || !v || !out) return fail(GP_ERR_INVALID_ARG, "NULL argument");
  if (nrhs < 1) return fail(GP_ERR_INVALID_ARG, "nrhs must be >= 1");
  Plan& pl = p->pl;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (nrhs > 1 && is_pinned(v) && is_pinned(out)) return kmvm_host_pipelined(p, v, nrhs, out, s);
  const size_t bytes = sizeof(double) * pl.n * nrhs;
  if (pl.stage_in.bytes < bytes) GPM_TRY(pl.stage_in.alloc(bytes));
  if (pl.stage_out.bytes < bytes) GPM_TRY(pl.stage_out.alloc(bytes));
  GPM_CUDA(cudaMemcpyAsync(pl.stage_in.ptr, v, bytes, cudaMemcpyHostToDevice, s));
  GPM_TRY(gp_kmvm(p, pl.stage_in.as<double>(), nrhs, pl.stage_out.as<double>(), stream));
  GPM_CUDA(cudaMemcpyAsync(out, pl.stage_out.ptr, bytes, cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  return GP_OK;
}

gp_status gp_kzx_setup(gp_plan p, const double* z, int64_t m, void* stream, gp_cross* out) {
  if (!out) return fail(GP_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (!p || !z) return fail(GP_ERR_INVALID_ARG, "NULL argument");
  if (m < 1) return fail(GP_ERR_INVALID_ARG, "m must be >= 1");
  Plan& pl = p->pl;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t nu = pl.n + m;
  if (nu >= (int64_t(1) << 30)) return fail(GP_ERR_UNSUPPORTED, "n + m >= 2^30 not supported");
  DevBuf xu;
  GPM_TRY(xu.alloc(sizeof(double) * nu * pl.d));
  GPM_CUDA(cudaMemcpyAsync(xu.ptr, pl.x_raw.ptr, sizeof(double) * pl.n * pl.d,
                           cudaMemcpyDeviceToDevice, s));
  GPM_CUDA(cudaMemcpyAsync(xu.as<double>() + pl.n * pl.d, z, sizeof(double) * m * pl.d,
                           cudaMemcpyDeviceToDevice, s));
  gp_cross c = new (std::nothrow) gp_cross_s();
  if (!c) return fail(GP_ERR_OOM, "host allocation failed");
  gp_status st = plan_build(c->pl, xu.as<double>(), nu, pl.d, pl.kern, s);
  xu.release();
  if (st != GP_OK) {
    plan_free(c->pl);
    delete c;
    return st == GP_ERR_NONFINITE ? fail(st, std::string("query points: ") + gp_last_error())
                                  : st;
  }
  c->pl.n_src = pl.n;     // sources: the data points
  c->pl.tgt_off = pl.n;   // targets: the queries
  c->n = pl.n;
  c->m = m;
  *out = c;
  return GP_OK;
}

gp_status gp_kzx(gp_cross c, const double* v, int nrhs, double* out, void* stream) {
  if (!c || !v || !out) return fail(GP_ERR_INVALID_ARG, "NULL argument");
  if (nrhs < 1) return fail(GP_ERR_INVALID_ARG, "nrhs must be >= 1");
  return apply_user(c->pl, v, out, nrhs, static_cast<cudaStream_t>(stream));
}

void gp_kzx_destroy(gp_cross c) {
  if (!c) return;
  plan_free(c->pl);
  delete c;
}

gp_status gp_cg_solve(gp_plan p, double sigma2, const double* y, int mean_kind,
                      const double* H, int L, double rtol, int max_iter, double* alpha,
                      double* beta, gp_cg_info* info, void* stream) {
  return gp_cg_solve_pc(p, nullptr, sigma2, y, mean_kind, H, L, rtol, max_iter, alpha, beta,
                        info, stream);
}

gp_status gp_cg_solve_pc(gp_plan p, gp_precond pc, double sigma2, const double* y, int mean_kind,
                         const double* H, int L, double rtol, int max_iter, double* alpha,
                         double* beta, gp_cg_info* info, void* stream) {
  return gp_cg_solve_ex(p, pc, sigma2, y, mean_kind, H, L, rtol, max_iter, alpha, beta, nullptr,
                        nullptr, info, stream);
}

gp_status gp_cg_solve_ex(gp_plan p, gp_precond pc, double sigma2, const double* y, int mean_kind,
                         const double* H, int L, double rtol, int max_iter, double* alpha,
                         double* beta, double* beta_ols, double* X, gp_cg_info* info,
                         void* stream) {
  if (!p || !y || !alpha) return fail(GP_ERR_INVALID_ARG, "NULL argument");
  if (pc && pc->owner != p) return fail(GP_ERR_INVALID_ARG, "preconditioner built on another plan");
  if (!(sigma2 > 0) || !std::isfinite(sigma2)) return fail(GP_ERR_INVALID_ARG, "sigma2 must be > 0");
  if (!(rtol > 0)) return fail(GP_ERR_INVALID_ARG, "rtol must be > 0");
  if (max_iter < 1) return fail(GP_ERR_INVALID_ARG, "max_iter must be >= 1");
  if (mean_kind != GP_MEAN_NONE && mean_kind != GP_MEAN_AFFINE && mean_kind != GP_MEAN_BASIS)
    return fail(GP_ERR_INVALID_ARG, "unknown mean_kind");
  if (mean_kind == GP_MEAN_BASIS && (!H || L < 1 || L > 16))
    return fail(GP_ERR_INVALID_ARG, "BASIS mean needs H and 1 <= L <= 16");
  return cg_solve(p->pl, sigma2, y, mean_kind, H, L, rtol, max_iter, alpha, beta, info,
                  static_cast<cudaStream_t>(stream), pc ? &pc->pc : nullptr, beta_ols, X);
}

// ---- §8(f) f3: preconditioner, Algorithm 2, likelihood
gp_status gp_precond_create(gp_plan p, int rank, void* stream, gp_precond* out) {
  if (!p || !out) return fail(GP_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  if (rank < 1 || rank > 1024 || rank > p->pl.n)
    return fail(GP_ERR_INVALID_ARG, "rank must be in [1, min(n, 1024)]");
  gp_precond c = new (std::nothrow) gp_precond_s();
  if (!c) return fail(GP_ERR_OOM, "host allocation failed");
  c->owner = p;
  gp_status st = precond_build(c->pc, p->pl, rank, static_cast<cudaStream_t>(stream));
  if (st != GP_OK) {
    precond_free(c->pc);
    delete c;
    return st;
  }
  ++p->live_preconds;
  *out = c;
  return GP_OK;
}

gp_status gp_precond_factor(gp_precond pc, int64_t* pivots, double* L, void* stream) {
  if (!pc) return fail(GP_ERR_INVALID_ARG, "NULL argument");
  Plan& pl = pc->owner->pl;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (pivots) {
    std::vector<int> perm(pl.n);
    GPM_CUDA(cudaMemcpy(perm.data(), pl.perm.ptr, 4 * (size_t)pl.n, cudaMemcpyDeviceToHost));
    for (int i = 0; i < pc->pc.k; ++i) pivots[i] = perm[pc->pc.piv[i]];
  }
  if (L)
    for (int c = 0; c < pc->pc.k; ++c)
      GPM_TRY(permute_vec(pl, pc->pc.L.as<double>() + (size_t)c * pl.n, L + (size_t)c * pl.n,
                          false, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  return GP_OK;
}

gp_status gp_precond_solve(gp_precond pc, double sigma2, const double* r, int nb, double* z,
                           void* stream) {
  if (!pc || !r || !z) return fail(GP_ERR_INVALID_ARG, "NULL argument");
  if (r == z) return fail(GP_ERR_INVALID_ARG, "z must not alias r");
  if (nb < 1) return fail(GP_ERR_INVALID_ARG, "nb must be >= 1");
  if (!(sigma2 > 0) || !std::isfinite(sigma2)) return fail(GP_ERR_INVALID_ARG, "sigma2 must be > 0");
  Plan& pl = pc->owner->pl;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t n = (size_t)pl.n;
  DevBuf a, b;
  GPM_TRY(a.alloc(8 * n * nb));
  GPM_TRY(b.alloc(8 * n * nb));
  for (int c = 0; c < nb; ++c) GPM_TRY(permute_vec(pl, r + c * n, a.as<double>() + c * n, true, s));
  GPM_TRY(precond_apply(pc->pc, sigma2, a.as<double>(), nb, b.as<double>(), s));
  for (int c = 0; c < nb; ++c) GPM_TRY(permute_vec(pl, b.as<double>() + c * n, z + c * n, false, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  return GP_OK;
}

gp_status gp_precond_logdet(gp_precond pc, double sigma2, double* logdet, void* stream) {
  if (!pc || !logdet) return fail(GP_ERR_INVALID_ARG, "NULL argument");
  if (!(sigma2 > 0) || !std::isfinite(sigma2)) return fail(GP_ERR_INVALID_ARG, "sigma2 must be > 0");
  return precond_logdet(pc->pc, sigma2, logdet, static_cast<cudaStream_t>(stream));
}

void gp_precond_destroy(gp_precond pc) {
  if (!pc) return;
  gp_plan owner = pc->owner;
  precond_free(pc->pc);
  delete pc;
  // a plan whose gp_destroy came first is freed with its last preconditioner
  if (owner && --owner->live_preconds == 0 && owner->destroy_pending) {
    owner->destroy_pending = false;
    gp_destroy(owner);
  }
}

gp_status gp_mbcg(gp_plan p, gp_precond pc, double sigma2, const double* B, int nb, int max_iter,
                  double rtol, double* X, double* alpha_hist, double* beta_hist, int* iters_done,
                  void* stream) {
  if (!p || !B || !X) return fail(GP_ERR_INVALID_ARG, "NULL argument");
  if (pc && pc->owner != p) return fail(GP_ERR_INVALID_ARG, "preconditioner built on another plan");
  if (nb < 1 || max_iter < 1) return fail(GP_ERR_INVALID_ARG, "nb and max_iter must be >= 1");
  if (!(rtol >= 0)) return fail(GP_ERR_INVALID_ARG, "rtol must be >= 0");
  if (!(sigma2 > 0) || !std::isfinite(sigma2)) return fail(GP_ERR_INVALID_ARG, "sigma2 must be > 0");
  if (B == X) return fail(GP_ERR_INVALID_ARG, "X must not alias B");
  Plan& pl = p->pl;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t n = (size_t)pl.n;
  DevBuf rb, xb, ah, bh;
  GPM_TRY(rb.alloc(8 * n * nb));
  GPM_TRY(xb.alloc(8 * n * nb));
  GPM_TRY(ah.alloc(8 * (size_t)max_iter * nb));
  GPM_TRY(bh.alloc(8 * (size_t)max_iter * nb));
  for (int c = 0; c < nb; ++c) GPM_TRY(permute_vec(pl, B + c * n, rb.as<double>() + c * n, true, s));
  // tolerance levels from ||b_c||^2
  std::vector<double> bn(nb), t2(nb);
  {
    std::vector<double> hb(n);
    for (int c = 0; c < nb; ++c) {
      GPM_CUDA(cudaMemcpyAsync(hb.data(), rb.as<double>() + c * n, 8 * n, cudaMemcpyDeviceToHost, s));
      GPM_CUDA(cudaStreamSynchronize(s));
      long double acc = 0.0L;
      for (size_t i = 0; i < n; ++i) acc += (long double)hb[i] * hb[i];
      t2[c] = rtol * rtol * (double)acc;
    }
  }
  std::vector<int> it, st;
  GPM_CUDA(cudaMemsetAsync(ah.ptr, 0, 8 * (size_t)max_iter * nb, s));
  GPM_CUDA(cudaMemsetAsync(bh.ptr, 0, 8 * (size_t)max_iter * nb, s));
  GPM_TRY(mbcg_rank(pl, pc ? &pc->pc : nullptr, sigma2, rb.as<double>(), nb, max_iter, t2,
                    xb.as<double>(), ah.as<double>(), bh.as<double>(), it, st, nullptr, s));
  for (int c = 0; c < nb; ++c) GPM_TRY(permute_vec(pl, xb.as<double>() + c * n, X + c * n, false, s));
  if (alpha_hist)
    GPM_CUDA(cudaMemcpyAsync(alpha_hist, ah.ptr, 8 * (size_t)max_iter * nb, cudaMemcpyDeviceToHost, s));
  if (beta_hist)
    GPM_CUDA(cudaMemcpyAsync(beta_hist, bh.ptr, 8 * (size_t)max_iter * nb, cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  if (iters_done) for (int c = 0; c < nb; ++c) iters_done[c] = it[c];
  for (int c = 0; c < nb; ++c)
    if (st[c] == 2) return fail(GP_ERR_BREAKDOWN, "CG breakdown (p^T A p <= 0) in column " + std::to_string(c));
  return GP_OK;
}

gp_status gp_fit(const double* x, int64_t n, int d, const gp_kernel* k0, double sigma0,
                 const double* y, const double* G, const double* W, int nprobe,
                 const gp_fit_opts* opts, gp_fit_result* out, void* stream) {
  if (!x || !k0 || !y || !G || !out) return fail(GP_ERR_INVALID_ARG, "NULL argument");
  if (n < 2) return fail(GP_ERR_INVALID_ARG, "n must be >= 2");
  if (n >= (int64_t(1) << 30)) return fail(GP_ERR_UNSUPPORTED, "n >= 2^30 not supported");
  GPM_TRY(check_kernel(k0, d));
  GPM_TRY(check_device());
  if (!(sigma0 > 0) || !std::isfinite(sigma0)) return fail(GP_ERR_INVALID_ARG, "sigma0 must be > 0");
  if (nprobe < 1) return fail(GP_ERR_INVALID_ARG, "nprobe must be >= 1");
  gp_fit_opts o{};
  if (opts) o = *opts;
  if (o.lr == 0) o.lr = 0.05;
  if (o.max_steps == 0) o.max_steps = 50;
  if (o.max_outer == 0) o.max_outer = 3;
  if (o.grad_tol == 0) o.grad_tol = 1e-4;
  if (o.beta_tol == 0) o.beta_tol = 1e-3;
  if (o.lanczos_iters == 0) o.lanczos_iters = 25;
  if (o.cg_rtol == 0) o.cg_rtol = 1e-8;
  if (!(o.lr > 0) || o.max_steps < 1 || o.max_outer < 0 || o.lanczos_iters < 1 ||
      !(o.cg_rtol > 0) || o.precond_rank < 0 || o.precond_rank > 1024 || o.precond_rank > n)
    return fail(GP_ERR_INVALID_ARG, "invalid gp_fit_opts");
  if (o.precond_rank > 0 && !W) return fail(GP_ERR_INVALID_ARG, "W required with precond_rank > 0");
  return fit_alg1(x, n, d, *k0, sigma0, y, G, W, nprobe, o, out, static_cast<cudaStream_t>(stream));
}

gp_status gp_lml(gp_plan p, gp_precond pc, double sigma2, const double* r, const double* G,
                 const double* W, int nprobe, int lanczos_iters, double cg_rtol,
                 gp_lml_result* out, void* stream) {
  if (!p || !r || !G || !out) return fail(GP_ERR_INVALID_ARG, "NULL argument");
  if (pc && pc->owner != p) return fail(GP_ERR_INVALID_ARG, "preconditioner built on another plan");
  if (pc && !W) return fail(GP_ERR_INVALID_ARG, "W (rank x nprobe normals) required with a preconditioner");
  if (nprobe < 1 || lanczos_iters < 1) return fail(GP_ERR_INVALID_ARG, "nprobe and lanczos_iters must be >= 1");
  if (!(cg_rtol > 0)) return fail(GP_ERR_INVALID_ARG, "cg_rtol must be > 0");
  if (!(sigma2 > 0) || !std::isfinite(sigma2)) return fail(GP_ERR_INVALID_ARG, "sigma2 must be > 0");
  return lml_eval(p->pl, pc ? &pc->pc : nullptr, sigma2, r, G, W, nprobe, lanczos_iters, cg_rtol,
                  out, static_cast<cudaStream_t>(stream));
}

gp_status gp_predict(gp_plan p, const double* z, int64_t m, const double* alpha,
                     const double* beta, const double* Hz, int L, double* out, void* stream) {
  if (!p || !z || !alpha || !out) return fail(GP_ERR_INVALID_ARG, "NULL argument");
  if (Hz && (L < 1 || !beta)) return fail(GP_ERR_INVALID_ARG, "basis mean needs beta and L >= 1");
  if (m < 1) return fail(GP_ERR_INVALID_ARG, "m must be >= 1");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t zn = (size_t)m * p->pl.d;
  bool reuse = false;
  if (p->pred_cross && p->pred_z == z && p->pred_m == m) {   // same query set?
    bool differs = true;
    GPM_TRY(device_differs(z, p->pred_zcopy.as<double>(), (int64_t)zn, p->pred_flag.as<int>(), s,
                           &differs));
    reuse = !differs;
  }
  if (!reuse) {
    if (p->pred_cross) {
      gp_kzx_destroy(p->pred_cross);
      p->pred_cross = nullptr;
    }
    gp_cross c = nullptr;
    GPM_TRY(gp_kzx_setup(p, z, m, stream, &c));
    p->pred_cross = c;
    p->pred_z = z;
    p->pred_m = m;
    if (p->pred_zcopy.bytes < sizeof(double) * zn) GPM_TRY(p->pred_zcopy.alloc(sizeof(double) * zn));
    if (!p->pred_flag.bytes) GPM_TRY(p->pred_flag.alloc(16));
    GPM_CUDA(cudaMemcpyAsync(p->pred_zcopy.ptr, z, sizeof(double) * zn, cudaMemcpyDeviceToDevice, s));
  }
  GPM_TRY(gp_kzx(p->pred_cross, alpha, 1, out, stream));
  if (beta) GPM_TRY(launch_affine_epilogue(z, m, p->pl.d, beta, Hz, L, out, s, p->pred_beta));
  GPM_CUDA(cudaStreamSynchronize(s));
  return GP_OK;
}

gp_status gp_plan_query(gp_plan p, int what, int64_t* value) {
  if (!p || !value) return fail(GP_ERR_INVALID_ARG, "NULL argument");
  const Plan& pl = p->pl;
  switch (what) {
    case 0: *value = pl.n; break;
    case 1: *value = pl.d; break;
    case 2: *value = pl.L; break;
    case 3: *value = pl.struct_bytes; break;
    case 4: *value = pl.launches_per_apply; break;
    case 5: *value = apply_model_bytes(pl); break;
    case 6: *value = pl.d == 1 ? pl.d1_path : 0; break;
    case 7: *value = pl.d == 1 ? pl.d1_shape_used : -1; break;
    default: {
      // debug (GPM_D1_TIMING, d = 1 single-chunk path, last launch): what = 100 + slot:
      // mean over warps of stamp[slot] - stamp[0] (SM cycles); 200 + slot: the max
      if (what < 100 || what >= 216 || (what >= 116 && what < 200))
        return fail(GP_ERR_INVALID_ARG, "unknown query");
      if (!pl.dbg.bytes) return fail(GP_ERR_INVALID_ARG, "GPM_D1_TIMING not enabled");
      std::vector<unsigned long long> h(pl.dbg.bytes / 8);
      if (cudaMemcpy(h.data(), pl.dbg.ptr, pl.dbg.bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
        return fail(GP_ERR_CUDA, "dbg copy failed");
      const int slot = what % 100;
      // per-warp cycle stamps [cta][32 warps][16] (SM clock64): slot minus the same
      // warp's slot 0; warps that never wrote slot 0 are unused
      unsigned long long mx = 0;
      double acc = 0;
      int cntw = 0;
      for (int b = 0; b < pl.d1_grid * 32; ++b) {
        if (!h[b * 16] || !h[b * 16 + slot]) continue;
        const unsigned long long dt = h[b * 16 + slot] > h[b * 16] ? h[b * 16 + slot] - h[b * 16] : 0;
        acc += (double)dt;
        mx = std::max(mx, dt);
        ++cntw;
      }
      if (!cntw) cntw = 1;
      *value = what >= 200 ? (int64_t)mx : (int64_t)(acc / cntw);
      return GP_OK;
    }
  }
  return GP_OK;
}

gp_status gp_plan_set_option(gp_plan p, int option, int64_t value) {
  if (!p) return fail(GP_ERR_INVALID_ARG, "NULL plan");
  if (option == 0) {
    if (value < 0 || value > 3 || value == 2)
      return fail(GP_ERR_INVALID_ARG, "bad value for option 0 (0 auto, 1 single-chunk, 3 reduce-then-scan)");
    p->pl.d1_force = (int)value;
  } else if (option == 1) {
    if (value < 0 || value > 2) return fail(GP_ERR_INVALID_ARG, "bad value for option 1 (shapes 0..2)");
    p->pl.d1_shape = (int)value;
  } else if (option == 2) {
    p->pl.d1_pdl = value != 0;
  } else if (option == 3) {
    p->pl.d1_prefetch = value != 0;
  } else {
    return fail(GP_ERR_INVALID_ARG, "unknown option");
  }
  if (p->pl.d != 1) return GP_OK;
  return apply_prepare(p->pl);
}

void gp_destroy(gp_plan p) {
  if (!p) return;
  if (p->live_preconds > 0) {   // preconditioners point into the plan: defer
    p->destroy_pending = true;
    return;
  }
  if (p->pred_cross) gp_kzx_destroy(p->pred_cross);
  p->pred_zcopy.release();
  p->pred_flag.release();
  p->pred_beta.release();
  plan_free(p->pl);
  delete p;
}

}  // extern "C"
