// internal.h -- plan layout in HBM and internal entry points of libgpmatern.so.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/gpmatern.h"

struct cublasContext;   // cuBLAS handle (lml.cu only includes cublas_v2.h)

namespace gpm {

// Error plumbing ------------------------------------------------------------
void set_error(const std::string& msg);
gp_status fail(gp_status st, const std::string& msg);
#define GPM_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (call);                                                             \
    if (_e != cudaSuccess)                                                               \
      return ::gpm::fail(GP_ERR_CUDA, std::string(#call " failed: ") + cudaGetErrorString(_e) + \
                                          " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)
#define GPM_TRY(expr)                 \
  do {                                \
    gp_status _s = (expr);            \
    if (_s != GP_OK) return _s;       \
  } while (0)

// Device buffer owned by a plan.
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  gp_free_fn fr = nullptr;   // allocator hook that owns ptr (gp_set_allocator), else cudaFree
  void* fctx = nullptr;
  gp_status alloc(size_t b);
  void release();
  template <class T> T* as() const { return static_cast<T*>(ptr); }
  // owning and move-only: scratch buffers are freed on every exit path
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), bytes(o.bytes), fr(o.fr), fctx(o.fctx) {
    o.ptr = nullptr; o.bytes = 0; o.fr = nullptr; o.fctx = nullptr;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      ptr = o.ptr; bytes = o.bytes; fr = o.fr; fctx = o.fctx;
      o.ptr = nullptr; o.bytes = 0; o.fr = nullptr; o.fctx = nullptr;
    }
    return *this;
  }
  ~DevBuf() { release(); }
};

// d = 1 tile-aggregate record (both scan directions), P <= 2.
struct D1Agg {
  double D, E;      // span and e^{-span}
  double F[3];      // forward moments of the segment's sources, referenced at its last point
  double B[3];      // backward moments, referenced one point before its first point
};

// Level-pass tile aggregate (one direction): up to 4 channels x 5 moments (L1, d = 3,
// nu = 9/2 or the nu = 7/2 gradient) or 2 channels x 9 mixed moments (product, d = 2,
// nu <= 5/2) in the 184 B record LvAgg; the wider product states (2 x 16 / 2 x 25 mixed
// moments: product nu = 7/2, 9/2 and the nu = 5/2, 7/2 gradients) use LvRec<32> / LvRec<50>.
template <int W>
struct LvRec {
  double D, E;
  double M[W];
  int flag;
  int pad;
};
using LvAgg = LvRec<20>;
// record width of an algebra with NS state doubles
template <int NS>
using LvRecFor = LvRec<(NS > 20 ? NS : 20)>;
// bytes of the widest record a plan's level passes can use (product d = 2: 2 (p+2)^2
// for the gradient, capped at the widest supported state)
inline size_t level_rec_bytes(int d, int form_product, int P) {
  int ns = 20;
  if (d == 3 && 4 * (P + 2) > ns) ns = 4 * (P + 2);   // gradient of nu = 9/2: 4 x 6 moments
  if (d == 2 && form_product) {
    const int w = 2 * (P + 2) * (P + 2);
    ns = w > 50 ? 50 : (w > 20 ? w : 20);
  }
  return sizeof(double) * (2 + (size_t)ns) + 2 * sizeof(int);
}

// The stored structure of P:191 [§1], P:338 [§2.1], P:539 [§2.2.3], in HBM.
//   "rank" = x1-rank: position of a point in the stable (t1, index) order.
struct Plan {
  int64_t n = 0;
  int d = 0, two_nu = 1, P = 0, form = 0;
  gp_kernel kern{};                 // kernel as given to gp_setup
  double os2 = 1.0;                 // outputscale^2
  double ell[3] = {1, 1, 1};
  double scale[3] = {1, 1, 1};      // sqrt(2 nu) / l_k
  int L = 0;                        // levels: ceil(log2 n)
  int64_t n_src = 0;                // sources are user indices < n_src (== n except unions)
  int64_t tgt_off = 0;              // targets are user indices >= tgt_off (0 except unions)

  DevBuf x_raw;                     // n x d row-major copy of the input (for unions / H)
  DevBuf perm;                      // int32 [n]: perm[r] = user index of rank r
  DevBuf t;                         // double [d][n]: t_k in rank order (SoA)
  DevBuf ord2;                      // int32 [L][n]: d>=2, level l order (ranks), t2-sorted per node
  DevBuf ord3;                      // int32 [L(L+1)/2][n]: d=3, positions into ord2[l1], t3-sorted
  // scratch (apply)
  DevBuf u;                         // double [n]: input in rank order
  DevBuf acc;                       // double [n]: level-pass accumulator (rank order)
  DevBuf w;                         // double [n]: rank-order output scratch
  DevBuf aggs;                      // tile aggregates
  DevBuf bar;                       // grid barrier words (d = 1 cooperative kernel)
  DevBuf stage_in, stage_out;       // gp_kmvm_host staging
  DevBuf dbg;                       // d=1 phase timestamps (env GPM_D1_TIMING)
  DevBuf d1e;                       // d=1: e^{-gap} per rank (plan data, padded with 1)
  DevBuf d1ends;                    // d=1: chunk-end coordinates of the chunking (plan data)
  DevBuf cg_scratch;                // gp_cg_solve scratch, cached (grow-only)
  DevBuf pts;                       // d>=2: packed (t1, t2, t3, u) per rank, rebuilt per apply
  DevBuf hpbuf;                     // d>=2: staged structure of the carried passes (setup)
  DevBuf hpdesc;                    // d>=2: per carried pass (offset, n_act, lseg, tiles)
  int hp_npass = 0, hp_maxtiles = 0, hp_items = 0;   // carried passes, max tiles, total tiles
  // d >= 2: side stream for the carried-pass aggregates (independent of the low levels)
  cudaStream_t s2 = nullptr, s3 = nullptr;   // s3: d = 3 mid levels (k_mid3) beside the low levels
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_join3 = nullptr;
  int low_unused = 0;       // trailing low-kernel part slots the last apply left unwritten
  int part_zero_cols = 0;   // columns of `part` whose never-written tail slots are zeroed
  // gp_kmvm_host pipelining: copy streams and per-slot events (in, compute, out) x 3
  cudaStream_t hs_in = nullptr, hs_out = nullptr;
  cudaEvent_t hev[9] = {};
  std::vector<char> hp_tail;        // carried pass has an inactive tail (slot must be zeroed)
  DevBuf part;                      // d>=2: per-pass contribution slots [nrhs][nparts][n]
  int near_lb2 = 4, near_lb3 = 7, near_lb3m = 5;   // near-field block log2 sizes (tuned)
  // d = 1 launch geometry
  int d1_grid = 0, d1_path = 1, d1_force = 0, d1_shape = -1;   // d1_shape: requested (-1 auto)
  int d1_shape_used = 0;            // the shape of the single-chunk kernel in use
  int d1_pdl = 1;                   // programmatic dependent launch for back-to-back applies
  int d1_prefetch = 1;    // d = 1 user order: L2 prefetch of v before the gathers (option 3)
  int64_t d1_chunk = 0;
  int64_t struct_bytes = 0;
  int shard = 0, nshards = 1;       // gp_kmvm_partial: this call's share of a sharded apply
  int launches_per_apply = 0;
};

// lml.cu -- pivoted-Cholesky preconditioner P = L L^T + sigma^2 I
struct Precond {
  Plan* pl = nullptr;
  int k = 0;
  int64_t n = 0;
  DevBuf L;                    // n x k column-major, rank order
  DevBuf Cinv, W, Y;           // (I + L^T L / s2)^-1 (k x k) for the cached s2; scratch
  DevBuf Wp;                   // L^T R row-block partials (k_wlt), summed in order by k_wred
  std::vector<int> piv;        // pivot ranks
  std::vector<double> G;       // L^T L (k x k, host)
  double s2 = -1.0, logdetC = 0.0;
  ::cublasContext* h = nullptr;
};
gp_status precond_build(Precond& pc, Plan& pl, int k, cudaStream_t s);
// zr_part (optional): when the streaming path runs, per-CTA partials of z_c . r_c are
// written there ([nb][*zr_nblk]) and *zr_nblk is set; otherwise *zr_nblk = 0
gp_status precond_apply(Precond& pc, double s2, const double* R, int nb, double* Z,
                        cudaStream_t s, double* zr_part = nullptr, int* zr_nblk = nullptr);
inline int precond_zr_blocks(int64_t n) { return (int)((n + 255) / 256); }
gp_status precond_sample(Precond& pc, double s2, const double* G, const double* W, int nb,
                         double* Z, cudaStream_t s);
gp_status precond_logdet(Precond& pc, double s2, double* out, cudaStream_t s);
void precond_free(Precond& pc);
gp_status mbcg_rank(Plan& pl, Precond* pc, double s2, const double* B, int nb, int max_iter,
                    const std::vector<double>& tol2, double* X, double* ahist, double* bhist,
                    std::vector<int>& iters, std::vector<int>& status, double* P0,
                    cudaStream_t s);
gp_status slq_column(const double* ah, const double* bh, int nb, int c, int m, double* q);
gp_status lml_eval(Plan& pl, Precond* pc, double s2, const double* r_user, const double* G_user,
                   const double* W, int nprobe, int m, double cg_rtol, gp_lml_result* out,
                   cudaStream_t s);

gp_status fit_alg1(const double* x, int64_t n, int d, const gp_kernel& k0, double sigma0,
                   const double* y, const double* G, const double* W, int nprobe,
                   const gp_fit_opts& o, gp_fit_result* out, cudaStream_t s);

// setup.cu
void set_allocator(gp_alloc_fn a, gp_free_fn f, void* ctx);
gp_status plan_build(Plan& pl, const double* x_dev, int64_t n, int d, const gp_kernel& k,
                     cudaStream_t s);
void plan_free(Plan& pl);

// apply.cu
// Rank-space apply: out_rank = K u_rank (no nugget).  u_rank, out_rank: n doubles.
// kind 0: K; kind 1: dK/dlog(l) (lengthscale gradient, L1 / d = 1 only).
// CG epilogue (solve.cu): with cg_part != nullptr the apply returns
// out = K u + cg_s2 u and writes per-block partial sums of u . out to
// cg_part[c * cg_nblk(pl) + block] (fixed-order reductions: deterministic).
// prepacked (d >= 2, nrhs <= LV_MAXB): the packed point records pl.pts already hold u_rank in
// their u field (the CG driver's k_cg_p writes p there): the pack launch is skipped.
gp_status apply_rank(Plan& pl, const double* u_rank, double* out_rank, int nrhs, cudaStream_t s,
                     int kind = 0, double cg_s2 = 0.0, double* cg_part = nullptr,
                     bool prepacked = false);
constexpr int LV_MAXB = 8;   // right-hand sides per level-pass batch (apply.cu)
int cg_nblk(const Plan& pl);
// User-order apply with gather/scatter: out = K v restricted to targets (unions).
// Columns: v stride n_src, out stride n - tgt_off.
gp_status apply_user(Plan& pl, const double* v, double* out, int nrhs, cudaStream_t s,
                     int kind = 0);
gp_status apply_prepare(Plan& pl);   // launch geometry + scratch
gp_status permute_vec(Plan& pl, const double* src, double* dst, bool to_rank, cudaStream_t s);
int64_t apply_model_bytes(const Plan& pl);
// apply_level.cu: tile range [r0, r1) and carried-pass item range [r2, r3) of a shard
void shard_ranges(int64_t n, int d, int shard, int nshards, int64_t* r);

// solve.cu
gp_status cg_solve(Plan& pl, double sigma2, const double* y, int mean_kind, const double* H,
                   int Lb, double rtol, int max_iter, double* alpha, double* beta,
                   gp_cg_info* info, cudaStream_t s, Precond* pc = nullptr,
                   double* beta_ols = nullptr, double* Xout = nullptr);
gp_status launch_affine_epilogue(const double* z, int64_t m, int d, const double* beta_host,
                                 const double* Hz, int Lb, double* out, cudaStream_t s,
                                 DevBuf& beta_dev);
gp_status device_differs(const double* a, const double* b, int64_t m, int* flag, cudaStream_t s,
                         bool* out);

}  // namespace gpm

struct gp_cross_s;
struct gp_plan_s {
  gpm::Plan pl;
  // gp_predict cache: the union structure x U z of the last query set, reused while the
  // same z pointer and m come back with bitwise-equal contents (checked on the device)
  gp_cross_s* pred_cross = nullptr;
  const double* pred_z = nullptr;
  int64_t pred_m = 0;
  gpm::DevBuf pred_zcopy, pred_flag, pred_beta;
  int live_preconds = 0;     // preconditioners built on this plan (they point into pl)
  bool destroy_pending = false;   // gp_destroy called while preconditioners were alive
};
struct gp_precond_s {
  gpm::Precond pc;
  gp_plan owner = nullptr;
};
struct gp_cross_s {
  gpm::Plan pl;        // structure of the union x U z
  int64_t n = 0, m = 0;
};
