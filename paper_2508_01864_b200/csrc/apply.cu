// apply.cu -- orchestration of one K.v (or K_zx.v) apply on a stored plan:
//   d = 1 : one cooperative launch (apply_d1.cu) with the gather / scatter fused in;
//   d >= 2: gather u[r] = v[perm[r]] -> level passes (apply_level.cu) into acc ->
//           epilogue out[perm[r]] = s^2 (u[r] + acc[r])  (self term + scale, a7).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "internal.h"

namespace gpm {

gp_status d1_prepare(Plan& pl);
gp_status d1_launch(Plan& pl, const double* v, double* out, int nrhs, bool user_order,
                    cudaStream_t s, int kind, double cg_s2 = 0.0, double* cg_part = nullptr);
gp_status level_passes(Plan& pl, int nrhs, cudaStream_t s, int* launches, int kind, int phase);
int level_phases(const Plan& pl, int kind);
gp_status level_pack(Plan& pl, const double* v, int nrhs, bool user_order, cudaStream_t s);
size_t level_pt_bytes();
int level_nparts(const Plan& pl);
int level_nab(const Plan& pl);
gp_status level_setup(Plan& pl, cudaStream_t s);
int64_t level_tiles(int64_t n);

namespace {

__global__ void k_gather(const int* __restrict__ perm, const double* __restrict__ v, int64_t n,
                         int64_t n_src, double* __restrict__ u) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int i = __ldg(perm + r);
    u[r] = i < n_src ? __ldg(v + i) : 0.0;
  }
}

// out[perm[r] - tgt_off] = os2 (self u[r] + acc[r]) for targets; perm == nullptr: rank order.
// u is read from the packed point records (stride 4 doubles, u at offset 3); self = k(0)
// (1 for K, 0 for the lengthscale gradient).
// accumulate: out += (the second run of a two-run apply, level_phases).
// CG epilogue (rank order only, cg_part != nullptr): out = K u + cg_s2 u and the block's
// partial sum of u . out -> cg_part[(col0 + blockIdx.y) * gridDim.x + blockIdx.x]
__global__ void k_epilogue(const int* __restrict__ perm, const double* __restrict__ pts,
                           const double* __restrict__ acc, const double* __restrict__ part,
                           int nparts, int64_t pstride, int64_t n, int64_t tgt_off, double os2, double self,
                           double* __restrict__ out, int64_t ostride, double cg_s2,
                           double* __restrict__ cg_part, int col0, int accumulate) {
  __shared__ double red[32];
  pts += blockIdx.y * 4 * n;
  acc += blockIdx.y * n;
  part += blockIdx.y * pstride;
  out += blockIdx.y * ostride;
  double pq = 0.0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    double a = acc[r];
    for (int p = 0; p < nparts; ++p) a += part[(int64_t)p * n + r];   // fixed order
    const double u = pts[4 * r + 3];
    double val = os2 * fma(self, u, a);
    if (perm) {
      const int i = __ldg(perm + r);
      if (i >= tgt_off) out[i - tgt_off] = accumulate ? out[i - tgt_off] + val : val;
    } else {
      if (cg_part) {
        val = fma(cg_s2, u, val);
        pq = fma(u, val, pq);
      }
      out[r] = accumulate ? out[r] + val : val;
    }
  }
  if (cg_part) {   // fixed-order block reduction
    for (int off = 16; off > 0; off >>= 1) pq += __shfl_down_sync(0xffffffffu, pq, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = pq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      cg_part[(size_t)(col0 + blockIdx.y) * gridDim.x + blockIdx.x] = t;
    }
  }
}

__global__ void k_scatter_user(const int* __restrict__ perm, const double* __restrict__ src,
                               int64_t n, double* __restrict__ dst) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    dst[__ldg(perm + r)] = src[r];
}

inline int egrid(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8));
}

}  // namespace

static gp_status level_buffers(Plan& pl, int nrhs);

gp_status apply_prepare(Plan& pl) {
  const int64_t n = pl.n;
  if (pl.d == 1) {
    GPM_TRY(d1_prepare(pl));
    pl.launches_per_apply = 1;
  } else {
    if (const char* e = getenv("GPM_NEAR_LB")) {   // tuning knob: "lb2,lb3,lb3m"
      int a = pl.near_lb2, b = pl.near_lb3, c = pl.near_lb3m;
      if (sscanf(e, "%d,%d,%d", &a, &b, &c) >= 1) { pl.near_lb2 = a; pl.near_lb3 = b; pl.near_lb3m = c; }
    }
    GPM_TRY(level_buffers(pl, 1));
    // stage the carried passes' structure (lv_elem reads t through the packed records)
    if (!pl.hpbuf.bytes) {
      GPM_TRY(level_pack(pl, pl.t.as<double>(), 1, false, nullptr));   // u := t1 (unused)
      GPM_TRY(level_setup(pl, nullptr));
      GPM_CUDA(cudaDeviceSynchronize());
    }
  }
  GPM_TRY(pl.w.alloc(sizeof(double) * n));
  return GP_OK;
}


static gp_status level_buffers(Plan& pl, int nrhs) {
  const size_t need = (size_t)nrhs * pl.n;
  if (pl.acc.bytes < sizeof(double) * need) GPM_TRY(pl.acc.alloc(sizeof(double) * need));
  if (pl.pts.bytes < level_pt_bytes() * need) GPM_TRY(pl.pts.alloc(level_pt_bytes() * need));
  // tile aggregates and (k_cp_carry) tile carries, same layout
  const size_t ag = 2 * level_rec_bytes(pl.d, pl.form == GP_FORM_PRODUCT, pl.P) * 2 *
                   (size_t)level_tiles(pl.n) * nrhs * level_nab(pl) *
                   std::max(1, pl.hp_npass);
  if (pl.aggs.bytes < ag) GPM_TRY(pl.aggs.alloc(ag));
  const size_t pb = sizeof(double) * (size_t)std::max(1, level_nparts(pl)) * pl.n * nrhs;
  if (pl.part.bytes < pb) {
    GPM_TRY(pl.part.alloc(pb));
    pl.part_zero_cols = 0;
  }
  return GP_OK;
}

int cg_nblk(const Plan& pl) {
  return pl.d == 1 ? (pl.d1_path == 3 ? 0 : pl.d1_grid) : egrid(pl.n);
}

static gp_status apply_levels(Plan& pl, const double* v, double* out, int nrhs, bool user_order,
                              cudaStream_t s, int kind, double cg_s2 = 0.0,
                              double* cg_part = nullptr, bool prepacked = false) {
  const int64_t vstride = user_order ? pl.n_src : pl.n;
  const int64_t ostride = user_order ? pl.n - pl.tgt_off : pl.n;
  for (int c0 = 0; c0 < nrhs; c0 += LV_MAXB) {
    const int nb = std::min(LV_MAXB, nrhs - c0);
    GPM_TRY(level_buffers(pl, nb));
    int launches = 0;
    if (!(prepacked && !user_order && nrhs <= LV_MAXB))
      GPM_TRY(level_pack(pl, v + c0 * vstride, nb, user_order, s));   // packed points (+ gather)
    const int nph = level_phases(pl, kind);
    if (nph > 1 && cg_part) return fail(GP_ERR_UNSUPPORTED, "internal: CG epilogue on a two-run apply");
    for (int ph = 0; ph < nph; ++ph) {
      GPM_TRY(level_passes(pl, nb, s, &launches, kind, ph));   // first level launch initialises acc
      k_epilogue<<<dim3(egrid(pl.n), nb), 256, 0, s>>>(
          user_order ? pl.perm.as<int>() : nullptr, pl.pts.as<double>(), pl.acc.as<double>(),
          pl.part.as<double>(), level_nparts(pl) - pl.low_unused, (int64_t)level_nparts(pl) * pl.n,
          pl.n, user_order ? pl.tgt_off : 0, pl.os2,
          (kind == 0 && pl.shard == 0) ? 1.0 : 0.0, out + c0 * ostride, ostride, cg_s2, cg_part,
          c0, ph > 0);   // a sharded apply adds the self term on shard 0 only
      GPM_CUDA(cudaGetLastError());
      launches += ph > 0 ? 1 : 0;
    }
    pl.launches_per_apply = launches + 2;   // + pack + epilogue (per batch of columns)
  }
  return GP_OK;
}

gp_status permute_vec(Plan& pl, const double* src, double* dst, bool to_rank, cudaStream_t s) {
  if (to_rank)
    k_gather<<<egrid(pl.n), 256, 0, s>>>(pl.perm.as<int>(), src, pl.n, pl.n, dst);
  else
    k_scatter_user<<<egrid(pl.n), 256, 0, s>>>(pl.perm.as<int>(), src, pl.n, dst);
  GPM_CUDA(cudaGetLastError());
  return GP_OK;
}

gp_status apply_rank(Plan& pl, const double* u_rank, double* out_rank, int nrhs, cudaStream_t s,
                     int kind, double cg_s2, double* cg_part, bool prepacked) {
  if (pl.d == 1) return d1_launch(pl, u_rank, out_rank, nrhs, false, s, kind, cg_s2, cg_part);
  return apply_levels(pl, u_rank, out_rank, nrhs, false, s, kind, cg_s2, cg_part, prepacked);
}

gp_status apply_user(Plan& pl, const double* v, double* out, int nrhs, cudaStream_t s, int kind) {
  if (pl.d == 1) return d1_launch(pl, v, out, nrhs, true, s, kind);
  return apply_levels(pl, v, out, nrhs, true, s, kind);
}

// Algorithmic HBM bytes of one single-RHS user-order apply:
// the stored structure is read once and v / out are touched once.
int64_t apply_model_bytes(const Plan& pl) {
  const int64_t n = pl.n;
  const int64_t L = pl.L;
  if (pl.d == 1) return n * (8 + 4 + 8 + 8);
  if (pl.d == 2) return n * (8 + 4 + 8 + 16 + 4 * L);
  return n * (8 + 4 + 8 + 24 + 4 * L + 2 * L * (L + 1));
}

}  // namespace gpm
