// apply_d1_fast.cu -- the d = 1 hot path when one CTA's chunk fits in shared memory
// (N <= #SMs x BLOCK x ITEMS, every config of BASELINE.json).  Same method and algebra
// as apply_d1.cu (P:314-340 [eq fast_exact_decomposition_1d, §2.1]); B200 layout:
//   * grid = #SMs CTAs (cooperative launch), one contiguous chunk of the sorted order
//     per CTA, BLOCK threads x ITEMS consecutive points each (ITEMS odd: conflict-free
//     8-byte shared-memory strides);
//   * the chunk's sorted coordinates and permutation arrive by TMA bulk copies
//     (cp.async.bulk -> UBLKCP) tracked by one mbarrier;
//   * user order: each thread issues its random gathers v[perm] first and computes its
//     e^{-gap} (branch-free fexp_neg) while they are in flight;
//   * loops are guard-free: points past the chunk end are neutral (gap 0, weight 0);
//   * block scan (warp shuffles) -> chunk aggregate -> cg grid.sync -> warp 0 / 1 fold
//     the other chunks' aggregates (forward / backward carries);
//   * pass 2 re-runs the two recurrences from the carries; outputs are scattered to
//     out[perm] (user order) or written back coalesced (rank order, the CG operator).
#include <cooperative_groups.h>

#include <algorithm>

#include "algebra.cuh"
#include "fexp.cuh"
#include "internal.h"
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace gpm {

struct DFArgs {
  const double* ts;   // sorted scaled coordinates (plan-owned, padded, 16B aligned)
  const int* perm;    // rank -> user index (plan-owned, padded)
  const double* v;    // input: user order (user_order) or rank order
  double* out;        // output: user order (targets only) or rank order
  int64_t n, n_src, tgt_off, chunk;
  int user_order;
  int nrhs;               // columns processed in this launch (multi-RHS, §8(f) f1)
  int prefetch;           // user order: L2 prefetch of v slices
  int64_t vstride, ostride;
  double os2;
  D1Agg* chunk_aggs;      // D1Pub[2][grid] (see below; double-buffered per column)
  unsigned* bar;          // [0]: finished-CTA counter, [2..3]: 64-bit launch epoch
  unsigned long long* dbg;   // optional per-CTA phase timestamps (GPM_D1_TIMING)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define DF_STAMP(k)                                                          \
  do {                                                                       \
    if (a.dbg && threadIdx.x == 0) a.dbg[blockIdx.x * 8 + (k)] = gtimer();   \
  } while (0)

template <int P>
struct SF {
  double D, E, M[P + 1];
};

template <int P>
__device__ __forceinline__ SF<P> sf_id() {
  SF<P> s;
  s.D = 0.0; s.E = 1.0;
#pragma unroll
  for (int q = 0; q <= P; ++q) s.M[q] = 0.0;
  return s;
}
template <int P>  // forward, A left of B
__device__ __forceinline__ SF<P> sf_cf(const SF<P>& A, const SF<P>& B) {
  SF<P> r;
#pragma unroll
  for (int q = 0; q <= P; ++q) r.M[q] = A.M[q];
  advance<P>(r.M, B.D, B.E);
#pragma unroll
  for (int q = 0; q <= P; ++q) r.M[q] += B.M[q];
  r.D = A.D + B.D; r.E = A.E * B.E;
  return r;
}
template <int P>  // backward, A left of B
__device__ __forceinline__ SF<P> sf_cb(const SF<P>& A, const SF<P>& B) {
  SF<P> r;
#pragma unroll
  for (int q = 0; q <= P; ++q) r.M[q] = B.M[q];
  advance<P>(r.M, A.D, A.E);
#pragma unroll
  for (int q = 0; q <= P; ++q) r.M[q] += A.M[q];
  r.D = A.D + B.D; r.E = A.E * B.E;
  return r;
}
template <int P>
__device__ __forceinline__ SF<P> sf_shfl(const SF<P>& s, int off, bool up) {
  SF<P> r;
  if (up) {
    r.D = __shfl_up_sync(0xffffffffu, s.D, off);
    r.E = __shfl_up_sync(0xffffffffu, s.E, off);
#pragma unroll
    for (int q = 0; q <= P; ++q) r.M[q] = __shfl_up_sync(0xffffffffu, s.M[q], off);
  } else {
    r.D = __shfl_down_sync(0xffffffffu, s.D, off);
    r.E = __shfl_down_sync(0xffffffffu, s.E, off);
#pragma unroll
    for (int q = 0; q <= P; ++q) r.M[q] = __shfl_down_sync(0xffffffffu, s.M[q], off);
  }
  return r;
}
template <int P>
__device__ __forceinline__ void sf_st(double* p, const SF<P>& s) {
  p[0] = s.D; p[1] = s.E;
#pragma unroll
  for (int q = 0; q <= P; ++q) p[2 + q] = s.M[q];
}
template <int P>
__device__ __forceinline__ SF<P> sf_ld(const double* p) {
  SF<P> s; s.D = p[0]; s.E = p[1];
#pragma unroll
  for (int q = 0; q <= P; ++q) s.M[q] = p[2 + q];
  return s;
}

// Published chunk aggregate: D, E, F[3], B[3] and the launch epoch (written last).
struct __align__(16) D1Pub {   // 128 B (apply_d1.cu allocates 128 x 2 x grid)
  double v[14];   // D, E, F[6], B[6]  (moment order <= 5)
  unsigned long long epoch;
  unsigned long long pad;
};

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

constexpr int DF_NPART = 4;   // TMA load pipeline depth (parts of the chunk)

template <int P, int KIND, int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK, 1) k_d1_fast(DFArgs a) {
  // P = moment order; KIND 0: K v (Matern nu = P + 1/2), KIND 1: dK/dlog(l) v (nu = P - 1/2)
  // Loops over the per-thread points are rolled where the body is large: every launch
  // walks the kernel once and instruction fetch from L2 is not free.
  constexpr int SUB = BLOCK * ITEMS;
  constexpr int NW = BLOCK / 32;
  constexpr int PT = BLOCK / DF_NPART;          // threads per load part
  constexpr int PSZ = PT * ITEMS;               // points per load part
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* s_t = reinterpret_cast<double*>(smem_raw);   // SUB + 8
  double* s_u = s_t + SUB + 8;                         // SUB
  double* s_e = s_u + SUB;                             // SUB
  int* s_pi = reinterpret_cast<int*>(s_e + SUB);       // SUB + 8
  __shared__ uint64_t mbar[DF_NPART];
  __shared__ double s_tab[64];
  constexpr int NSF = P + 3;   // D, E, M[0..P]
  __shared__ double s_wf[NW][NSF], s_wb[NW][NSF];
  __shared__ double s_tot[2][NSF];
  __shared__ double s_part[2][8][NSF];
  __shared__ double s_carry[2][P + 1];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c0 = (int64_t)blockIdx.x * a.chunk;
  const int cnt = (int)max((int64_t)0, min(a.chunk, a.n - c0));
  D1Pub* pub = reinterpret_cast<D1Pub*>(a.chunk_aggs);

  DF_STAMP(0);
  fexp_table_init(s_tab);
  if (tid == 0) {
    for (int p = 0; p < DF_NPART; ++p) mbar_init(&mbar[p], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // v is read only after griddepcontrol.wait (PDL: the previous kernel may produce it);
  // t and perm are plan-owned and read-only, so their TMA copies start immediately
  const bool u_tma = false;
  if (tid < DF_NPART && cnt > 0) {
    const int p = tid;
    const int lo = p * PSZ;
    const int hi = min(cnt, lo + PSZ);
    if (lo < hi) {   // lo is a multiple of 4 (PSZ = PT * ITEMS with PT % 4 == 0)
      const unsigned nt = (unsigned)(((hi - lo) + 1) & ~1);     // padded plan arrays
      const unsigned np = (unsigned)(((hi - lo) + 3) & ~3);
      const unsigned nu = (unsigned)((hi - lo) & ~1);           // never over-read v
      unsigned bytes = nt * 8;
      if (a.user_order) bytes += np * 4;
      if (u_tma) bytes += nu * 8;
      mbar_expect_tx(&mbar[p], bytes);
      tma_load_1d(s_t + lo, a.ts + c0 + lo, nt * 8, &mbar[p]);
      if (a.user_order) tma_load_1d(s_pi + lo, a.perm + c0 + lo, np * 4, &mbar[p]);
      if (u_tma && nu) tma_load_1d(s_u + lo, a.v + c0 + lo, nu * 8, &mbar[p]);
    }
  }
  // user order: the random gathers of v hit L2 if v was streamed in first -- each CTA
  // prefetches an equal slice of the first column (L2 is coherent: safe under PDL)
  auto prefetch_v = [&](int col) {
    const int64_t lo = min((int64_t)blockIdx.x * ((a.n_src + gridDim.x - 1) / gridDim.x), a.n_src);
    const int64_t hi = min(lo + (a.n_src + gridDim.x - 1) / gridDim.x, a.n_src);
    if (hi > lo) prefetch_l2_range(a.v + col * a.vstride + lo, (size_t)(hi - lo) * 8);
  };
  if (a.user_order && a.prefetch && tid == 32) prefetch_v(0);
  const int j0 = tid * ITEMS;
  const int mypart = tid / PT;
  double tprev = 0.0, tlast = 0.0;
  if (cnt > 0) {
    tlast = __ldg(a.ts + c0 + cnt - 1);
    const int64_t gp = c0 + min(j0, cnt) - 1;
    tprev = gp >= 0 ? __ldg(a.ts + gp) : __ldg(a.ts);
    if (j0 >= cnt) tprev = tlast;
    if (mypart * PSZ < cnt)
      while (!mbar_try_wait(&mbar[mypart], 0)) {
      }
  }
  DF_STAMP(1);
  // gaps and e^{-gap}: plan data only -> overlaps the previous kernel's tail under PDL
  {
    double tp = tprev;
#pragma unroll 1
    for (int k = 0; k < ITEMS; ++k) {
      const int j = j0 + k;
      const double t = j < cnt ? s_t[j] : tlast;
      const double dl = t - tp;            // neutral (0) past the chunk end
      tp = t;
      s_t[j] = dl;                         // t -> gap (own slot; neighbours use tprev)
      s_e[j] = fexp_neg(dl, s_tab);
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");   // no-op without a PDL predecessor

#pragma unroll 1
  for (int col = 0; col < a.nrhs; ++col) {
  const double* vcol = a.v + col * a.vstride;
  double* ocol = a.out + col * a.ostride;
  D1Pub* pubc = pub + (col & 1) * gridDim.x;   // slots alternate: a CTA runs <= 1 sync ahead
  if (a.user_order && a.prefetch && tid == 32 && col + 1 < a.nrhs) prefetch_v(col + 1);
  {
    if (col > 0) __syncthreads();   // s_u of the previous column fully consumed
    if (!a.user_order) {
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        const int j = k * BLOCK + tid;
        s_u[j] = j < cnt ? __ldg(vcol + c0 + j) : 0.0;
      }
      __syncthreads();
    }
  }
  // ---- gathers (user order) first: all ITEMS loads in flight ...
  double uu[ITEMS];
  if (a.user_order) {
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const int j = j0 + k;
      const int pi = j < cnt ? s_pi[j] : INT_MAX;
      uu[k] = pi < a.n_src ? __ldg(vcol + pi) : 0.0;
    }
  }
  if (a.user_order) {
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) s_u[j0 + k] = uu[k];
  }

  // ---- pass 1: forward partial moments by the recurrence; backward partial moments
  // (referenced one point before my first point) accumulated directly from the
  // cumulative span Dc and e^{-Dc}.
  SF<P> F = sf_id<P>(), B = sf_id<P>();
  {
    double Dc = 0.0, Ec = 1.0;
#pragma unroll 1
    for (int k = 0; k < ITEMS; ++k) {
      const int j = j0 + k;
      const double dl = s_t[j], e = s_e[j], u = s_u[j];
      Dc += dl;
      Ec *= e;
      double wq = u * Ec;                  // u Dc^q e^{-Dc}, q = 0..P
#pragma unroll
      for (int q = 0; q <= P; ++q) {
        B.M[q] += wq;
        wq *= Dc;
      }
      advance<P>(F.M, dl, e);
      F.M[0] += u;
    }
    F.D = B.D = Dc;
    F.E = B.E = Ec;
  }
  DF_STAMP(2);

  // ---- block scan: warp level (forward inclusive up, backward inclusive down)
  SF<P> fi = F, bi = B;
#pragma unroll 1
  for (int off = 1; off < 32; off <<= 1) {
    SF<P> l = sf_shfl<P>(fi, off, true);
    SF<P> r = sf_shfl<P>(bi, off, false);
    if (lane >= off) fi = sf_cf<P>(l, fi);
    if (lane + off < 32) bi = sf_cb<P>(bi, r);
  }
  if (lane == 31) sf_st<P>(s_wf[warp], fi);
  if (lane == 0) sf_st<P>(s_wb[warp], bi);
  SF<P> fe = sf_shfl<P>(fi, 1, true);
  SF<P> be = sf_shfl<P>(bi, 1, false);
  if (lane == 0) fe = sf_id<P>();
  if (lane == 31) be = sf_id<P>();
  __syncthreads();
  if (warp < 2) {   // warp 0: exclusive scan of forward warp totals; warp 1: backward
    const bool fw = warp == 0;
    SF<P> x = lane < NW ? sf_ld<P>(fw ? s_wf[lane] : s_wb[lane]) : sf_id<P>();
#pragma unroll 1
    for (int off = 1; off < NW; off <<= 1) {
      SF<P> y = sf_shfl<P>(x, off, fw);
      if (fw && lane >= off) x = sf_cf<P>(y, x);
      if (!fw && lane + off < 32) x = sf_cb<P>(x, y);
    }
    SF<P> xe = sf_shfl<P>(x, 1, fw);
    if ((fw && lane == 0) || (!fw && lane >= NW - 1)) xe = sf_id<P>();
    __syncwarp();
    if (lane < NW) sf_st<P>(fw ? s_wf[lane] : s_wb[lane], xe);
    if (fw && lane == NW - 1) sf_st<P>(s_tot[0], x);
    if (!fw && lane == 0) sf_st<P>(s_tot[1], x);
  }
  __syncthreads();
  // ---- publish the chunk aggregate, grid-wide sync (cooperative launch)
  if (tid == 0) {
    D1Pub* me = pubc + blockIdx.x;
    me->v[0] = s_tot[0][0];
    me->v[1] = s_tot[0][1];
#pragma unroll
    for (int q = 0; q <= P; ++q) {
      me->v[2 + q] = s_tot[0][2 + q];
      me->v[8 + q] = s_tot[1][2 + q];
    }
    __threadfence();
  }
  DF_STAMP(3);
  const SF<P> Fx = sf_cf<P>(sf_ld<P>(s_wf[warp]), fe);
  const SF<P> Bx = sf_cb<P>(be, sf_ld<P>(s_wb[warp]));
  cg::this_grid().sync();
  // ---- carries: warp pair (2g, 2g+1) folds chunks [32g, 32g+32) forward / backward;
  // one aggregate per lane, all loads in flight at once.
  {
    const int G = gridDim.x, b = blockIdx.x;
    const int ngroups = (G + 31) / 32;
    if (warp < 2 * ngroups) {
      const bool fw = (warp & 1) == 0;
      const int grp = warp >> 1;
      const int jj = grp * 32 + lane;
      const bool take = fw ? (jj < b) : (jj > b && jj < G);
      SF<P> X = sf_id<P>();
      if (take) {
        const D1Pub* o = pubc + jj;
        X.D = __ldcg(&o->v[0]);
        X.E = __ldcg(&o->v[1]);
#pragma unroll
        for (int q = 0; q <= P; ++q) X.M[q] = __ldcg(&o->v[(fw ? 2 : 8) + q]);
      }
#pragma unroll 1
      for (int off = 1; off < 32; off <<= 1) {
        SF<P> Y = sf_shfl<P>(X, off, false);
        if (lane + off < 32) X = fw ? sf_cf<P>(X, Y) : sf_cb<P>(X, Y);
      }
      if (lane == 0) sf_st<P>(s_part[fw ? 0 : 1][grp], X);
    }
    __syncthreads();
    if (tid < 2) {
      const bool fw = tid == 0;
      SF<P> X = sf_id<P>();
#pragma unroll 1
      for (int gi = 0; gi < ngroups; ++gi) {
        const SF<P> y = sf_ld<P>(s_part[fw ? 0 : 1][gi]);
        X = fw ? sf_cf<P>(X, y) : sf_cb<P>(X, y);
      }
#pragma unroll
      for (int q = 0; q <= P; ++q) s_carry[tid][q] = X.M[q];
    }
    __syncthreads();
  }
  DF_STAMP(4);
  DF_STAMP(5);

  // ---- pass 2 (unrolled: the forward reads stay in registers; the body is small)
  double M[P + 1], rf[ITEMS];
  {
    double Cf[P + 1];
#pragma unroll
    for (int q = 0; q <= P; ++q) Cf[q] = s_carry[0][q];
    advance<P>(Cf, Fx.D, Fx.E);
#pragma unroll
    for (int q = 0; q <= P; ++q) M[q] = Cf[q] + Fx.M[q];
  }
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const int j = j0 + k;
    advance<P>(M, s_t[j], s_e[j]);       // s_t now holds the gaps
    rf[k] = readc0<P, KIND>(M);
    M[0] += s_u[j];
  }
  {
    double Cb[P + 1];
#pragma unroll
    for (int q = 0; q <= P; ++q) Cb[q] = s_carry[1][q];
    advance<P>(Cb, Bx.D, Bx.E);
#pragma unroll
    for (int q = 0; q <= P; ++q) M[q] = Bx.M[q] + Cb[q];
  }
#pragma unroll
  for (int k = ITEMS - 1; k >= 0; --k) {
    const int j = j0 + k;
    const double uj = s_u[j];
    const double val = a.os2 * ((KIND == 0 ? uj : 0.0) + (rf[k] + readc0<P, KIND>(M)));
    M[0] += uj;
    advance<P>(M, s_t[j], s_e[j]);
    if (a.user_order) {
      if (j < cnt) {
        const int pi = s_pi[j];
        if (pi >= a.tgt_off) ocol[pi - a.tgt_off] = val;
      }
    } else {
      s_u[j] = val;   // staged for a coalesced write-back
    }
  }
  if (!a.user_order) {
    __syncthreads();
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const int j = k * BLOCK + tid;
      if (j < cnt) ocol[c0 + j] = s_u[j];
    }
  }
  }   // column loop
  asm volatile("griddepcontrol.launch_dependents;");
  if (a.dbg) {
    __syncthreads();
    DF_STAMP(6);
  }
}

// ---------------------------------------------------------------------------
// Host side.  Shapes (BLOCK, ITEMS): 0 = (512, 15), 1 = (640, 11), 2 = (768, 9),
// 3 = (1024, 7).  The default is chosen by measurement.
template <int BLOCK, int ITEMS>
static size_t df_smem() {
  constexpr int SUB = BLOCK * ITEMS;
  return sizeof(double) * (3 * SUB + 8) + sizeof(int) * (SUB + 8);
}

struct DFShape {
  int block, items;
  const void* fn[10];  // [KIND * 5 + p]: KIND 0 moment order p, KIND 1 moment order p + 1
  size_t smem;
};

template <int BLOCK, int ITEMS>
static DFShape make_shape() {
  DFShape s;
  s.block = BLOCK;
  s.items = ITEMS;
  s.fn[0] = (const void*)k_d1_fast<0, 0, BLOCK, ITEMS>;
  s.fn[1] = (const void*)k_d1_fast<1, 0, BLOCK, ITEMS>;
  s.fn[2] = (const void*)k_d1_fast<2, 0, BLOCK, ITEMS>;
  s.fn[3] = (const void*)k_d1_fast<3, 0, BLOCK, ITEMS>;
  s.fn[4] = (const void*)k_d1_fast<4, 0, BLOCK, ITEMS>;
  s.fn[5] = (const void*)k_d1_fast<1, 1, BLOCK, ITEMS>;
  s.fn[6] = (const void*)k_d1_fast<2, 1, BLOCK, ITEMS>;
  s.fn[7] = (const void*)k_d1_fast<3, 1, BLOCK, ITEMS>;
  s.fn[8] = (const void*)k_d1_fast<4, 1, BLOCK, ITEMS>;
  s.fn[9] = (const void*)k_d1_fast<5, 1, BLOCK, ITEMS>;
  s.smem = df_smem<BLOCK, ITEMS>();
  return s;
}

static DFShape g_shapes[4];
static int g_shapes_ready = 0;
static int g_default_shape = 2;   // 768 x 9: best measured (profiles/)

static gp_status df_init() {
  if (g_shapes_ready) return GP_OK;
  g_shapes[0] = make_shape<512, 15>();
  g_shapes[1] = make_shape<640, 11>();
  g_shapes[2] = make_shape<768, 9>();
  g_shapes[3] = make_shape<1024, 7>();
  for (auto& s : g_shapes)
    for (int p = 0; p < 10; ++p)
      GPM_CUDA(cudaFuncSetAttribute(s.fn[p], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)s.smem));
  if (const char* e = getenv("GPM_D1_SHAPE")) g_default_shape = std::max(0, std::min(3, atoi(e)));
  g_shapes_ready = 1;
  return GP_OK;
}

int df_default_shape() { return g_default_shape; }

// capacity per CTA and max co-resident grid for a shape
gp_status df_shape_info(int shape, int* capacity, int* max_grid) {
  GPM_TRY(df_init());
  const DFShape& s = g_shapes[shape];
  int dev = 0, nsm = 0, occ = 0;
  GPM_CUDA(cudaGetDevice(&dev));
  GPM_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  GPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, s.fn[2], s.block, s.smem));
  *capacity = s.block * s.items;
  *max_grid = occ * nsm;
  return GP_OK;
}

gp_status df_launch(Plan& pl, const double* v, double* out, int nrhs, bool user_order,
                    cudaStream_t s, int kind) {
  const DFShape& sh = g_shapes[pl.d1_shape];
  DFArgs a;
  a.ts = pl.t.as<double>();
  a.perm = pl.perm.as<int>();
  a.v = v;
  a.out = out;
  a.n = pl.n;
  a.n_src = user_order ? pl.n_src : pl.n;
  a.tgt_off = user_order ? pl.tgt_off : 0;
  a.chunk = pl.d1_chunk;
  a.user_order = user_order ? 1 : 0;
  a.nrhs = nrhs;
  a.prefetch = pl.d1_prefetch;
  a.vstride = user_order ? pl.n_src : pl.n;
  a.ostride = user_order ? pl.n - pl.tgt_off : pl.n;
  a.os2 = pl.os2;
  a.chunk_aggs = pl.aggs.as<D1Agg>();
  a.bar = pl.bar.as<unsigned>();
  a.dbg = pl.dbg.bytes ? pl.dbg.as<unsigned long long>() : nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.d1_grid);
  cfg.blockDim = dim3(sh.block);
  cfg.dynamicSmemBytes = sh.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pl.d1_pdl ? 2 : 1;
  void* args[] = {&a};
  GPM_CUDA(cudaLaunchKernelExC(&cfg, sh.fn[kind * 5 + pl.P], args));
  return GP_OK;
}

}  // namespace gpm
