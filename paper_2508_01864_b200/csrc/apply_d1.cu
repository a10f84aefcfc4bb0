// apply_d1.cu -- d = 1 hot path: K v by the 1-D ECDF decomposition
//   sum_i y_i k(|x_i - z|) = sum_p phi1_p(z) CDF_p(z) + phi1_p(-z) SURV_p(z)
// (P:314-325 [eq fast_exact_decomposition_1d]) evaluated by "fast sum updating"
// over the presorted data (P:326-340 [§2.1]) as two prefix scans -- a forward scan
// (sources left of the target: the CDF part) and a backward scan (sources right of
// it: the survival part) -- in the overflow-free moment basis of algebra.cuh.
//
// B200 design: ONE cooperative launch, grid = 148 CTAs x 512 threads
// (one per SM, every CTA co-resident).  CTA b owns a contiguous chunk of the sorted
// order; the chunk's t, perm and the gathered v sit in 215 KB of shared memory.
//   pass 1: per-thread sequential recurrences -> block scan of (span, moments) in both
//           directions (warp shuffles) -> chunk aggregate published to global memory;
//   barrier: self-resetting grid barrier (all CTAs resident, so no deadlock);
//   carries: warp 0 folds the aggregates of chunks < b (forward), warp 1 those > b
//           (backward) -- a decoupled look-back/look-ahead in one step;
//   pass 2: re-run the per-thread recurrences from the carries, scatter out[perm].
// The data is read from HBM exactly once: t (8 B) + perm (4 B) + v (8 B) + out (8 B).
// Chunks larger than one shared-memory sub-tile stream through sub-tiles (re-read).
#include <cooperative_groups.h>

#include <algorithm>

#include "algebra.cuh"
#include "internal.h"

namespace gpm {

__device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t lmax(int64_t a, int64_t b) { return a > b ? a : b; }

constexpr int D1_BLOCK = 512;
constexpr int D1_ITEMS = 15;                 // odd: conflict-free strided 8-byte smem access
constexpr int D1_SUB = D1_BLOCK * D1_ITEMS;  // 7680 points per shared-memory sub-tile
constexpr int D1_WARPS = D1_BLOCK / 32;
constexpr int D1_MAXSUB = 64;

template <int P>
struct St {  // one-direction scan element: span D, E = e^{-D}, moments M
  double D, E, M[P + 1];
};

template <int P>
__device__ __forceinline__ St<P> st_identity() {
  St<P> s;
  s.D = 0.0; s.E = 1.0;
#pragma unroll
  for (int q = 0; q <= P; ++q) s.M[q] = 0.0;
  return s;
}

// forward: A then B (A left of B): M = S(B.D) A.M + B.M
template <int P>
__device__ __forceinline__ St<P> comb_f(const St<P>& A, const St<P>& B) {
  St<P> r;
#pragma unroll
  for (int q = 0; q <= P; ++q) r.M[q] = A.M[q];
  advance<P>(r.M, B.D, B.E);
#pragma unroll
  for (int q = 0; q <= P; ++q) r.M[q] += B.M[q];
  r.D = A.D + B.D; r.E = A.E * B.E;
  return r;
}

// backward: A left of B: M = A.M + S(A.D) B.M
template <int P>
__device__ __forceinline__ St<P> comb_b(const St<P>& A, const St<P>& B) {
  St<P> r;
#pragma unroll
  for (int q = 0; q <= P; ++q) r.M[q] = B.M[q];
  advance<P>(r.M, A.D, A.E);
#pragma unroll
  for (int q = 0; q <= P; ++q) r.M[q] += A.M[q];
  r.D = A.D + B.D; r.E = A.E * B.E;
  return r;
}

template <int P>
__device__ __forceinline__ St<P> shfl_st_up(const St<P>& s, int off) {
  St<P> r;
  r.D = __shfl_up_sync(0xffffffffu, s.D, off);
  r.E = __shfl_up_sync(0xffffffffu, s.E, off);
#pragma unroll
  for (int q = 0; q <= P; ++q) r.M[q] = __shfl_up_sync(0xffffffffu, s.M[q], off);
  return r;
}
template <int P>
__device__ __forceinline__ St<P> shfl_st_down(const St<P>& s, int off) {
  St<P> r;
  r.D = __shfl_down_sync(0xffffffffu, s.D, off);
  r.E = __shfl_down_sync(0xffffffffu, s.E, off);
#pragma unroll
  for (int q = 0; q <= P; ++q) r.M[q] = __shfl_down_sync(0xffffffffu, s.M[q], off);
  return r;
}

template <int P>
__device__ __forceinline__ St<P> agg_f(const D1Agg& a) {
  St<P> s; s.D = a.D; s.E = a.E;
#pragma unroll
  for (int q = 0; q <= P; ++q) s.M[q] = a.F[q];
  return s;
}
template <int P>
__device__ __forceinline__ St<P> agg_b(const D1Agg& a) {
  St<P> s; s.D = a.D; s.E = a.E;
#pragma unroll
  for (int q = 0; q <= P; ++q) s.M[q] = a.B[q];
  return s;
}
__device__ __forceinline__ D1Agg ldcg_agg(const D1Agg* p) {
  D1Agg a;
  const double* s = reinterpret_cast<const double*>(p);
  double* d = reinterpret_cast<double*>(&a);
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i] = __ldcg(s + i);
  return a;
}

struct D1Smem {
  double x[D1_SUB];   // t, then the gap Delta_j = t_j - t_{j-1}
  double e[D1_SUB];   // e^{-Delta_j}
  double u[D1_SUB];   // v[perm_j] (0 for non-sources)
  int pi[D1_SUB];     // perm_j (user index)
};

struct D1Scratch {
  double wf[D1_WARPS][5];  // warp totals, forward (D, E, M0..M2)
  double wb[D1_WARPS][5];
  double wfx[D1_WARPS][5]; // exclusive prefixes of the warp totals
  double wbx[D1_WARPS][5];
  double tot[2][5];        // sub-tile totals (forward, backward)
  double carry[2][5];      // forward / backward carry of the current sub-tile
  double subB[D1_MAXSUB][3];
};

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = bar + 1;
    const unsigned gen = *vgen;
    __threadfence();
    const unsigned arrived = atomicAdd(bar, 1u);
    if (arrived == nblocks - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      unsigned cur;
      do {
        __nanosleep(32);
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory");
      } while (cur == gen);
    }
    __threadfence();
  }
  __syncthreads();
}

struct D1Args {
  const double* ts;   // sorted scaled coordinate (rank order)
  const int* perm;    // rank -> user index, or nullptr (rank-space vectors)
  const double* v;    // input (user order if perm, else rank order)
  double* out;        // output (user order if perm, else rank order)
  int64_t n, n_src, tgt_off, chunk;
  int nsub;
  double os2;
  D1Agg* chunk_aggs;  // [grid]
  D1Agg* sub_aggs;    // [grid][D1_MAXSUB] (only when nsub > 1)
  unsigned* bar;
};

// Load sub-tile [g0, g0+cnt) into smem and convert t -> gaps; compute e^{-gap}.
__device__ __forceinline__ void d1_load(const D1Args& a, D1Smem& sm, int64_t g0, int cnt) {
  const int tid = threadIdx.x;
  double tv[D1_ITEMS];
  int pv[D1_ITEMS];
#pragma unroll
  for (int k = 0; k < D1_ITEMS; ++k) {
    const int i = k * D1_BLOCK + tid;
    if (i < cnt) {
      tv[k] = __ldg(a.ts + g0 + i);
      pv[k] = a.perm ? __ldg(a.perm + g0 + i) : static_cast<int>(g0 + i);
    }
  }
#pragma unroll
  for (int k = 0; k < D1_ITEMS; ++k) {
    const int i = k * D1_BLOCK + tid;
    if (i < cnt) {
      sm.x[i] = tv[k];
      sm.pi[i] = pv[k];
      tv[k] = (pv[k] < a.n_src) ? __ldg(a.v + pv[k]) : 0.0;  // gather
    }
  }
#pragma unroll
  for (int k = 0; k < D1_ITEMS; ++k) {
    const int i = k * D1_BLOCK + tid;
    if (i < cnt) sm.u[i] = tv[k];
  }
  __syncthreads();
  const int i0 = tid * D1_ITEMS;
  double tprev = 0.0;
  if (i0 < cnt) {
    if (i0 > 0) tprev = sm.x[i0 - 1];
    else tprev = (g0 > 0) ? __ldg(a.ts + g0 - 1) : sm.x[0];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < D1_ITEMS; ++k) {
    const int i = i0 + k;
    if (i < cnt) {
      const double t = sm.x[i];
      const double dl = t - tprev;
      tprev = t;
      sm.x[i] = dl;
      sm.e[i] = exp(-dl);
    }
  }
  __syncthreads();
}

// Per-thread aggregates of its items (forward F, backward B, common D/E).
template <int P>
__device__ __forceinline__ void d1_thread_aggs(const D1Smem& sm, int cnt, St<P>& F, St<P>& B) {
  const int i0 = threadIdx.x * D1_ITEMS;
  F = st_identity<P>();
  B = st_identity<P>();
#pragma unroll
  for (int k = 0; k < D1_ITEMS; ++k) {
    const int i = i0 + k;
    if (i < cnt) {
      const double dl = sm.x[i], e = sm.e[i];
      advance<P>(F.M, dl, e);
      F.M[0] += sm.u[i];
      F.D += dl;
      F.E *= e;
    }
  }
#pragma unroll
  for (int k = D1_ITEMS - 1; k >= 0; --k) {
    const int i = i0 + k;
    if (i < cnt) {
      B.M[0] += sm.u[i];
      advance<P>(B.M, sm.x[i], sm.e[i]);
    }
  }
  B.D = F.D;
  B.E = F.E;
}

// Block-wide exclusive scans: Fx = combine of threads < me (forward),
// Bx = combine of threads > me (backward); sub-tile totals returned in Ft / Bt.
template <int P>
__device__ __forceinline__ St<P> ld_st(const double* p) {
  St<P> s; s.D = p[0]; s.E = p[1];
#pragma unroll
  for (int q = 0; q <= P; ++q) s.M[q] = p[2 + q];
  return s;
}
template <int P>
__device__ __forceinline__ void st_st(double* p, const St<P>& s) {
  p[0] = s.D; p[1] = s.E;
#pragma unroll
  for (int q = 0; q <= P; ++q) p[2 + q] = s.M[q];
}

template <int P>
__device__ __forceinline__ void d1_block_scan(D1Scratch& sc, const St<P>& F, const St<P>& B,
                                              St<P>& Fx, St<P>& Bx, St<P>& Ft, St<P>& Bt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  St<P> fi = F, bi = B;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    St<P> l = shfl_st_up<P>(fi, off);
    if (lane >= off) fi = comb_f<P>(l, fi);
    St<P> r = shfl_st_down<P>(bi, off);
    if (lane + off < 32) bi = comb_b<P>(bi, r);
  }
  if (lane == 31) st_st<P>(sc.wf[warp], fi);
  if (lane == 0) st_st<P>(sc.wb[warp], bi);
  St<P> fe = shfl_st_up<P>(fi, 1);
  if (lane == 0) fe = st_identity<P>();
  St<P> be = shfl_st_down<P>(bi, 1);
  if (lane == 31) be = st_identity<P>();
  __syncthreads();
  if (warp == 0) {          // exclusive scan of the forward warp totals
    St<P> x = lane < D1_WARPS ? ld_st<P>(sc.wf[lane]) : st_identity<P>();
#pragma unroll
    for (int off = 1; off < D1_WARPS; off <<= 1) {
      St<P> l = shfl_st_up<P>(x, off);
      if (lane >= off) x = comb_f<P>(l, x);
    }
    St<P> xe = shfl_st_up<P>(x, 1);
    if (lane == 0) xe = st_identity<P>();
    if (lane < D1_WARPS) st_st<P>(sc.wfx[lane], xe);
    if (lane == D1_WARPS - 1) st_st<P>(sc.tot[0], x);
  } else if (warp == 1) {   // exclusive suffix scan of the backward warp totals
    St<P> x = lane < D1_WARPS ? ld_st<P>(sc.wb[lane]) : st_identity<P>();
#pragma unroll
    for (int off = 1; off < D1_WARPS; off <<= 1) {
      St<P> r = shfl_st_down<P>(x, off);
      if (lane + off < 32) x = comb_b<P>(x, r);
    }
    St<P> xe = shfl_st_down<P>(x, 1);
    if (lane >= D1_WARPS - 1) xe = st_identity<P>();
    if (lane < D1_WARPS) st_st<P>(sc.wbx[lane], xe);
    if (lane == 0) st_st<P>(sc.tot[1], x);
  }
  __syncthreads();
  Fx = comb_f<P>(ld_st<P>(sc.wfx[warp]), fe);
  Bx = comb_b<P>(be, ld_st<P>(sc.wbx[warp]));
  Ft = ld_st<P>(sc.tot[0]);
  Bt = ld_st<P>(sc.tot[1]);
}

// Pass 2 for one sub-tile: per-thread recurrences from carries, scatter.
template <int P>
__device__ __forceinline__ void d1_apply_items(const D1Args& a, const D1Smem& sm, int cnt,
                                               const double* Fin, const double* Bin) {
  const int i0 = threadIdx.x * D1_ITEMS;
  double M[P + 1], rf[D1_ITEMS];
#pragma unroll
  for (int q = 0; q <= P; ++q) M[q] = Fin[q];
#pragma unroll
  for (int k = 0; k < D1_ITEMS; ++k) {
    const int i = i0 + k;
    rf[k] = 0.0;
    if (i < cnt) {
      advance<P>(M, sm.x[i], sm.e[i]);
      rf[k] = read0<P>(M);
      M[0] += sm.u[i];
    }
  }
#pragma unroll
  for (int q = 0; q <= P; ++q) M[q] = Bin[q];
#pragma unroll
  for (int k = D1_ITEMS - 1; k >= 0; --k) {
    const int i = i0 + k;
    if (i < cnt) {
      const double uu = sm.u[i];
      const double val = a.os2 * (uu + (rf[k] + read0<P>(M)));
      M[0] += uu;
      advance<P>(M, sm.x[i], sm.e[i]);
      const int pi = sm.pi[i];
      if (pi >= a.tgt_off) a.out[pi - a.tgt_off] = val;
    }
  }
}

template <int P>
__global__ void __launch_bounds__(D1_BLOCK, 1) k_d1_coop(D1Args a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  D1Smem& sm = *reinterpret_cast<D1Smem*>(smem_raw);
  __shared__ D1Scratch sc;

  const int64_t c0 = blockIdx.x * a.chunk;
  const int64_t c1 = min(a.n, c0 + a.chunk);
  const int64_t len = lmax(0, c1 - c0);
  St<P> F, B, Fx, Bx, Ft, Bt;
  St<P> chF = st_identity<P>(), chB = st_identity<P>();

  // ---- pass 1: chunk aggregate
  for (int s = 0; s < a.nsub; ++s) {
    const int64_t g0 = c0 + (int64_t)s * D1_SUB;
    const int cnt = (int)lmax(0, lmin(D1_SUB, c1 - g0));
    if (s > 0) __syncthreads();
    d1_load(a, sm, g0, cnt);
    d1_thread_aggs<P>(sm, cnt, F, B);
    d1_block_scan<P>(sc, F, B, Fx, Bx, Ft, Bt);
    if (a.nsub > 1 && threadIdx.x == 0) {
      D1Agg g; g.D = Ft.D; g.E = Ft.E;
      for (int q = 0; q < 3; ++q) { g.F[q] = q <= P ? Ft.M[q] : 0.0; g.B[q] = q <= P ? Bt.M[q] : 0.0; }
      a.sub_aggs[(int64_t)blockIdx.x * D1_MAXSUB + s] = g;
    }
    chF = comb_f<P>(chF, Ft);
    chB = comb_b<P>(chB, Bt);   // sub-tiles are visited left to right
  }
  (void)len;
  if (threadIdx.x == 0) {
    D1Agg g; g.D = chF.D; g.E = chF.E;
    for (int q = 0; q < 3; ++q) { g.F[q] = q <= P ? chF.M[q] : 0.0; g.B[q] = q <= P ? chB.M[q] : 0.0; }
    a.chunk_aggs[blockIdx.x] = g;
  }
  grid_barrier(a.bar, gridDim.x);

  // ---- carries from the other chunks (warp 0: forward, warp 1: backward)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp < 2) {
    const int b = blockIdx.x;
    const int lo = warp == 0 ? 0 : b + 1;
    const int hi = warp == 0 ? b : (int)gridDim.x;
    const int cntc = max(0, hi - lo);
    const int per = (cntc + 31) / 32;
    St<P> X = st_identity<P>();
    for (int k = 0; k < per; ++k) {
      const int j = lo + lane * per + k;
      if (j < hi) {
        const D1Agg g = ldcg_agg(a.chunk_aggs + j);
        X = warp == 0 ? comb_f<P>(X, agg_f<P>(g)) : comb_b<P>(X, agg_b<P>(g));
      }
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      St<P> Y = shfl_st_down<P>(X, off);
      if (lane + off < 32) X = warp == 0 ? comb_f<P>(X, Y) : comb_b<P>(X, Y);
    }
    if (lane == 0) {
      for (int q = 0; q <= P; ++q) sc.carry[warp][2 + q] = X.M[q];
    }
  }
  __syncthreads();

  if (a.nsub == 1) {
    // data, thread aggregates and block scan are still live: apply directly
    const int cnt = (int)len;
    double Fin[P + 1], Bin[P + 1];
#pragma unroll
    for (int q = 0; q <= P; ++q) { Fin[q] = sc.carry[0][2 + q]; Bin[q] = sc.carry[1][2 + q]; }
    // thread carry = combine(chunk carry, block-exclusive part)
    advance<P>(Fin, Fx.D, Fx.E);
    double tmp[P + 1];
#pragma unroll
    for (int q = 0; q <= P; ++q) { Fin[q] += Fx.M[q]; tmp[q] = Bin[q]; }
    advance<P>(tmp, Bx.D, Bx.E);
#pragma unroll
    for (int q = 0; q <= P; ++q) Bin[q] = Bx.M[q] + tmp[q];
    d1_apply_items<P>(a, sm, cnt, Fin, Bin);
    return;
  }

  // ---- nsub > 1: backward carries of each sub-tile (thread 0, sequential)
  if (threadIdx.x == 0) {
    double Bc[P + 1];
    for (int q = 0; q <= P; ++q) Bc[q] = sc.carry[1][2 + q];
    for (int s = a.nsub - 1; s >= 0; --s) {
      for (int q = 0; q <= P; ++q) sc.subB[s][q] = Bc[q];
      const D1Agg g = ldcg_agg(a.sub_aggs + (int64_t)blockIdx.x * D1_MAXSUB + s);
      St<P> A = agg_b<P>(g);
      double t2[P + 1];
      for (int q = 0; q <= P; ++q) t2[q] = Bc[q];
      advance<P>(t2, A.D, A.E);
      for (int q = 0; q <= P; ++q) Bc[q] = A.M[q] + t2[q];
    }
  }
  __syncthreads();
  double Fc[P + 1];
#pragma unroll
  for (int q = 0; q <= P; ++q) Fc[q] = sc.carry[0][2 + q];
  for (int s = 0; s < a.nsub; ++s) {
    const int64_t g0 = c0 + (int64_t)s * D1_SUB;
    const int cnt = (int)lmax(0, lmin(D1_SUB, c1 - g0));
    __syncthreads();
    d1_load(a, sm, g0, cnt);
    d1_thread_aggs<P>(sm, cnt, F, B);
    d1_block_scan<P>(sc, F, B, Fx, Bx, Ft, Bt);
    double Fin[P + 1], Bin[P + 1], tmp[P + 1];
#pragma unroll
    for (int q = 0; q <= P; ++q) { Fin[q] = Fc[q]; tmp[q] = sc.subB[s][q]; }
    advance<P>(Fin, Fx.D, Fx.E);
    advance<P>(tmp, Bx.D, Bx.E);
#pragma unroll
    for (int q = 0; q <= P; ++q) { Fin[q] += Fx.M[q]; Bin[q] = Bx.M[q] + tmp[q]; }
    d1_apply_items<P>(a, sm, cnt, Fin, Bin);
    // advance the forward carry over this sub-tile
    advance<P>(Fc, Ft.D, Ft.E);
#pragma unroll
    for (int q = 0; q <= P; ++q) Fc[q] += Ft.M[q];
  }
}

// ---------------------------------------------------------------------------
size_t d1_smem_bytes() { return sizeof(D1Smem); }

template <int P>
static cudaError_t d1_set_attr() {
  return cudaFuncSetAttribute(k_d1_coop<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)sizeof(D1Smem));
}

gp_status df_shape_info(int shape, int* capacity, int* max_grid);
gp_status df_launch(Plan& pl, const double* v, double* out, int nrhs, bool user_order,
                    cudaStream_t s, int kind);
int df_default_shape();

int df_large_shape();
int db_capacity_sub();
gp_status db_launch(Plan& pl, const double* v, double* out, int nrhs, bool user_order,
                    cudaStream_t s, int kind);

gp_status d1_prepare(Plan& pl) {
  static int attr_done = 0;
  if (!attr_done) {
    GPM_CUDA(d1_set_attr<0>());
    GPM_CUDA(d1_set_attr<1>());
    GPM_CUDA(d1_set_attr<2>());
    attr_done = 1;
  }
  int dev = 0, nsm = 0, coop = 0;
  GPM_CUDA(cudaGetDevice(&dev));
  GPM_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  GPM_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  if (!coop) return fail(GP_ERR_UNSUPPORTED, "device does not support cooperative launch");
  // fast path: one shared-memory chunk per CTA (apply_d1_fast.cu)
  int fast_grid = 0, cap = 0;
  if (pl.d1_force == 3) {   // testing knob: the reduce-then-scan path at any size
    const int64_t nsub = (pl.n + db_capacity_sub() - 1) / db_capacity_sub();
    pl.d1_grid = (int)nsub;
    pl.d1_chunk = db_capacity_sub();
    pl.d1_path = 3;
    GPM_TRY(pl.aggs.alloc(128 * 2 * (size_t)nsub));
    return GP_OK;
  }
  if (pl.d1_shape < 0) {
    // default shape; above its capacity (#SMs x 6912) the 31-point-per-thread shape keeps
    // the single-chunk kernel up to #SMs x 7936 (N = 2^20 and a little beyond)
    pl.d1_shape = df_default_shape();
    GPM_TRY(df_shape_info(pl.d1_shape, &cap, &fast_grid));
    const int large = df_large_shape();
    if (large >= 0 && pl.n > (int64_t)cap * fast_grid) pl.d1_shape = large;
  }
  GPM_TRY(df_shape_info(pl.d1_shape, &cap, &fast_grid));
  if (pl.d1_force != 2 && fast_grid > 0) {
    int64_t g = std::min<int64_t>(fast_grid, std::max<int64_t>(1, (pl.n + 1023) / 1024));
    int64_t chunk = ((pl.n + g - 1) / g + 3) & ~int64_t(3);   // multiple of 4 (TMA alignment)
    g = (pl.n + chunk - 1) / chunk;
    if (chunk <= cap && g <= fast_grid) {
      pl.d1_grid = (int)g;
      pl.d1_chunk = chunk;
      pl.d1_path = 1;
      GPM_TRY(pl.aggs.alloc(128 * 2 * 4 * (size_t)g));   // D1Pub [2 parities][4 replicas][g] (apply_d1_fast.cu)
      GPM_CUDA(cudaMemset(pl.aggs.ptr, 0, pl.aggs.bytes));
      GPM_TRY(pl.bar.alloc(64));
      GPM_CUDA(cudaMemset(pl.bar.ptr, 0, 64));
      if (getenv("GPM_D1_TIMING")) {
        GPM_TRY(pl.dbg.alloc(sizeof(unsigned long long) * 8 * (size_t)g));
        GPM_CUDA(cudaMemset(pl.dbg.ptr, 0, pl.dbg.bytes));
      }
      return GP_OK;
    }
  }
  if (pl.d1_force != 2) {
    // path 3: reduce-then-scan over sub-tiles in three plain launches (apply_d1_fast.cu
    // k_d1_big), any N, every nu and the lengthscale gradient
    const int64_t nsub = (pl.n + db_capacity_sub() - 1) / db_capacity_sub();
    if (nsub > (int64_t)1 << 30) return fail(GP_ERR_UNSUPPORTED, "d=1 problem too large");
    pl.d1_grid = (int)nsub;
    pl.d1_chunk = db_capacity_sub();
    pl.d1_path = 3;
    GPM_TRY(pl.aggs.alloc(128 * 2 * (size_t)nsub));   // sub-tile records + carries
    return GP_OK;
  }
  int occ = 0;
  GPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_d1_coop<2>, D1_BLOCK,
                                                         sizeof(D1Smem)));
  if (occ < 1) return fail(GP_ERR_CUDA, "d=1 kernel cannot be resident (shared memory)");
  const int64_t maxg = (int64_t)nsm * occ;
  int64_t g = std::min<int64_t>(maxg, std::max<int64_t>(1, (pl.n + 1023) / 1024));
  int64_t chunk = (pl.n + g - 1) / g;
  if (pl.d1_force == 2 && chunk <= D1_SUB) {
    // testing knob: force the multi-sub-tile path with tiny grids
    g = std::max<int64_t>(1, std::min<int64_t>(g, (pl.n + 3 * D1_SUB - 1) / (3 * D1_SUB)));
    chunk = (pl.n + g - 1) / g;
  }
  g = (pl.n + chunk - 1) / chunk;
  const int64_t nsub = (chunk + D1_SUB - 1) / D1_SUB;
  if (nsub > D1_MAXSUB)
    return fail(GP_ERR_UNSUPPORTED, "d=1 problem too large for one device (n=" +
                                        std::to_string(pl.n) + ")");
  pl.d1_grid = (int)g;
  pl.d1_chunk = chunk;
  pl.d1_path = 2;
  GPM_TRY(pl.aggs.alloc(sizeof(D1Agg) * (size_t)g * (1 + D1_MAXSUB)));
  GPM_TRY(pl.bar.alloc(64));
  GPM_CUDA(cudaMemset(pl.bar.ptr, 0, 64));
  return GP_OK;
}

gp_status d1_launch(Plan& pl, const double* v, double* out, int nrhs, bool user_order,
                    cudaStream_t s, int kind) {
  if (pl.d1_path == 1) return df_launch(pl, v, out, nrhs, user_order, s, kind);
  if (pl.d1_path == 3) return db_launch(pl, v, out, nrhs, user_order, s, kind);
  if (kind != 0)
    return fail(GP_ERR_UNSUPPORTED, "lengthscale-gradient MVM for d=1 needs n <= #SMs x 6912");
  if (pl.P > 2)
    return fail(GP_ERR_UNSUPPORTED, "nu >= 7/2 in d=1 needs n <= #SMs x 6912 (single-sub-tile path)");
  const int64_t vs = user_order ? pl.n_src : pl.n, os = user_order ? pl.n - pl.tgt_off : pl.n;
  for (int c = 0; c + 1 < nrhs; ++c)
    GPM_TRY(d1_launch(pl, v + c * vs, out + c * os, 1, user_order, s, 0));
  v += (nrhs - 1) * vs;
  out += (nrhs - 1) * os;
  D1Args a;
  a.ts = pl.t.as<double>();
  a.perm = user_order ? pl.perm.as<int>() : nullptr;
  a.v = v;
  a.out = out;
  a.n = pl.n;
  a.n_src = user_order ? pl.n_src : pl.n;
  a.tgt_off = user_order ? pl.tgt_off : 0;
  a.chunk = pl.d1_chunk;
  a.nsub = (int)((pl.d1_chunk + D1_SUB - 1) / D1_SUB);
  a.os2 = pl.os2;
  a.chunk_aggs = pl.aggs.as<D1Agg>();
  a.sub_aggs = pl.aggs.as<D1Agg>() + pl.d1_grid;
  a.bar = pl.bar.as<unsigned>();
  void* args[] = {&a};
  const void* fn = pl.P == 0 ? (const void*)k_d1_coop<0>
                   : pl.P == 1 ? (const void*)k_d1_coop<1> : (const void*)k_d1_coop<2>;
  GPM_CUDA(cudaLaunchCooperativeKernel(fn, dim3(pl.d1_grid), dim3(D1_BLOCK), args,
                                       sizeof(D1Smem), s));
  return GP_OK;
}

}  // namespace gpm
