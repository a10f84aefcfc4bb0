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
// k_d1_ov: the same scan with the grid-wide exchange taken off the critical path
// (measured on B200, tools/micro/{lat,xchg}.cu: one grid-wide exchange of per-CTA records
// costs ~2.5 us whatever the mechanism -- cg grid.sync, counter, per-slot flags -- and
// a 24-warp shuffle scan of (span, moments) is bound by the one-shuffle-per-clock pipe):
//   1. t (+perm) by bulk copies at launch; after griddepcontrol.wait v by bulk copies
//      (rank order) or the random gathers (user order);
//   2. pass 1: each thread's forward / backward aggregates (as k_d1_fast);
//   3. the CHUNK aggregate is a plain sum: each thread shifts its aggregates to the chunk's
//      reference points (one e^{-x} each, x from the sorted t directly), warp xor-sums,
//      one warp adds the warp sums in a fixed order (deterministic);
//   4. thread 0 publishes it and arrives on a monotone counter (red.release.gpu) -- a
//      split barrier: the wait comes only after steps 5-6;
//   5. meanwhile: the block scan (warp shuffles) for the within-chunk prefixes and
//   6. the local pass 2: both recurrences from the within-chunk prefixes only, storing
//      loc_j = u_j + read_F + read_B;
//   7. wait (thread 0 polls the counter with ld.acquire.gpu, then __syncthreads; the
//      records are read with ld.global.cg, i.e. from L2, the point of coherence), fold the
//      other chunks' records (4 replicas, one record per lane, 16-byte loads) into the
//      carries C_F, C_B;
//   8. carry pass: the carries' contribution at a point Delta after their reference is
//      e^{-Delta} sum_r beta_r Delta^r (beta from C once per CTA), Delta and e^{-Delta}
//      as running sums / products of the stored gaps: P + 1 FMAs per point and direction;
//      out = os2 (loc + both contributions), stored per warp (rank order) or scattered.
// Counter: bar[4..5] (u64) counts published columns x CTAs over the plan's life (zeroed at
// prepare); a CTA's record holds its own published-column count, so every CTA derives
// the same target (base + col + 1) x grid at kernel start (CUDA-graph safe: no host epoch).
// The dependent launch is released right after griddepcontrol.wait: its CTAs get an SM
// only when one of ours exits, and its own wait covers this whole grid.
constexpr int DF_REPL = 4;   // k_d1_ov record replicas (readers spread over 4 lines per record)

template <int P, int KIND, int BLOCK, int ITEMS, bool USER>
__global__ void __launch_bounds__(BLOCK, 1) k_d1_ov(DFArgs a) {
  constexpr int SUB = BLOCK * ITEMS;
  constexpr int NW = BLOCK / 32;
  constexpr int PT = BLOCK / DF_NPART;
  constexpr int PSZ = PT * ITEMS;
  constexpr int NM = 2 * (P + 1);   // chunk-sum values: forward and backward moments
  static_assert(PSZ % 4 == 0, "load parts must stay 16-byte aligned");
  static_assert(NW <= 32 && NM <= 32, "one warp adds the warp sums");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* s_t = reinterpret_cast<double*>(smem_raw);   // SUB + 8: t, then gaps
  double* s_u = s_t + SUB + 8;                         // SUB: u, then loc, then out
  double* s_e = s_u + SUB;                             // SUB: e^{-gap}
  int* s_pi = reinterpret_cast<int*>(s_e + SUB);       // SUB + 8 (user order)
  __shared__ uint64_t mbar[DF_NPART], mbar_v[DF_NPART];
  __shared__ double s_tab[64];
  constexpr int NSF = P + 3;
  __shared__ double s_wf[NW][NSF], s_wb[NW][NSF];
  __shared__ double s_wsum[NW][NM];
  __shared__ double s_beta[2][P + 1];
  __shared__ double s_part[2][16][NSF];   // warp partials of the record fold (grid <= 512)
  __shared__ unsigned long long s_base;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c0 = (int64_t)blockIdx.x * a.chunk;
  const int cnt = (int)max((int64_t)0, min(a.chunk, a.n - c0));
  const int G = gridDim.x, b = blockIdx.x;
  D1Pub* pub = reinterpret_cast<D1Pub*>(a.chunk_aggs);
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(a.bar + 8);

  DF_STAMP(0);
  fexp_table_init(s_tab);
  if (tid == 0) {
    for (int p = 0; p < DF_NPART; ++p) {
      mbar_init(&mbar[p], 1);
      mbar_init(&mbar_v[p], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid < DF_NPART && cnt > 0) {   // plan data: before griddepcontrol.wait
    const int lo = tid * PSZ, hi = min(cnt, lo + PSZ);
    if (lo < hi) {
      const unsigned nt = (unsigned)(((hi - lo) + 1) & ~1);   // padded plan arrays
      const unsigned np = (unsigned)(((hi - lo) + 3) & ~3);
      mbar_expect_tx(&mbar[tid], nt * 8 + (USER ? np * 4 : 0));
      tma_load_1d(s_t + lo, a.ts + c0 + lo, nt * 8, &mbar[tid]);
      if (USER) tma_load_1d(s_pi + lo, a.perm + c0 + lo, np * 4, &mbar[tid]);
    }
  }
  auto prefetch_v = [&](int col) {
    const int64_t per = (a.n_src + G - 1) / G;
    const int64_t lo = min((int64_t)b * per, a.n_src);
    const int64_t hi = min(lo + per, a.n_src);
    if (hi > lo) prefetch_l2_range(a.v + col * a.vstride + lo, (size_t)(hi - lo) * 8);
  };
  if (USER && a.prefetch && tid == 32) prefetch_v(0);
  const int j0 = tid * ITEMS;
  const int mypart = tid / PT;
  const bool part_live = mypart * PSZ < cnt;
  // reference points: chunk forward ref = its last point; chunk backward ref = the point
  // before its first point (t[0] for chunk 0: the first gap is 0); thread likewise
  double tprev = 0.0, tlast = 0.0, tcref = 0.0, tmy = 0.0;
  if (cnt > 0) {
    tlast = __ldg(a.ts + c0 + cnt - 1);
    tcref = c0 > 0 ? __ldg(a.ts + c0 - 1) : __ldg(a.ts);
    const int64_t gp = c0 + min(j0, cnt) - 1;
    tprev = gp >= 0 ? __ldg(a.ts + gp) : __ldg(a.ts);
    if (j0 >= cnt) tprev = tlast;
    tmy = j0 + ITEMS - 1 < cnt ? __ldg(a.ts + c0 + j0 + ITEMS - 1) : tlast;
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");   // v, records, counter of the previous apply
  // the next launch may be scheduled now: its CTAs only get an SM when one of ours exits,
  // and its griddepcontrol.wait still waits for this whole grid (memory included)
  asm volatile("griddepcontrol.launch_dependents;");
  if (tid == 0) {
    const unsigned long long b0 = __ldcg(&pub[b].epoch), b1 = __ldcg(&pub[DF_REPL * G + b].epoch);
    s_base = b0 > b1 ? b0 : b1;
  }
  const bool v_bulk = !USER && ((reinterpret_cast<uintptr_t>(a.v + c0) & 15) == 0) &&
                      (a.vstride % 2 == 0 || a.nrhs == 1);
  auto issue_v = [&](int col) {   // rank order: every column by bulk copy, or none
    const double* vcol = a.v + col * a.vstride + c0;
    if (v_bulk && tid < DF_NPART && cnt > 0) {
      const int lo = tid * PSZ, hi = min(cnt, lo + PSZ);
      const unsigned nu = (unsigned)((hi - lo) & ~1);   // never over-read v
      if (lo < hi) {
        fence_proxy_async_smem();
        mbar_expect_tx(&mbar_v[tid], nu * 8);
        if (nu) tma_load_1d(s_u + lo, vcol + lo, nu * 8, &mbar_v[tid]);
      }
    }
  };
  if (!USER) issue_v(0);
  if (part_live) mbar_wait(&mbar[mypart], 0);
  DF_STAMP(1);
  {   // independent per point: unrolled for ILP
    double tv[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) tv[k] = j0 + k < cnt ? s_t[j0 + k] : tlast;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const double dl = tv[k] - (k ? tv[k - 1] : tprev);   // neutral (0) past the chunk end
      s_t[j0 + k] = dl;
      s_e[j0 + k] = fexp_neg(dl, s_tab);
    }
  }
  // shifts of this thread's aggregates to the chunk references (plan data only)
  const double dF = tlast - tmy, eF = fexp_neg(dF, s_tab);
  const double dB = tprev - tcref, eB = fexp_neg(dB, s_tab);
  const double dC = tlast - tcref, eC = fexp_neg(dC, s_tab);
  __syncthreads();   // s_base

#pragma unroll 1
  for (int col = 0; col < a.nrhs; ++col) {
    const double* vcol = a.v + col * a.vstride;
    double* ocol = a.out + col * a.ostride;
    D1Pub* pubc = pub + (col & 1) * DF_REPL * G;   // [parity][replica][chunk]
    const unsigned long long mycount = s_base + (unsigned long long)col + 1ull;
    if (USER && a.prefetch && tid == 32 && col + 1 < a.nrhs) prefetch_v(col + 1);
    if (USER) {
      double uu[ITEMS];
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        const int j = j0 + k;
        const int pi = j < cnt ? s_pi[j] : INT_MAX;
        uu[k] = pi < a.n_src ? __ldg(vcol + pi) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) s_u[j0 + k] = uu[k];
    } else {
      if (v_bulk) {
        if (part_live) mbar_wait(&mbar_v[mypart], (unsigned)(col & 1));
        const int lo = mypart * PSZ, hi = min(cnt, lo + PSZ);
        if (lo < hi && ((hi - lo) & 1) && tid == (hi - 1) / ITEMS)   // odd tail element
          s_u[hi - 1] = __ldg(vcol + c0 + hi - 1);
      }
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        const int j = j0 + k;
        if (!v_bulk) s_u[j] = j < cnt ? __ldg(vcol + c0 + j) : 0.0;
        else if (j >= cnt) s_u[j] = 0.0;
      }
    }
    // ---- pass 1: this thread's aggregates by direct accumulation (short dependency
    // chains: a running span and e^{-span} per direction), forward from the suffix spans
    // (referenced at my last point), backward from the prefix spans (referenced at tprev)
    SF<P> F = sf_id<P>(), B = sf_id<P>();
    {
      double Dc = 0.0, Ec = 1.0, Ds = 0.0, Es = 1.0;
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        const int jb = j0 + k, jf = j0 + ITEMS - 1 - k;
        Dc += s_t[jb];
        Ec *= s_e[jb];
        double wb = s_u[jb] * Ec, wf = s_u[jf] * Es;
#pragma unroll
        for (int q = 0; q <= P; ++q) {
          B.M[q] += wb;
          F.M[q] += wf;
          wb *= Dc;
          wf *= Ds;
        }
        Ds += s_t[jf];
        Es *= s_e[jf];
      }
      F.D = B.D = Dc;
      F.E = B.E = Ec;
    }
    DF_STAMP(2);
    // ---- chunk aggregate = sum of the shifted thread aggregates (fixed order)
    {
      double m[NM];
#pragma unroll
      for (int q = 0; q <= P; ++q) {
        m[q] = F.M[q];
        m[P + 1 + q] = B.M[q];
      }
      advance<P>(m, dF, eF);
      advance<P>(m + P + 1, dB, eB);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int q = 0; q < NM; ++q) m[q] += __shfl_xor_sync(0xffffffffu, m[q], off);
      if (lane == 0)
#pragma unroll
        for (int q = 0; q < NM; ++q) s_wsum[warp][q] = m[q];
    }
    __syncthreads();
    if (warp == 0) {
      double s = 0.0;
      if (lane < NM)
#pragma unroll 1
        for (int w = 0; w < NW; ++w) s += s_wsum[w][lane];
      __syncwarp();
      if (lane < NM) s_wsum[0][lane] = s;
      __syncwarp();
      if (lane == 0) {   // publish (all replicas), then arrive: the release orders them
#pragma unroll 1
        for (int r = 0; r < DF_REPL; ++r) {
          D1Pub* me = pubc + r * G + b;
          me->v[0] = dC;
          me->v[1] = eC;
#pragma unroll
          for (int q = 0; q <= P; ++q) {
            me->v[2 + q] = s_wsum[0][q];
            me->v[8 + q] = s_wsum[0][P + 1 + q];
          }
          me->epoch = mycount;
        }
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
      }
    }
    DF_STAMP(3);
    // ---- overlapped with the exchange: block scan for the within-chunk prefixes
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
    if (warp < 2) {
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
    }
    __syncthreads();
    const SF<P> Fx = sf_cf<P>(sf_ld<P>(s_wf[warp]), fe);   // chunk ref -> my ref (forward)
    const SF<P> Bx = sf_cb<P>(be, sf_ld<P>(s_wb[warp]));   // my last point -> chunk last
    // ---- local pass 2: both recurrences (without the other chunks) interleaved, forward
    // over item k and backward over item ITEMS-1-k (two independent chains); an item's
    // first read waits in r1[] until the other direction reaches it, then
    // loc = u + read_F + read_B replaces u (about ITEMS values live at once, not 2 ITEMS)
    {
      double MF[P + 1], MB[P + 1], r1[ITEMS];
#pragma unroll
      for (int q = 0; q <= P; ++q) {
        MF[q] = Fx.M[q];
        MB[q] = Bx.M[q];
      }
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        const int kf = k, kb = ITEMS - 1 - k;
        advance<P>(MF, s_t[j0 + kf], s_e[j0 + kf]);
        const double rfk = readc0<P, KIND>(MF);
        const double uf = s_u[j0 + kf];
        MF[0] += uf;
        if (kb < kf) s_u[j0 + kf] = (KIND == 0 ? uf : 0.0) + (rfk + r1[kf]);   // B came first
        else if (kb > kf) r1[kf] = rfk;
        const double rbk = readc0<P, KIND>(MB);
        const double ub = s_u[j0 + kb];
        MB[0] += ub;
        advance<P>(MB, s_t[j0 + kb], s_e[j0 + kb]);
        if (kb < kf) s_u[j0 + kb] = (KIND == 0 ? ub : 0.0) + (r1[kb] + rbk);   // F came first
        else if (kb > kf) r1[kb] = rbk;
        else s_u[j0 + kb] = (KIND == 0 ? ub : 0.0) + (rfk + rbk);              // middle item
      }
    }
    // ---- wait for every chunk's record of this column
    if (tid == 0) {
      const unsigned long long target = mycount * (unsigned long long)G;
      while (ld_acquire_u64(ctr) < target) {
      }
    }
    __syncthreads();
    DF_STAMP(4);
    {   // one record per lane (replica b % DF_REPL), all loads in flight at once; each
        // warp folds its 32 records both ways, two threads fold the warp partials
      const int ngroups = (G + 31) / 32;
      const D1Pub* rep = pubc + (b % DF_REPL) * G;
#pragma unroll 1
      for (int grp = warp; grp < ngroups; grp += NW) {
        const int jj = grp * 32 + lane;
        const bool tf = jj < b, tb = jj > b && jj < G;
        SF<P> XF = sf_id<P>(), XB = sf_id<P>();
        if (tf || tb) {
          const double* o = rep[jj].v;
          const double2 de = __ldcg(reinterpret_cast<const double2*>(o));
          const double* m = o + (tf ? 2 : 8);
          double mv[P + 1];
#pragma unroll
          for (int q = 0; q + 1 <= P; q += 2) {
            const double2 w = __ldcg(reinterpret_cast<const double2*>(m + q));
            mv[q] = w.x;
            mv[q + 1] = w.y;
          }
          if ((P + 1) & 1) mv[P] = __ldcg(m + P);
          SF<P> Y;
          Y.D = de.x;
          Y.E = de.y;
#pragma unroll
          for (int q = 0; q <= P; ++q) Y.M[q] = mv[q];
          if (tf) XF = Y;
          else XB = Y;
        }
#pragma unroll 1
        for (int off = 1; off < 32; off <<= 1) {
          SF<P> YF = sf_shfl<P>(XF, off, false);
          SF<P> YB = sf_shfl<P>(XB, off, false);
          if (lane + off < 32) {
            XF = sf_cf<P>(XF, YF);
            XB = sf_cb<P>(XB, YB);
          }
        }
        if (lane == 0) {
          sf_st<P>(s_part[0][grp], XF);
          sf_st<P>(s_part[1][grp], XB);
        }
      }
      __syncthreads();
      if (tid < 2) {   // fold the partials in order; the carry's read polynomial coefficients
        const bool fw = tid == 0;
        SF<P> X = sf_id<P>();
#pragma unroll 1
        for (int gi = 0; gi < ngroups; ++gi) {
          const SF<P> y = sf_ld<P>(s_part[tid][gi]);
          X = fw ? sf_cf<P>(X, y) : sf_cb<P>(X, y);
        }
        // read(S(Delta) C) = e^{-Delta} sum_r beta_r Delta^r,
        // beta_r = sum_{q >= r} c_q C(q, q - r) C_{q - r}
#pragma unroll
        for (int r = 0; r <= P; ++r) {
          double br = 0.0;
#pragma unroll
          for (int q = r; q <= P; ++q) br = fma(rcoef(P, KIND, q) * binom(q, q - r), X.M[q - r], br);
          s_beta[tid][r] = br;
        }
      }
    }
    __syncthreads();
    DF_STAMP(5);
    // ---- carry pass and output
    {
      double bF[P + 1], bB[P + 1];
#pragma unroll
      for (int r = 0; r <= P; ++r) {
        bF[r] = s_beta[0][r];
        bB[r] = s_beta[1][r];
      }
      double D = Fx.D, E = Fx.E;
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        const int j = j0 + k;
        D += s_t[j];
        E *= s_e[j];
        double h = bF[P];
#pragma unroll
        for (int r = P - 1; r >= 0; --r) h = fma(h, D, bF[r]);
        s_u[j] = fma(E, h, s_u[j]);
      }
      D = Bx.D;
      E = Bx.E;
#pragma unroll
      for (int k = ITEMS - 1; k >= 0; --k) {
        const int j = j0 + k;
        double h = bB[P];
#pragma unroll
        for (int r = P - 1; r >= 0; --r) h = fma(h, D, bB[r]);
        const double val = a.os2 * fma(E, h, s_u[j]);
        D += s_t[j];
        E *= s_e[j];
        if (USER) {
          if (j < cnt) {
            const int pi = s_pi[j];
            if (pi >= a.tgt_off) ocol[pi - a.tgt_off] = val;
          }
        } else {
          s_u[j] = val;
        }
      }
    }
    if (!USER) {   // this warp's contiguous outputs
      __syncwarp();
      const int wb = warp * 32 * ITEMS;
      const int we = min(cnt, wb + 32 * ITEMS);
#pragma unroll 1
      for (int j = wb + lane; j < we; j += 32) ocol[c0 + j] = s_u[j];
    }
    if (col + 1 < a.nrhs) {
      __syncthreads();   // s_u / s_beta / s_wsum of this column consumed
      if (!USER) issue_v(col + 1);
    }
  }   // column loop
  if (a.dbg) {
    __syncthreads();
    DF_STAMP(6);
  }
}

// ---------------------------------------------------------------------------
// k_d1_big: d = 1 above the single-chunk capacity (N > #SMs x 7936).  A reduce-then-scan
// in three plain launches (no cooperative residency, any N): sub-tiles of BLOCK x ITEMS
// sorted points, one per CTA,
//   MODE 1: load, gaps / e^{-gap}, pass 1, the sub-tile aggregate (as k_d1_ov's chunk sum)
//           -> rec[sub]; user order also stores the gathered u in rank order (ur);
//   k_d1_big_scan: one CTA folds the records into each sub-tile's carries (exclusive,
//           forward and backward) -> carr[sub];
//   MODE 2: reload t and u (rank order: v; user order: ur, coalesced), gaps, pass 1, block
//           scan, local pass 2, carry pass with the sub-tile's carries, output.
// Model traffic: rank order 40 B/pt (t and v twice, out), user order 56 B/pt (t twice, perm
// twice, the gather, ur written and read, out) -- against 24 / 28 B/pt for the single-chunk
// kernel, which keeps the chunk resident between the passes.
struct D1Carr {   // 128 B: forward carry moments [0..5], backward [8..13]
  double m[16];
};

template <int P, int KIND, int BLOCK, int ITEMS, bool USER, int MODE>
__global__ void __launch_bounds__(BLOCK, BLOCK >= 256 ? 1 : (ITEMS > 16 ? 2 : 4)) k_d1_big(DFArgs a, double* ur, D1Pub* rec,
                                                     const D1Carr* carr) {
  constexpr int SUB = BLOCK * ITEMS;
  constexpr int NW = BLOCK / 32;
  constexpr int PT = BLOCK / DF_NPART;
  constexpr int PSZ = PT * ITEMS;
  constexpr int NM = 2 * (P + 1);
  static_assert(PSZ % 4 == 0, "load parts must stay 16-byte aligned");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* s_t = reinterpret_cast<double*>(smem_raw);   // SUB + 8: t, then gaps
  double* s_u = s_t + SUB + 8;                         // SUB: u, then loc, then out
  double* s_e = s_u + SUB;                             // SUB: e^{-gap}
  int* s_pi = reinterpret_cast<int*>(s_e + SUB);       // SUB + 8 (user order)
  __shared__ uint64_t mbar[DF_NPART], mbar_v[DF_NPART];
  __shared__ double s_tab[64];
  constexpr int NSF = P + 3;
  __shared__ double s_wf[NW][NSF], s_wb[NW][NSF];
  __shared__ double s_wsum[NW][NM];
  __shared__ double s_beta[2][P + 1];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c0 = (int64_t)blockIdx.x * SUB;
  const int cnt = (int)max((int64_t)0, min((int64_t)SUB, a.n - c0));
  const bool need_pi = USER;   // gathers (pass 1) / scatter (pass 2)
  fexp_table_init(s_tab);
  if (tid == 0) {
    for (int p = 0; p < DF_NPART; ++p) {
      mbar_init(&mbar[p], 1);
      mbar_init(&mbar_v[p], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // the u source of this pass in rank order: v (rank order) or ur (user order, pass 2)
  const double* urank = USER ? ur : a.v;
  const bool u_bulk = (!USER || MODE == 2) && ((reinterpret_cast<uintptr_t>(urank + c0) & 15) == 0);
  if (tid < DF_NPART && cnt > 0) {
    const int lo = tid * PSZ, hi = min(cnt, lo + PSZ);
    if (lo < hi) {
      const unsigned nt = (unsigned)(((hi - lo) + 1) & ~1);   // padded plan arrays
      const unsigned np = (unsigned)(((hi - lo) + 3) & ~3);
      mbar_expect_tx(&mbar[tid], nt * 8 + (need_pi ? np * 4 : 0));
      tma_load_1d(s_t + lo, a.ts + c0 + lo, nt * 8, &mbar[tid]);
      if (need_pi) tma_load_1d(s_pi + lo, a.perm + c0 + lo, np * 4, &mbar[tid]);
      if (u_bulk) {
        const unsigned nu = (unsigned)((hi - lo) & ~1);
        mbar_expect_tx(&mbar_v[tid], nu * 8);
        if (nu) tma_load_1d(s_u + lo, urank + c0 + lo, nu * 8, &mbar_v[tid]);
      }
    }
  }
  const int j0 = tid * ITEMS;
  const int mypart = tid / PT;
  const bool part_live = mypart * PSZ < cnt;
  double tprev = 0.0, tlast = 0.0, tcref = 0.0, tmy = 0.0;
  if (cnt > 0) {
    tlast = __ldg(a.ts + c0 + cnt - 1);
    tcref = c0 > 0 ? __ldg(a.ts + c0 - 1) : __ldg(a.ts);
    const int64_t gp = c0 + min(j0, cnt) - 1;
    tprev = gp >= 0 ? __ldg(a.ts + gp) : __ldg(a.ts);
    if (j0 >= cnt) tprev = tlast;
    tmy = j0 + ITEMS - 1 < cnt ? __ldg(a.ts + c0 + j0 + ITEMS - 1) : tlast;
  }
  if (part_live) mbar_wait(&mbar[mypart], 0);
  {
    double tp = tprev;
#pragma unroll 9
    for (int k = 0; k < ITEMS; ++k) {
      const double t = j0 + k < cnt ? s_t[j0 + k] : tlast;
      const double dl = t - tp;
      tp = t;
      s_t[j0 + k] = dl;
      s_e[j0 + k] = fexp_neg(dl, s_tab);
    }
  }
  // u of my points
  if (USER && MODE == 1) {
    double uu[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const int j = j0 + k;
      const int pi = j < cnt ? s_pi[j] : INT_MAX;
      uu[k] = pi < a.n_src ? __ldg(a.v + pi) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) s_u[j0 + k] = uu[k];
    __syncwarp();   // this warp's u, stored in rank order (coalesced) for pass 2
    const int wb = warp * 32 * ITEMS, we = min(cnt, wb + 32 * ITEMS);
#pragma unroll 1
    for (int j = wb + lane; j < we; j += 32) ur[c0 + j] = s_u[j];
  } else {
    if (u_bulk) {
      if (part_live) mbar_wait(&mbar_v[mypart], 0);
      const int lo = mypart * PSZ, hi = min(cnt, lo + PSZ);
      if (lo < hi && ((hi - lo) & 1) && tid == (hi - 1) / ITEMS) s_u[hi - 1] = __ldg(urank + c0 + hi - 1);
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const int j = j0 + k;
      if (!u_bulk) s_u[j] = j < cnt ? __ldg(urank + c0 + j) : 0.0;
      else if (j >= cnt) s_u[j] = 0.0;
    }
  }
  // pass 1: my aggregates (direct accumulation, as k_d1_ov)
  SF<P> F = sf_id<P>(), B = sf_id<P>();
  {
    double Dc = 0.0, Ec = 1.0, Ds = 0.0, Es = 1.0;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const int jb = j0 + k, jf = j0 + ITEMS - 1 - k;
      Dc += s_t[jb];
      Ec *= s_e[jb];
      double wb = s_u[jb] * Ec, wf = s_u[jf] * Es;
#pragma unroll
      for (int q = 0; q <= P; ++q) {
        B.M[q] += wb;
        F.M[q] += wf;
        wb *= Dc;
        wf *= Ds;
      }
      Ds += s_t[jf];
      Es *= s_e[jf];
    }
    F.D = B.D = Dc;
    F.E = B.E = Ec;
  }
  if (MODE == 1) {   // the sub-tile aggregate: sum of the shifted thread aggregates
    const double dF = tlast - tmy, eF = fexp_neg(dF, s_tab);
    const double dB = tprev - tcref, eB = fexp_neg(dB, s_tab);
    double m[NM];
#pragma unroll
    for (int q = 0; q <= P; ++q) {
      m[q] = F.M[q];
      m[P + 1 + q] = B.M[q];
    }
    advance<P>(m, dF, eF);
    advance<P>(m + P + 1, dB, eB);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
      for (int q = 0; q < NM; ++q) m[q] += __shfl_xor_sync(0xffffffffu, m[q], off);
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < NM; ++q) s_wsum[warp][q] = m[q];
    __syncthreads();
    if (warp == 0) {
      double s = 0.0;
      if (lane < NM)
#pragma unroll 1
        for (int w = 0; w < NW; ++w) s += s_wsum[w][lane];
      D1Pub* me = rec + blockIdx.x;
      if (lane < P + 1) me->v[2 + lane] = s;
      else if (lane < NM) me->v[8 + lane - (P + 1)] = s;
      if (lane == 0) {
        const double dC = tlast - tcref;
        me->v[0] = dC;
        me->v[1] = fexp_neg(dC, s_tab);
      }
    }
    return;
  }
  // ---- MODE 2: block scan, local pass 2, carry pass, output
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
  if (warp < 2) {
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
    if (lane == 0) {   // the carries' read polynomial coefficients (see k_d1_ov)
      const D1Carr& c = carr[blockIdx.x];
#pragma unroll
      for (int r = 0; r <= P; ++r) {
        double br = 0.0;
#pragma unroll
        for (int q = r; q <= P; ++q)
          br = fma(rcoef(P, KIND, q) * binom(q, q - r), __ldg(&c.m[(fw ? 0 : 8) + q - r]), br);
        s_beta[warp][r] = br;
      }
    }
  }
  __syncthreads();
  const SF<P> Fx = sf_cf<P>(sf_ld<P>(s_wf[warp]), fe);
  const SF<P> Bx = sf_cb<P>(be, sf_ld<P>(s_wb[warp]));
  {
    double MF[P + 1], MB[P + 1], r1[ITEMS];
#pragma unroll
    for (int q = 0; q <= P; ++q) {
      MF[q] = Fx.M[q];
      MB[q] = Bx.M[q];
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const int kf = k, kb = ITEMS - 1 - k;
      advance<P>(MF, s_t[j0 + kf], s_e[j0 + kf]);
      const double rfk = readc0<P, KIND>(MF);
      const double uf = s_u[j0 + kf];
      MF[0] += uf;
      if (kb < kf) s_u[j0 + kf] = (KIND == 0 ? uf : 0.0) + (rfk + r1[kf]);
      else if (kb > kf) r1[kf] = rfk;
      const double rbk = readc0<P, KIND>(MB);
      const double ub = s_u[j0 + kb];
      MB[0] += ub;
      advance<P>(MB, s_t[j0 + kb], s_e[j0 + kb]);
      if (kb < kf) s_u[j0 + kb] = (KIND == 0 ? ub : 0.0) + (r1[kb] + rbk);
      else if (kb > kf) r1[kb] = rbk;
      else s_u[j0 + kb] = (KIND == 0 ? ub : 0.0) + (rfk + rbk);
    }
  }
  {
    double bF[P + 1], bB[P + 1];
#pragma unroll
    for (int r = 0; r <= P; ++r) {
      bF[r] = s_beta[0][r];
      bB[r] = s_beta[1][r];
    }
    double D = Fx.D, E = Fx.E;
#pragma unroll 9
    for (int k = 0; k < ITEMS; ++k) {
      const int j = j0 + k;
      D += s_t[j];
      E *= s_e[j];
      double h = bF[P];
#pragma unroll
      for (int r = P - 1; r >= 0; --r) h = fma(h, D, bF[r]);
      s_u[j] = fma(E, h, s_u[j]);
    }
    D = Bx.D;
    E = Bx.E;
#pragma unroll 9
    for (int k = ITEMS - 1; k >= 0; --k) {
      const int j = j0 + k;
      double h = bB[P];
#pragma unroll
      for (int r = P - 1; r >= 0; --r) h = fma(h, D, bB[r]);
      const double val = a.os2 * fma(E, h, s_u[j]);
      D += s_t[j];
      E *= s_e[j];
      if (USER) {
        if (j < cnt) {
          const int pi = s_pi[j];
          if (pi >= a.tgt_off) a.out[pi - a.tgt_off] = val;
        }
      } else {
        s_u[j] = val;
      }
    }
  }
  if (!USER) {
    __syncwarp();
    const int wb = warp * 32 * ITEMS, we = min(cnt, wb + 32 * ITEMS);
#pragma unroll 1
    for (int j = wb + lane; j < we; j += 32) a.out[c0 + j] = s_u[j];
  }
}

// the sub-tile carries: exclusive forward and backward folds of the sub-tile records
template <int P>
__global__ void __launch_bounds__(1024, 1) k_d1_big_scan(const D1Pub* rec, D1Carr* carr, int nsub) {
  __shared__ double s_w[2][32][P + 3];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = (nsub + 1023) / 1024;
  const int r0 = min(tid * per, nsub), r1 = min(r0 + per, nsub);
  auto ld = [&](int r, bool fw) {
    SF<P> s;
    s.D = rec[r].v[0];
    s.E = rec[r].v[1];
#pragma unroll
    for (int q = 0; q <= P; ++q) s.M[q] = rec[r].v[(fw ? 2 : 8) + q];
    return s;
  };
  SF<P> XF = sf_id<P>(), XB = sf_id<P>();
#pragma unroll 1
  for (int r = r0; r < r1; ++r) {
    XF = sf_cf<P>(XF, ld(r, true));
    XB = sf_cb<P>(XB, ld(r, false));
  }
  // block exclusive scans: forward (prefix over threads), backward (suffix)
  SF<P> fi = XF, bi = XB;
#pragma unroll 1
  for (int off = 1; off < 32; off <<= 1) {
    SF<P> l = sf_shfl<P>(fi, off, true);
    SF<P> r = sf_shfl<P>(bi, off, false);
    if (lane >= off) fi = sf_cf<P>(l, fi);
    if (lane + off < 32) bi = sf_cb<P>(bi, r);
  }
  if (lane == 31) sf_st<P>(s_w[0][warp], fi);
  if (lane == 0) sf_st<P>(s_w[1][warp], bi);
  SF<P> fe = sf_shfl<P>(fi, 1, true);
  SF<P> be = sf_shfl<P>(bi, 1, false);
  if (lane == 0) fe = sf_id<P>();
  if (lane == 31) be = sf_id<P>();
  __syncthreads();
  if (warp < 2) {
    const bool fw = warp == 0;
    SF<P> x = sf_ld<P>(s_w[fw ? 0 : 1][lane]);
#pragma unroll 1
    for (int off = 1; off < 32; off <<= 1) {
      SF<P> y = sf_shfl<P>(x, off, fw);
      if (fw && lane >= off) x = sf_cf<P>(y, x);
      if (!fw && lane + off < 32) x = sf_cb<P>(x, y);
    }
    SF<P> xe = sf_shfl<P>(x, 1, fw);
    if ((fw && lane == 0) || (!fw && lane == 31)) xe = sf_id<P>();
    __syncwarp();
    sf_st<P>(s_w[fw ? 0 : 1][lane], xe);
  }
  __syncthreads();
  SF<P> CF = sf_cf<P>(sf_ld<P>(s_w[0][warp]), fe);
  SF<P> CB = sf_cb<P>(be, sf_ld<P>(s_w[1][warp]));
#pragma unroll 1
  for (int r = r0; r < r1; ++r) {
#pragma unroll
    for (int q = 0; q <= P; ++q) carr[r].m[q] = CF.M[q];
    CF = sf_cf<P>(CF, ld(r, true));
  }
#pragma unroll 1
  for (int r = r1 - 1; r >= r0; --r) {
#pragma unroll
    for (int q = 0; q <= P; ++q) carr[r].m[8 + q] = CB.M[q];
    CB = sf_cb<P>(ld(r, false), CB);
  }
}

template <int P, int KIND, bool USER, int BLK, int IT>
static cudaError_t db_launch3(const DFArgs& a, double* ur, D1Pub* rec, D1Carr* carr, int nsub,
                              cudaStream_t s) {
  const size_t smem = sizeof(double) * (3 * BLK * IT + 8) +
                      (USER ? sizeof(int) * (BLK * IT + 8) : 0);
  auto k1 = k_d1_big<P, KIND, BLK, IT, USER, 1>;
  auto k2 = k_d1_big<P, KIND, BLK, IT, USER, 2>;
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
  if ((e = cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
  k1<<<nsub, BLK, smem, s>>>(a, ur, rec, carr);
  k_d1_big_scan<P><<<1, 1024, 0, s>>>(rec, carr, nsub);
  k2<<<nsub, BLK, smem, s>>>(a, ur, rec, carr);
  return cudaGetLastError();
}

// k_d1_big sub-tile shapes (BLOCK x ITEMS): 0 = 256 x 27 (one CTA per SM), 1 = 128 x 27 (two),
// 2 = 128 x 13 (four); the default by measurement (profiles/r01_notes.md)
static int db_shape() {
  static int sh = -1;
  if (sh < 0) {
    sh = 1;
    if (const char* e = getenv("GPM_DB_SHAPE")) sh = std::max(0, std::min(2, atoi(e)));
  }
  return sh;
}

template <int P, int KIND>
static cudaError_t db_launch2(bool user, const DFArgs& a, double* ur, D1Pub* rec, D1Carr* carr,
                              int nsub, cudaStream_t s) {
  switch (db_shape()) {
    case 0: return user ? db_launch3<P, KIND, true, 256, 27>(a, ur, rec, carr, nsub, s)
                        : db_launch3<P, KIND, false, 256, 27>(a, ur, rec, carr, nsub, s);
    case 2: return user ? db_launch3<P, KIND, true, 128, 13>(a, ur, rec, carr, nsub, s)
                        : db_launch3<P, KIND, false, 128, 13>(a, ur, rec, carr, nsub, s);
    default: return user ? db_launch3<P, KIND, true, 128, 27>(a, ur, rec, carr, nsub, s)
                         : db_launch3<P, KIND, false, 128, 27>(a, ur, rec, carr, nsub, s);
  }
}

int db_capacity_sub() { return db_shape() == 0 ? 256 * 27 : db_shape() == 2 ? 128 * 13 : 128 * 27; }

// path 3: d = 1 above the single-chunk capacity; columns one at a time (three launches each)
gp_status db_launch(Plan& pl, const double* v, double* out, int nrhs, bool user_order,
                    cudaStream_t s, int kind) {
  const int nsub = (int)((pl.n + db_capacity_sub() - 1) / db_capacity_sub());
  D1Pub* rec = reinterpret_cast<D1Pub*>(pl.aggs.ptr);
  D1Carr* carr = reinterpret_cast<D1Carr*>(rec + nsub);
  const int64_t vs = user_order ? pl.n_src : pl.n, os = user_order ? pl.n - pl.tgt_off : pl.n;
  for (int c = 0; c < nrhs; ++c) {
    DFArgs a = {};
    a.ts = pl.t.as<double>();
    a.perm = pl.perm.as<int>();
    a.v = v + c * vs;
    a.out = out + c * os;
    a.n = pl.n;
    a.n_src = user_order ? pl.n_src : pl.n;
    a.tgt_off = user_order ? pl.tgt_off : 0;
    a.chunk = db_capacity_sub();
    a.user_order = user_order ? 1 : 0;
    a.nrhs = 1;
    a.vstride = vs;
    a.ostride = os;
    a.os2 = pl.os2;
    double* ur = pl.w.as<double>();
    const int key = kind * 5 + pl.P;
    cudaError_t e = cudaErrorInvalidValue;
    switch (key) {
      case 0: e = db_launch2<0, 0>(user_order, a, ur, rec, carr, nsub, s); break;
      case 1: e = db_launch2<1, 0>(user_order, a, ur, rec, carr, nsub, s); break;
      case 2: e = db_launch2<2, 0>(user_order, a, ur, rec, carr, nsub, s); break;
      case 3: e = db_launch2<3, 0>(user_order, a, ur, rec, carr, nsub, s); break;
      case 4: e = db_launch2<4, 0>(user_order, a, ur, rec, carr, nsub, s); break;
      case 5: e = db_launch2<1, 1>(user_order, a, ur, rec, carr, nsub, s); break;
      case 6: e = db_launch2<2, 1>(user_order, a, ur, rec, carr, nsub, s); break;
      case 7: e = db_launch2<3, 1>(user_order, a, ur, rec, carr, nsub, s); break;
      case 8: e = db_launch2<4, 1>(user_order, a, ur, rec, carr, nsub, s); break;
      case 9: e = db_launch2<5, 1>(user_order, a, ur, rec, carr, nsub, s); break;
    }
    GPM_CUDA(e);
  }
  return GP_OK;
}

// ---------------------------------------------------------------------------
// Host side.  Shapes (BLOCK, ITEMS): k_d1_fast 0 = (512, 15), 1 = (640, 11), 2 = (768, 9),
// 3 = (1024, 7); k_d1_ov 4 = (256, 27), 5 = (256, 31) (chosen above 4's capacity), 6 = (512, 15), 7 = (128, 27) (two CTAs
// per SM).
// The default is chosen by measurement.
template <int BLOCK, int ITEMS>
static size_t df_smem() {
  constexpr int SUB = BLOCK * ITEMS;
  return sizeof(double) * (3 * SUB + 8) + sizeof(int) * (SUB + 8);
}

struct DFShape {
  int block, items;
  // [user order][KIND * 5 + p]: KIND 0 moment order p, KIND 1 moment order p + 1
  const void* fn[2][10];
  size_t smem[2];   // [user order]: k_d1_ov in rank order has no permutation in smem
};

template <int BLOCK, int ITEMS>
static DFShape make_shape() {
  DFShape s;
  s.block = BLOCK;
  s.items = ITEMS;
  const void* f[10] = {
      (const void*)k_d1_fast<0, 0, BLOCK, ITEMS>, (const void*)k_d1_fast<1, 0, BLOCK, ITEMS>,
      (const void*)k_d1_fast<2, 0, BLOCK, ITEMS>, (const void*)k_d1_fast<3, 0, BLOCK, ITEMS>,
      (const void*)k_d1_fast<4, 0, BLOCK, ITEMS>, (const void*)k_d1_fast<1, 1, BLOCK, ITEMS>,
      (const void*)k_d1_fast<2, 1, BLOCK, ITEMS>, (const void*)k_d1_fast<3, 1, BLOCK, ITEMS>,
      (const void*)k_d1_fast<4, 1, BLOCK, ITEMS>, (const void*)k_d1_fast<5, 1, BLOCK, ITEMS>};
  for (int p = 0; p < 10; ++p) s.fn[0][p] = s.fn[1][p] = f[p];
  s.smem[0] = s.smem[1] = df_smem<BLOCK, ITEMS>();
  return s;
}

template <int BLOCK, int ITEMS, bool USER>
static void flag_fns(const void** f) {
  f[0] = (const void*)k_d1_ov<0, 0, BLOCK, ITEMS, USER>;
  f[1] = (const void*)k_d1_ov<1, 0, BLOCK, ITEMS, USER>;
  f[2] = (const void*)k_d1_ov<2, 0, BLOCK, ITEMS, USER>;
  f[3] = (const void*)k_d1_ov<3, 0, BLOCK, ITEMS, USER>;
  f[4] = (const void*)k_d1_ov<4, 0, BLOCK, ITEMS, USER>;
  f[5] = (const void*)k_d1_ov<1, 1, BLOCK, ITEMS, USER>;
  f[6] = (const void*)k_d1_ov<2, 1, BLOCK, ITEMS, USER>;
  f[7] = (const void*)k_d1_ov<3, 1, BLOCK, ITEMS, USER>;
  f[8] = (const void*)k_d1_ov<4, 1, BLOCK, ITEMS, USER>;
  f[9] = (const void*)k_d1_ov<5, 1, BLOCK, ITEMS, USER>;
}
template <int BLOCK, int ITEMS>
static DFShape make_shape_flag() {
  DFShape s;
  s.block = BLOCK;
  s.items = ITEMS;
  flag_fns<BLOCK, ITEMS, false>(s.fn[0]);
  flag_fns<BLOCK, ITEMS, true>(s.fn[1]);
  s.smem[0] = sizeof(double) * (3 * BLOCK * ITEMS + 8);   // t, u, e (a larger L1 carve-out)
  s.smem[1] = df_smem<BLOCK, ITEMS>();
  return s;
}

constexpr int DF_NSHAPE = 8;
static DFShape g_shapes[DF_NSHAPE];
static int g_shapes_ready = 0;
static int g_default_shape = 4;   // k_d1_ov 256 x 27: best measured (tools/sweep_d1.py)

static gp_status df_init() {
  if (g_shapes_ready) return GP_OK;
  g_shapes[0] = make_shape<512, 15>();
  g_shapes[1] = make_shape<640, 11>();
  g_shapes[2] = make_shape<768, 9>();
  g_shapes[3] = make_shape<1024, 7>();
  g_shapes[4] = make_shape_flag<256, 27>();
  g_shapes[5] = make_shape_flag<256, 31>();   // larger chunks: N up to #SMs x 7936
  g_shapes[6] = make_shape_flag<512, 15>();
  g_shapes[7] = make_shape_flag<128, 27>();   // 97 KB: two CTAs per SM
  for (auto& s : g_shapes)
    for (int u = 0; u < 2; ++u)
      for (int p = 0; p < 10; ++p)
        GPM_CUDA(cudaFuncSetAttribute(s.fn[u][p], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)s.smem[u]));
  if (const char* e = getenv("GPM_D1_SHAPE"))
    g_default_shape = std::max(0, std::min(DF_NSHAPE - 1, atoi(e)));
  g_shapes_ready = 1;
  return GP_OK;
}

int df_default_shape() { return g_default_shape; }
int df_large_shape() { return g_default_shape == 4 ? 5 : -1; }

// capacity per CTA and max co-resident grid for a shape
gp_status df_shape_info(int shape, int* capacity, int* max_grid) {
  GPM_TRY(df_init());
  const DFShape& s = g_shapes[shape];
  int dev = 0, nsm = 0, occ = 0;
  GPM_CUDA(cudaGetDevice(&dev));
  GPM_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  GPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, s.fn[1][2], s.block, s.smem[1]));
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
  cfg.dynamicSmemBytes = sh.smem[user_order ? 1 : 0];
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pl.d1_pdl ? 2 : 1;
  void* args[] = {&a};
  GPM_CUDA(cudaLaunchKernelExC(&cfg, sh.fn[user_order ? 1 : 0][kind * 5 + pl.P], args));
  return GP_OK;
}

}  // namespace gpm
