// apply_level.cu -- d >= 2 hot path: the multivariate ECDF decomposition of
// P:459-509 [Props 1-2] computed by Bentley's divide and conquer over the stored
// level structure (P:531-539 [§2.2.3]) in the overflow-free moment basis.
//
// One "pass" = one level of the D&C (d = 2: level l over x1-ranks; d = 3: outer level
// l1 over x1-ranks x inner level l2 over the node's x2-order).  Within a pass the
// positions are grouped in aligned segments of 2^lseg points (the D&C nodes), each
// sorted by the last coordinate.  Every pair i != j is counted exactly once, at the
// pass where it is split, in one scan direction:
//   source i injects u_i alpha_i^q e^{-alpha_i} into channel c_i (its split sides),
//   target j reads channel NCH-1-c_j with offset beta_j = alpha_j,
// where alpha = |t1 - m1| (+ |t2 - m2| for d = 3) is the distance to the node's split
// reference.  This realises the 2^d orthant CDFs F(delta z, delta; delta x, w_p)
// of eq L1_decomposition / product_decomposition without forming the overflowing
// weights of eq matern_weights (R5).
//
// B200 layout: 128 threads x 8 consecutive positions of a 1024-position tile
// per CTA; nodes are aligned power-of-two position blocks, so node boundaries fall between
// threads and the scans need no per-position flags.  Launch structure per apply:
//   k_pack: rank-order point records (t1, t2, t3, u);
//   d = 2: k_low2 / k_low2m -- near field (pairs split at levels <= lb) + levels lb < l <= 10
//          of each tile (point data staged once in shared memory), run in parts (blockIdx.z:
//          near-field partner slices, then groups of levels; one output slot per part);
//   d = 3: k_low3 -- the same for (l1 <= 10, all l2); k_mid3 -- every l1 > 10 with l2 <= 10
//          (one launch, blockIdx.z = l1);
//   carried passes (nodes longer than a tile): k_cp<1> tile aggregates, k_cp_carry (exclusive
//          scan of a node's tile aggregates), k_cp<2> apply; persistent over all passes with a
//          bulk-copy pipeline of setup-staged tiles;
//   k_epilogue (apply.cu): fixed-order sum of the per-pass slots, scale, scatter.
// Product forms: d = 2 carries (P+1)^2 mixed moments per channel (Alg PROD); d = 3, and the
// gradients the mixed state cannot hold, run the (P+1)-moment engine once per separated
// sub-pass (Alg SEP, algebra.cuh): level_apply in the tile kernels, extra columns in k_cp.
#include <algorithm>
#include <vector>

#include "algebra.cuh"
#include "fexp.cuh"
#include "internal.h"
#include "tma.cuh"

// This file is compiled four times (build.py: apply_level.cu and apply_level_p{1,2,3}.cu, which
// only set GPM_LEVEL_PART and include it) so that the template instantiations build in
// parallel: part 0 = the non-template host code and the d = 2 value algebras, 1 = the d = 2
// gradients, 2 = the d = 3 value algebras, 3 = the d = 3 gradients.
#ifndef GPM_LEVEL_PART
#define GPM_LEVEL_PART 0
#endif

namespace gpm {

int level_nparts(const Plan& pl);
bool level_p3(const Plan& pl);
int level_nab(const Plan& pl);
int level_phases(const Plan& pl, int kind);
int64_t hp_item_count(int64_t n, int d);
gp_status level_passes_p1(Plan& pl, int nrhs, cudaStream_t s, int* launches, int kind, int phase);
gp_status level_passes_p2(Plan& pl, int nrhs, cudaStream_t s, int* launches, int kind, int phase);
gp_status level_passes_p3(Plan& pl, int nrhs, cudaStream_t s, int* launches, int kind, int phase);

constexpr int LV_LOGTILE = 10;
constexpr int LV_TILE = 1 << LV_LOGTILE;

// Point arrays of the fused kernels (tile-local point index).
struct LvPoints {
  double u[LV_TILE], t1[LV_TILE], t2[LV_TILE], t3[LV_TILE], acc[LV_TILE];
  int o2[LV_TILE];     // d = 3: ord2[l1] tile (local ranks) / global ranks (mid kernel)
};

// Packed per-point record (rank order), rebuilt per apply by k_pack: one random access
// touches one 32-byte sector instead of four.
struct __align__(32) Pt4 {
  double t1, t2, t3, u;
};

struct LvArgs {
  const Pt4* pts;      // [n] packed points (rank order)
  int lb, lb2;         // near-field block log2 sizes: low (x1 ranks) / mid (ord2[l1] positions)
  const int* ord2;     // [L][n]
  const int* ord3;     // [L(L+1)/2][n]
  const double* t1;
  const double* t2;
  const double* t3;
  const double* u;     // rank-order input
  double* acc;         // rank-order accumulator
  LvAgg* aggs;
  int64_t n;
  int L;
  // single-pass kernels
  const int* ord;      // this pass's order
  const int* ord2l1;   // d = 3: ord2[l1]
  int lseg, l1, ntiles;
  int64_t n_act;
  int mode;            // 2 or 3 (dimension)
  int64_t agg_stride;  // LvAgg records per right-hand side
  double* part;        // [nparts][n] per-pass contributions (rank order), summed in order
  int npass;           // carried passes (their part slots come first, then d=3 mid levels)
  int64_t part_stride; // doubles per right-hand side in part
  int tile0;           // sharded applies (gp_kmvm_partial): first tile of the tile kernels
  int low_slot0;       // part slot of the fused low kernels' part 1 (part 0 writes acc)
};

// right-hand side handled by this CTA (blockIdx.y): offset the per-column buffers
__device__ __forceinline__ void lv_col(LvArgs& g) {
  const int64_t c = blockIdx.y;
  g.pts += c * g.n;
  g.acc += c * g.n;
  g.aggs += c * g.agg_stride;
  g.part += c * g.part_stride;
}

__device__ __forceinline__ int ord3_index(int l1, int l2) { return (l1 - 1) * l1 / 2 + (l2 - 1); }

// sum_q c_q s^q of a read profile (rcoef: Matern a_q for KIND 0, gradient b_q for KIND 1)
template <int PM, int KIND>
__device__ __forceinline__ double kpoly(double s) {
  double poly = rcoef(PM, KIND, PM);
#pragma unroll
  for (int q = PM - 1; q >= 0; --q) poly = fma(poly, s, rcoef(PM, KIND, q));
  return poly;
}

// Kernel value from per-dimension distances d_k = |t_ik - t_jk| (scaled coordinates):
// L1: k(d1+d2(+d3)); product (d = 2): k(d1) k(d2); k(s) = sum_q a_q s^q e^{-s}.
template <class A, int D>
__device__ __forceinline__ double kval(double d1, double d2, double d3, const double* tab) {
  constexpr int P = A::P;
  if constexpr (A::SEP == 1) {   // product form, d = 3 (P:416 [eq product_kernel])
    const double e = fexp_neg((d1 + d2) + d3, tab);
    return e * (kpoly<P, 0>(d1) * kpoly<P, 0>(d2) * kpoly<P, 0>(d3));
  } else if constexpr (A::SEP == 2) {   // its lengthscale gradient (product rule)
    constexpr int P0 = A::P0;
    const double e = fexp_neg((d1 + d2) + d3, tab);
    const double k1 = kpoly<P0, 0>(d1), k2 = kpoly<P0, 0>(d2);
    const double g1 = kpoly<P0 + 1, 1>(d1), g2 = kpoly<P0 + 1, 1>(d2);
    if constexpr (D == 3) {
      const double k3 = kpoly<P0, 0>(d3), g3 = kpoly<P0 + 1, 1>(d3);
      return e * fma(g1, k2 * k3, k1 * fma(g2, k3, k2 * g3));
    } else {
      return e * fma(g1, k2, k1 * g2);
    }
  } else if constexpr (A::SEP == 3) {   // second gradient run: the near field is in the first
    return 0.0;
  } else if constexpr (!A::PROD) {
    // L1: sum_q c_q s^q e^{-s} with the read coefficients of the algebra (Matern a_q for
    // KIND 0, gradient b_q = a_{q-1} - q a_q for KIND 1), Horner in s
    const double s = D == 3 ? (d1 + d2) + d3 : d1 + d2;
    const double e = fexp_neg(s, tab);
    double poly = rcoef(P, A::KIND, P);
#pragma unroll
    for (int q = P - 1; q >= 0; --q) poly = fma(poly, s, rcoef(P, A::KIND, q));
    return e * poly;
  } else {
    const double e = fexp_neg(d1 + d2, tab);
    if constexpr (A::KIND == 0) {
      if constexpr (P == 0) return e;
      else if constexpr (P == 1) return e * ((1.0 + d1) * (1.0 + d2));
      else if constexpr (P == 2)
        return e * (fma(d1, fma(d1, 1.0 / 3.0, 1.0), 1.0) * fma(d2, fma(d2, 1.0 / 3.0, 1.0), 1.0));
      else return e * (kpoly<P, 0>(d1) * kpoly<P, 0>(d2));   // nu = 7/2, 9/2
    } else {   // product rule: g(d1) k(d2) + k(d1) g(d2); k of order P - 1, g = -s k'(s) of order P
      if constexpr (P == 1) return e * (d1 + d2);
      else if constexpr (P == 2) return e * ((d1 * d1) * (1.0 + d2) + (1.0 + d1) * (d2 * d2));
      else
        return e * fma(kpoly<P, 1>(d1), kpoly<P - 1, 0>(d2), kpoly<P - 1, 0>(d1) * kpoly<P, 1>(d2));
    }
  }
}

#ifndef GPM_CP_MINB    // resident CTAs per SM the kernels are compiled for (register caps)
#define GPM_CP_MINB 3
#endif
#ifndef GPM_LOW_MINB
#define GPM_LOW_MINB 3
#endif
constexpr int CP_BLOCK = 128;
constexpr int CP_ITEMS = 8;
constexpr int CP_WARPS = CP_BLOCK / 32;
static_assert(CP_BLOCK * CP_ITEMS == LV_TILE, "tile = block x items");
// Swizzle of the 8-item rows (no padding): thread t's item k lives at 8t + ((k + t/2) & 7),
// so the 16 lanes of each half-warp 64-bit shared access hit 16 distinct bank pairs.
__host__ __device__ __forceinline__ int cpz(int i) { return (i & ~7) | ((i + (i >> 4)) & 7); }

template <int NS>
struct CSt {
  double D, E;
  double M[NS];
};
template <class A>
__device__ __forceinline__ CSt<A::NS> cs_id() {
  CSt<A::NS> s;
  s.D = 0.0; s.E = 1.0;
#pragma unroll
  for (int i = 0; i < A::NS; ++i) s.M[i] = 0.0;
  return s;
}
// forward: X then Y along the scan, moments referenced at the end of Y
template <class A>
__device__ __forceinline__ CSt<A::NS> cs_fw(const CSt<A::NS>& X, const CSt<A::NS>& Y) {
  CSt<A::NS> R;
#pragma unroll
  for (int i = 0; i < A::NS; ++i) R.M[i] = X.M[i];
  A::advance_all(R.M, Y.D, Y.E);
#pragma unroll
  for (int i = 0; i < A::NS; ++i) R.M[i] += Y.M[i];
  R.D = X.D + Y.D; R.E = X.E * Y.E;
  return R;
}
// backward: X left of Y, moments referenced just before the start of X
template <class A>
__device__ __forceinline__ CSt<A::NS> cs_bw(const CSt<A::NS>& X, const CSt<A::NS>& Y) {
  CSt<A::NS> R;
#pragma unroll
  for (int i = 0; i < A::NS; ++i) R.M[i] = Y.M[i];
  A::advance_all(R.M, X.D, X.E);
#pragma unroll
  for (int i = 0; i < A::NS; ++i) R.M[i] += X.M[i];
  R.D = X.D + Y.D; R.E = X.E * Y.E;
  return R;
}
template <int NS>
__device__ __forceinline__ CSt<NS> cs_shfl(const CSt<NS>& s, int off, bool up) {
  CSt<NS> r;
  if (up) {
    r.D = __shfl_up_sync(0xffffffffu, s.D, off);
    r.E = __shfl_up_sync(0xffffffffu, s.E, off);
#pragma unroll
    for (int i = 0; i < NS; ++i) r.M[i] = __shfl_up_sync(0xffffffffu, s.M[i], off);
  } else {
    r.D = __shfl_down_sync(0xffffffffu, s.D, off);
    r.E = __shfl_down_sync(0xffffffffu, s.E, off);
#pragma unroll
    for (int i = 0; i < NS; ++i) r.M[i] = __shfl_down_sync(0xffffffffu, s.M[i], off);
  }
  return r;
}
template <int NS>
__device__ __forceinline__ CSt<NS> cs_bcast(const CSt<NS>& s, int src) {
  CSt<NS> r;
  r.D = __shfl_sync(0xffffffffu, s.D, src);
  r.E = __shfl_sync(0xffffffffu, s.E, src);
#pragma unroll
  for (int i = 0; i < NS; ++i) r.M[i] = __shfl_sync(0xffffffffu, s.M[i], src);
  return r;
}
template <int NS, class R>
__device__ __forceinline__ void cs_put(R* g, const CSt<NS>& s) {
  g->D = s.D; g->E = s.E;
#pragma unroll
  for (int i = 0; i < NS; ++i) g->M[i] = s.M[i];
}
template <int NS, class R>
__device__ __forceinline__ CSt<NS> cs_get(const R* g) {
  CSt<NS> s;
  s.D = __ldcg(&g->D); s.E = __ldcg(&g->E);
#pragma unroll
  for (int i = 0; i < NS; ++i) s.M[i] = __ldcg(&g->M[i]);
  return s;
}

template <class A>
struct CpScratch {
  CSt<A::NS> wf[CP_WARPS], wb[CP_WARPS], cf, cb;
  double wsp[CP_WARPS];   // k_cp<1>: warp sums of the thread spans
};

// ---------------------------------------------------------------------------
// Within-tile levels: k_low2 / k_low3 / k_mid3.  One 1024-point tile per CTA of 128
// threads; point data staged once in shared memory (LvPoints); per level each thread
// builds its 8 consecutive positions of the level order in registers.  Nodes are aligned
// blocks of 2^ls positions with ls >= 3, so node boundaries fall between threads: the
// scans need no per-position flags (masked warp scans, per-warp carries).

// Near field by direct summation: every pair i != j of the same aligned block of 2^lb
// tile-local positions (x1-rank blocks in k_low2 / k_low3: exactly the pairs split at
// levels <= lb; position blocks of ord2[l1] with opposite x1 sides (l1side > 0): exactly
// the pairs split at (l1, l2 <= lb)).  IND: position p holds point Pt.o2[p] (k_low3's inner
// blocks), else point p.  Pt.acc[point] += sum_j K(i,j) u_j.
// (zz, znf): this CTA's slice of the partners (the block's partners in znf equal ranges).
template <class A, int D, bool IND>
__device__ __forceinline__ void near_field(LvPoints& Pt, int cnt, int lb, int l1side,
                                           const double* tab, int zz = 0, int znf = 1) {
  if constexpr (A::SEP == 3) return;   // second gradient run: near field done by the first
  const int i0 = threadIdx.x * CP_ITEMS;
  if (i0 >= cnt) return;
  double ti1[CP_ITEMS], ti2[CP_ITEMS], ti3[CP_ITEMS], acc[CP_ITEMS];
  int hi[CP_ITEMS];
#pragma unroll
  for (int k = 0; k < CP_ITEMS; ++k) {
    const int i = min(i0 + k, cnt - 1);
    const int pi = IND ? Pt.o2[i] : i;
    ti1[k] = Pt.t1[pi];
    ti2[k] = Pt.t2[pi];
    ti3[k] = D == 3 ? Pt.t3[pi] : 0.0;
    hi[k] = l1side ? ((IND ? pi : Pt.o2[i]) >> (l1side - 1)) & 1 : 0;
    acc[k] = 0.0;
  }
  const int sub = (1 << lb) / znf;
  const int bs = ((i0 >> lb) << lb) + zz * sub;
  const int be = min(bs + sub, cnt);
#pragma unroll 1
  for (int j = bs; j < be; ++j) {
    const int pj = IND ? Pt.o2[j] : j;
    const double tj1 = Pt.t1[pj], tj2 = Pt.t2[pj], uj = Pt.u[pj];
    const double tj3 = D == 3 ? Pt.t3[pj] : 0.0;
    const int hj = l1side ? ((IND ? pj : Pt.o2[j]) >> (l1side - 1)) & 1 : 0;
#pragma unroll
    for (int k = 0; k < CP_ITEMS; ++k) {
      const bool ok = (i0 + k != j) && (!l1side || hj != hi[k]);
      const double v = kval<A, D>(fabs(ti1[k] - tj1), fabs(ti2[k] - tj2), fabs(ti3[k] - tj3), tab);
      acc[k] = ok ? fma(v, uj, acc[k]) : acc[k];
    }
  }
#pragma unroll
  for (int k = 0; k < CP_ITEMS; ++k)
    if (i0 + k < cnt) Pt.acc[IND ? Pt.o2[i0 + k] : i0 + k] += acc[k];
}

// One thread's 8 positions of a level: gap to the previous position of the node (0 at a
// node start), e^{-gap}, split offset alpha, e^{-alpha}, source weight, channel (-1: the
// node has no cross pairs), output point (-1: none).
struct TItems {
  double d[CP_ITEMS], e[CP_ITEMS], a[CP_ITEMS], ea[CP_ITEMS], u[CP_ITEMS];
  int ch[CP_ITEMS], o[CP_ITEMS];
};

template <class A>
struct TScratch {
  CSt<A::NS> wf[CP_WARPS], wb[CP_WARPS];
  double tab[64];
};

// The level scan of one tile, nodes of 2^ls positions (ls >= 3): of[k] = the level's
// contribution to item k (both directions).  Barriers inside; uniform call.
template <class A>
__device__ __forceinline__ void seg_engine(const TItems& it, int ls, double* of,
                                           TScratch<A>& sc) {
  using S = CSt<A::NS>;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int i0 = tid * CP_ITEMS;
  const int smask = (1 << ls) - 1;
  const int seg = i0 >> ls;
  const int nthr = min(32, 1 << (ls - 3));   // threads of a node within a warp: scan steps beyond are masked off
  // ---- forward
  {
    S X;
    double D = 0.0, Ee = 1.0;
#pragma unroll
    for (int q = 0; q < A::NS; ++q) X.M[q] = 0.0;
#pragma unroll
    for (int k = CP_ITEMS - 1; k >= 0; --k) {
      A::inject_at(X.M, it.ch[k], it.u[k], it.a[k], it.ea[k], D, Ee);
      D += it.d[k];
      Ee *= it.e[k];
    }
    X.D = D; X.E = Ee;
#pragma unroll 1
    for (int off = 1; off < nthr; off <<= 1) {
      const S Y = cs_shfl<A::NS>(X, off, true);
      if (lane >= off && ((i0 - CP_ITEMS * off) >> ls) == seg) X = cs_fw<A>(Y, X);
    }
    if (lane == 31) sc.wf[warp] = X;
    S C = cs_shfl<A::NS>(X, 1, true);
    if (lane == 0 || (i0 & smask) == 0) C = cs_id<A>();
    __syncthreads();
    const int w0 = (i0 & ~smask) / (32 * CP_ITEMS);   // first warp of my node
    if (w0 < warp) {
      S W = sc.wf[w0];
#pragma unroll 1
      for (int w = w0 + 1; w < warp; ++w) W = cs_fw<A>(W, sc.wf[w]);
      C = cs_fw<A>(W, C);
    }
    double M[A::NS];
#pragma unroll
    for (int q = 0; q < A::NS; ++q) M[q] = C.M[q];
#pragma unroll
    for (int k = 0; k < CP_ITEMS; ++k) {
      A::advance_all(M, it.d[k], it.e[k]);
      of[k] = A::read(M, A::NCH - 1 - it.ch[k], it.a[k], it.ea[k]);
      A::inject(M, it.ch[k], it.u[k], it.a[k], it.ea[k]);
    }
  }
  // ---- backward
  {
    S X;
    double D = 0.0, Ee = 1.0;
#pragma unroll
    for (int q = 0; q < A::NS; ++q) X.M[q] = 0.0;
#pragma unroll
    for (int k = 0; k < CP_ITEMS; ++k) {
      D += it.d[k];
      Ee *= it.e[k];
      A::inject_at(X.M, it.ch[k], it.u[k], it.a[k], it.ea[k], D, Ee);
    }
    X.D = D; X.E = Ee;
#pragma unroll 1
    for (int off = 1; off < nthr; off <<= 1) {
      const S Y = cs_shfl<A::NS>(X, off, false);
      if (lane + off < 32 && ((i0 + CP_ITEMS * off) >> ls) == seg) X = cs_bw<A>(X, Y);
    }
    if (lane == 0) sc.wb[warp] = X;
    S C = cs_shfl<A::NS>(X, 1, false);
    if (lane == 31 || ((i0 + CP_ITEMS) & smask) == 0) C = cs_id<A>();
    const int w1 = min(((i0 | smask) + 1) / (32 * CP_ITEMS), CP_WARPS) - 1;   // last warp of my node
    __syncthreads();
    if (w1 > warp) {
      S W = sc.wb[w1];
#pragma unroll 1
      for (int w = w1 - 1; w > warp; --w) W = cs_bw<A>(sc.wb[w], W);
      C = cs_bw<A>(C, W);
    }
    double M[A::NS];
#pragma unroll
    for (int q = 0; q < A::NS; ++q) M[q] = C.M[q];
#pragma unroll
    for (int k = CP_ITEMS - 1; k >= 0; --k) {
      const double v = of[k] + A::read(M, A::NCH - 1 - it.ch[k], it.a[k], it.ea[k]);
      of[k] = it.ch[k] >= 0 ? v : 0.0;
      A::inject(M, it.ch[k], it.u[k], it.a[k], it.ea[k]);
      A::advance_all(M, it.d[k], it.e[k]);
    }
  }
  __syncthreads();   // scratch reuse
}

// One level of a tile kernel: the engine once, or (separated product forms, algebra.cuh) once
// per sub-pass (a, b) with sources re-weighted by alpha1^a alpha2^b and the target factor of
// the sub-pass; it.ea = e^{-(alpha1+alpha2)} as for L1, the split offset of the scan is 0.
template <class A>
__device__ __forceinline__ void level_apply(TItems& it, const double* a1, const double* a2, int ls,
                                            double* of, TScratch<A>& sc) {
  if constexpr (!A::P3) {
    seg_engine<A>(it, ls, of, sc);
  } else {
    double ub[CP_ITEMS], tot[CP_ITEMS];
#pragma unroll
    for (int k = 0; k < CP_ITEMS; ++k) {
      ub[k] = it.u[k];
      tot[k] = 0.0;
      it.a[k] = 0.0;
    }
#pragma unroll 1
    for (int ab = 0; ab < A::NAB; ++ab) {
#pragma unroll
      for (int k = 0; k < CP_ITEMS; ++k) it.u[k] = ub[k] * A::srcw(a1[k], a2[k], ab);
      double o[CP_ITEMS];
      seg_engine<A>(it, ls, o, sc);
#pragma unroll
      for (int k = 0; k < CP_ITEMS; ++k) tot[k] = fma(o[k], A::tgtw(a1[k], a2[k], ab), tot[k]);
    }
#pragma unroll
    for (int k = 0; k < CP_ITEMS; ++k) {
      of[k] = tot[k];
      it.u[k] = ub[k];
    }
  }
}

// Gaps from the scan coordinates y[k] (ypre: y of the position before the thread's first,
// ignored at a node start); padding items (o < 0) repeat the last y (gap 0).
__device__ __forceinline__ void titems_gaps(TItems& it, const double* y, double ypre,
                                            bool node_start, const double* tab) {
#pragma unroll
  for (int k = 0; k < CP_ITEMS; ++k) {
    const double dl = k == 0 ? (node_start ? 0.0 : y[0] - ypre) : y[k] - y[k - 1];
    it.d[k] = dl;
    it.e[k] = fexp_neg(dl, tab);
    it.ea[k] = fexp_neg(it.a[k], tab);
  }
}

// this thread's 8 entries of a tile-local order array (ranks relative to T0)
__device__ __forceinline__ void load_ord8(const int* ord, int i0, int cnt, int base, int* r) {
  if (i0 + CP_ITEMS <= cnt && (reinterpret_cast<uintptr_t>(ord) & 15) == 0) {
    const int4 a = __ldg(reinterpret_cast<const int4*>(ord + i0));
    const int4 b = __ldg(reinterpret_cast<const int4*>(ord + i0) + 1);
    r[0] = a.x - base; r[1] = a.y - base; r[2] = a.z - base; r[3] = a.w - base;
    r[4] = b.x - base; r[5] = b.y - base; r[6] = b.z - base; r[7] = b.w - base;
  } else {
#pragma unroll
    for (int k = 0; k < CP_ITEMS; ++k) r[k] = i0 + k < cnt ? __ldg(ord + i0 + k) - base : -1;
  }
}

// L1 prefetch of this thread's 8 entries (32 B) of a later level's order: the level loops
// are long, and the first use of the order stalls on an L2 round trip otherwise
__device__ __forceinline__ void prefetch_ord8(const int* ord, int i0, int cnt) {
  if (i0 < cnt) asm volatile("prefetch.global.L1 [%0];" ::"l"(ord + i0));
}

__host__ __device__ __forceinline__ int lv_clamp_lb(int lb, int lmax) {
  return lb < 3 ? (3 < lmax ? 3 : lmax) : (lb < lmax ? lb : lmax);
}
// The fused low kernels run in parts (blockIdx.z), each with its own output slot (summed in
// a fixed order by the epilogue): the near field in low_znf partner slices (a 256-rank block
// costs as much as four engine levels), then the engine levels -- d = 2: two levels per part,
// d = 3: one outer level l1 per part.  More, shorter CTAs: small n fills the SMs and the last
// wave of a large grid is short.
__host__ __device__ __forceinline__ int low_lb(int lb_opt, int L) {
  const int lmax = L < LV_LOGTILE ? L : LV_LOGTILE;
  const int lb = lv_clamp_lb(lb_opt, LV_LOGTILE);
  return lb < lmax ? lb : lmax;
}
__host__ __device__ __forceinline__ int low_znf(int lb) { return lb >= 8 ? 4 : (lb == 7 ? 2 : 1); }
__host__ __device__ __forceinline__ int low_lpart(int d, int lb, int l) {   // part of level l > lb
  return low_znf(lb) + (d == 2 ? (l - lb - 1) / 2 : l - lb - 1);
}
__host__ __device__ __forceinline__ int low_parts(int d, int lb_opt, int L) {
  const int lmax = L < LV_LOGTILE ? L : LV_LOGTILE;
  const int lb = low_lb(lb_opt, L);
  return lmax > lb ? low_lpart(d, lb, lmax) + 1 : low_znf(lb);
}

// ---- fused low levels, d = 2: every level l <= min(10, L) of one 1024-rank tile
template <class A>
__global__ void __launch_bounds__(CP_BLOCK, GPM_LOW_MINB) k_low2(LvArgs g) {
  lv_col(g);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LvPoints& Pt = *reinterpret_cast<LvPoints*>(smem_raw);
  __shared__ TScratch<A> sc;
  const int tid = threadIdx.x;
  const int i0 = tid * CP_ITEMS;
  const int64_t T0 = (int64_t)(blockIdx.x + g.tile0) * LV_TILE;
  const int cnt = (int)min((int64_t)LV_TILE, g.n - T0);
  fexp_table_init(sc.tab);
#pragma unroll 4
  for (int i = tid; i < LV_TILE; i += CP_BLOCK) if (i < cnt) {
    const Pt4 p = g.pts[T0 + i];
    Pt.u[i] = p.u;
    Pt.t1[i] = p.t1;
    Pt.t2[i] = p.t2;
    Pt.acc[i] = 0.0;
  }
  __syncthreads();
  const int lmax = min(LV_LOGTILE, g.L);
  const int lb = low_lb(g.lb, g.L);
  const int z = blockIdx.z, znf = low_znf(lb);
  if (lb > 0 && z < znf) near_field<A, 2, false>(Pt, cnt, lb, 0, sc.tab, z, znf);
  __syncthreads();
#pragma unroll 1
  for (int l = lb + 1; l <= lmax; ++l) {
    if (low_lpart(2, lb, l) != z) continue;
    const int* ord = g.ord2 + (size_t)(l - 1) * g.n + T0;
    TItems it;
    double y[CP_ITEMS];
    load_ord8(ord, i0, cnt, (int)T0, it.o);
    if (l < lmax) prefetch_ord8(ord + g.n, i0, cnt);   // the next level's order
#pragma unroll
    for (int k = 0; k < CP_ITEMS; ++k) {
      const int i = i0 + k;
      const int r = it.o[k];
      const int mid = ((i >> l) << l) + (1 << (l - 1));
      const bool act = r >= 0 && T0 + mid < g.n;
      y[k] = r >= 0 ? Pt.t2[r] : (k > 0 ? y[k - 1] : 0.0);
      it.u[k] = r >= 0 ? Pt.u[r] : 0.0;
      it.a[k] = act ? fabs(Pt.t1[r] - Pt.t1[mid]) : 0.0;
      it.ch[k] = act ? (r >> (l - 1)) & 1 : -1;
    }
    const bool nstart = (i0 & ((1 << l) - 1)) == 0;
    const double ypre = (!nstart && i0 <= cnt) ? Pt.t2[__ldg(ord + i0 - 1) - (int)T0] : 0.0;
    titems_gaps(it, y, ypre, nstart, sc.tab);
    double of[CP_ITEMS], a1k[CP_ITEMS], a2k[CP_ITEMS];
#pragma unroll
    for (int k = 0; k < CP_ITEMS; ++k) { a1k[k] = it.a[k]; a2k[k] = 0.0; }
    level_apply<A>(it, a1k, a2k, l, of, sc);
#pragma unroll
    for (int k = 0; k < CP_ITEMS; ++k) if (it.o[k] >= 0) Pt.acc[it.o[k]] += of[k];
  }
  __syncthreads();
  double* dst = z == 0 ? g.acc : g.part + (int64_t)(g.low_slot0 + z - 1) * g.n;
#pragma unroll 4
  for (int i = tid; i < LV_TILE; i += CP_BLOCK) if (i < cnt) dst[T0 + i] = Pt.acc[i];
}

// ---- fused low levels, d = 2, NC right-hand sides per CTA (nrhs >= 2, e.g. config 5's CG
// with [y, 1, x1, x2]): the kernel values of the near field and each level's gaps,
// e^{-gap}, alpha, e^{-alpha} do not depend on v -- computed once per tile and shared by the
// columns (k_low2 recomputes them per column).  acc / pts of column c at c * n.
template <int NC>
struct LvPointsM {
  double u[NC][LV_TILE], t1[LV_TILE], t2[LV_TILE], acc[NC][LV_TILE];
};

template <class A, int NC>
__global__ void __launch_bounds__(CP_BLOCK, NC <= 2 ? 3 : 2) k_low2m(LvArgs g, int nrhs) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LvPointsM<NC>& Pt = *reinterpret_cast<LvPointsM<NC>*>(smem_raw);
  __shared__ TScratch<A> sc;
  const int tid = threadIdx.x;
  const int i0 = tid * CP_ITEMS;
  const int c0 = blockIdx.y * NC;
  const int nc = min(NC, nrhs - c0);
  const int64_t T0 = (int64_t)(blockIdx.x + g.tile0) * LV_TILE;
  const int cnt = (int)min((int64_t)LV_TILE, g.n - T0);
  fexp_table_init(sc.tab);
#pragma unroll 2
  for (int i = tid; i < LV_TILE; i += CP_BLOCK) if (i < cnt) {
    const Pt4 p = g.pts[T0 + i];
    Pt.t1[i] = p.t1;
    Pt.t2[i] = p.t2;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      Pt.u[c][i] = c < nc ? g.pts[(int64_t)(c0 + c) * g.n + T0 + i].u : 0.0;
      Pt.acc[c][i] = 0.0;
    }
  }
  __syncthreads();
  const int lmax = min(LV_LOGTILE, g.L);
  const int lb = low_lb(g.lb, g.L);
  const bool split = gridDim.z > 1;   // large grids run every part in one CTA (one staging)
  const int z = blockIdx.z, znf = split ? low_znf(lb) : 1;
  if (lb > 0 && i0 < cnt && z < znf) {   // near field: one kernel value per pair, NC columns
    double ti1[CP_ITEMS], ti2[CP_ITEMS], acc[CP_ITEMS][NC];
#pragma unroll
    for (int k = 0; k < CP_ITEMS; ++k) {
      const int i = min(i0 + k, cnt - 1);
      ti1[k] = Pt.t1[i];
      ti2[k] = Pt.t2[i];
#pragma unroll
      for (int c = 0; c < NC; ++c) acc[k][c] = 0.0;
    }
    const int sub = (1 << lb) / znf;
    const int bs = ((i0 >> lb) << lb) + z * sub;
    const int be = min(bs + sub, cnt);
#pragma unroll 1
    for (int j = bs; j < be; ++j) {
      const double tj1 = Pt.t1[j], tj2 = Pt.t2[j];
      double uj[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) uj[c] = Pt.u[c][j];
#pragma unroll
      for (int k = 0; k < CP_ITEMS; ++k) {
        const double v = (i0 + k != j) ? kval<A, 2>(fabs(ti1[k] - tj1), fabs(ti2[k] - tj2), 0.0, sc.tab)
                                       : 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[k][c] = fma(v, uj[c], acc[k][c]);
      }
    }
#pragma unroll
    for (int k = 0; k < CP_ITEMS; ++k)
      if (i0 + k < cnt)
#pragma unroll
        for (int c = 0; c < NC; ++c) Pt.acc[c][i0 + k] += acc[k][c];
  }
  __syncthreads();
#pragma unroll 1
  for (int l = lb + 1; l <= lmax; ++l) {
    if (split && low_lpart(2, lb, l) != z) continue;
    const int* ord = g.ord2 + (size_t)(l - 1) * g.n + T0;
    TItems it;
    double y[CP_ITEMS];
    load_ord8(ord, i0, cnt, (int)T0, it.o);
    if (l < lmax) prefetch_ord8(ord + g.n, i0, cnt);   // the next level's order
#pragma unroll
    for (int k = 0; k < CP_ITEMS; ++k) {
      const int i = i0 + k;
      const int r = it.o[k];
      const int mid = ((i >> l) << l) + (1 << (l - 1));
      const bool act = r >= 0 && T0 + mid < g.n;
      y[k] = r >= 0 ? Pt.t2[r] : (k > 0 ? y[k - 1] : 0.0);
      it.a[k] = act ? fabs(Pt.t1[r] - Pt.t1[mid]) : 0.0;
      it.ch[k] = act ? (r >> (l - 1)) & 1 : -1;
    }
    const bool nstart = (i0 & ((1 << l) - 1)) == 0;
    const double ypre = (!nstart && i0 <= cnt) ? Pt.t2[__ldg(ord + i0 - 1) - (int)T0] : 0.0;
    titems_gaps(it, y, ypre, nstart, sc.tab);
    double a1k[CP_ITEMS], a2k[CP_ITEMS];
#pragma unroll
    for (int k = 0; k < CP_ITEMS; ++k) { a1k[k] = it.a[k]; a2k[k] = 0.0; }
#pragma unroll 1
    for (int c = 0; c < nc; ++c) {
#pragma unroll
      for (int k = 0; k < CP_ITEMS; ++k) it.u[k] = it.o[k] >= 0 ? Pt.u[c][it.o[k]] : 0.0;
      double of[CP_ITEMS];
      level_apply<A>(it, a1k, a2k, l, of, sc);
#pragma unroll
      for (int k = 0; k < CP_ITEMS; ++k) if (it.o[k] >= 0) Pt.acc[c][it.o[k]] += of[k];
    }
  }
  __syncthreads();
#pragma unroll 1
  for (int c = 0; c < nc; ++c) {
    double* dst = z == 0 ? g.acc + (int64_t)(c0 + c) * g.n
                         : g.part + (int64_t)(c0 + c) * g.part_stride +
                               (int64_t)(g.low_slot0 + z - 1) * g.n;
#pragma unroll 4
    for (int i = tid; i < LV_TILE; i += CP_BLOCK)
      if (i < cnt) dst[T0 + i] = Pt.acc[c][i];
  }
}

// ---- fused low levels, d = 3: every (l1 <= min(10, L), l2 <= l1) of one tile
template <class A>
__global__ void __launch_bounds__(CP_BLOCK, GPM_LOW_MINB) k_low3(LvArgs g) {
  lv_col(g);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LvPoints& Pt = *reinterpret_cast<LvPoints*>(smem_raw);
  __shared__ TScratch<A> sc;
  const int tid = threadIdx.x;
  const int i0 = tid * CP_ITEMS;
  const int64_t T0 = (int64_t)(blockIdx.x + g.tile0) * LV_TILE;
  const int cnt = (int)min((int64_t)LV_TILE, g.n - T0);
  fexp_table_init(sc.tab);
#pragma unroll 4
  for (int i = tid; i < LV_TILE; i += CP_BLOCK) if (i < cnt) {
    const Pt4 p = g.pts[T0 + i];
    Pt.u[i] = p.u;
    Pt.t1[i] = p.t1;
    Pt.t2[i] = p.t2;
    Pt.t3[i] = p.t3;
    Pt.acc[i] = 0.0;
  }
  __syncthreads();
  const int lmax = min(LV_LOGTILE, g.L);
  const int lb = low_lb(g.lb, g.L);
  const int z = blockIdx.z, znf = low_znf(lb);
  if (lb > 0 && z < znf) near_field<A, 3, false>(Pt, cnt, lb, 0, sc.tab, z, znf);
#pragma unroll 1
  for (int l1 = lb + 1; l1 <= lmax; ++l1) {
    if (low_lpart(3, lb, l1) != z) continue;
    __syncthreads();
#pragma unroll 4
    for (int i = tid; i < LV_TILE; i += CP_BLOCK) if (i < cnt)
      Pt.o2[i] = __ldg(g.ord2 + (size_t)(l1 - 1) * g.n + T0 + i) - (int)T0;
    __syncthreads();
    // inner levels l2 <= 3: opposite-x1-side pairs of the same 8-position block of ord2[l1]
    near_field<A, 3, true>(Pt, cnt, 3, l1, sc.tab);
    __syncthreads();
#pragma unroll 1
    for (int l2 = 4; l2 <= l1; ++l2) {
      const int* ord = g.ord3 + (size_t)ord3_index(l1, l2) * g.n + T0;
      TItems it;
      double y[CP_ITEMS], a1k[CP_ITEMS], a2k[CP_ITEMS];
      int qq[CP_ITEMS];
      load_ord8(ord, i0, cnt, (int)T0, qq);
      if (l2 < l1) prefetch_ord8(ord + g.n, i0, cnt);   // ord3[(l1, l2 + 1)] follows
#pragma unroll
      for (int k = 0; k < CP_ITEMS; ++k) {
        const int i = i0 + k;
        const int q = qq[k];                       // position in ord2[l1] (tile-local)
        const int r = q >= 0 ? Pt.o2[q] : -1;      // rank (tile-local)
        const int mid1 = ((max(q, 0) >> l1) << l1) + (1 << (l1 - 1));
        const int mid2 = ((i >> l2) << l2) + (1 << (l2 - 1));
        const bool act = r >= 0 && (T0 + mid1 < g.n) && (T0 + mid2 < g.n);
        it.o[k] = r;
        y[k] = r >= 0 ? Pt.t3[r] : (k > 0 ? y[k - 1] : 0.0);
        it.u[k] = r >= 0 ? Pt.u[r] : 0.0;
        a1k[k] = act ? fabs(Pt.t1[r] - Pt.t1[mid1]) : 0.0;
        a2k[k] = act ? fabs(Pt.t2[r] - Pt.t2[Pt.o2[mid2]]) : 0.0;
        it.a[k] = a1k[k] + a2k[k];
        it.ch[k] = act ? 2 * ((r >> (l1 - 1)) & 1) + ((q >> (l2 - 1)) & 1) : -1;
      }
      const bool nstart = (i0 & ((1 << l2) - 1)) == 0;
      const double ypre =
          (!nstart && i0 <= cnt) ? Pt.t3[Pt.o2[__ldg(ord + i0 - 1) - (int)T0]] : 0.0;
      titems_gaps(it, y, ypre, nstart, sc.tab);
      double of[CP_ITEMS];
      level_apply<A>(it, a1k, a2k, l2, of, sc);
#pragma unroll
      for (int k = 0; k < CP_ITEMS; ++k) if (it.o[k] >= 0) Pt.acc[it.o[k]] += of[k];
    }
  }
  __syncthreads();
  double* dst = z == 0 ? g.acc : g.part + (int64_t)(g.low_slot0 + z - 1) * g.n;
#pragma unroll 4
  for (int i = tid; i < LV_TILE; i += CP_BLOCK) if (i < cnt) dst[T0 + i] = Pt.acc[i];
}

// ---- d = 3, one outer level l1 > 10, all inner levels l2 <= 10 (tile = 1024 positions of
// ord2[l1], i.e. one slice of one outer node; its points are gathered once)
template <class A>
__global__ void __launch_bounds__(CP_BLOCK, GPM_LOW_MINB) k_mid3(LvArgs g) {
  lv_col(g);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LvPoints& Pt = *reinterpret_cast<LvPoints*>(smem_raw);
  __shared__ TScratch<A> sc;
  const int tid = threadIdx.x;
  const int i0 = tid * CP_ITEMS;
  const int l1 = g.l1 + (int)blockIdx.z;   // one launch covers every outer level l1 > 10
  const int64_t T0 = (int64_t)(blockIdx.x + g.tile0) * LV_TILE;
  const int cnt = (int)min((int64_t)LV_TILE, g.n - T0);
  const int64_t mid1 = ((T0 >> l1) << l1) + (int64_t(1) << (l1 - 1));
  double* slot = g.part + (int64_t)(g.npass + blockIdx.z) * g.n;
  if (mid1 >= g.n) {   // outer node without cross pairs (uniform per CTA): zero contribution
    const int* o2z = g.ord2 + (size_t)(l1 - 1) * g.n + T0;
    for (int i = tid; i < cnt; i += CP_BLOCK) slot[__ldg(o2z + i)] = 0.0;
    return;
  }
  fexp_table_init(sc.tab);
  const double m1 = __ldg(g.t1 + mid1);
  const int* o2g = g.ord2 + (size_t)(l1 - 1) * g.n + T0;
#pragma unroll 4
  for (int i = tid; i < LV_TILE; i += CP_BLOCK) if (i < cnt) {
    const int r = __ldg(o2g + i);
    const Pt4 p = g.pts[r];
    Pt.o2[i] = r;
    Pt.u[i] = p.u;
    Pt.t1[i] = p.t1;
    Pt.t2[i] = p.t2;
    Pt.t3[i] = p.t3;
    Pt.acc[i] = 0.0;
  }
  __syncthreads();
  const int lb2 = lv_clamp_lb(g.lb2, LV_LOGTILE);
  near_field<A, 3, false>(Pt, cnt, lb2, l1, sc.tab);
  __syncthreads();
#pragma unroll 1
  for (int l2 = lb2 + 1; l2 <= LV_LOGTILE; ++l2) {
    const int* ord = g.ord3 + (size_t)ord3_index(l1, l2) * g.n + T0;
    TItems it;
    double y[CP_ITEMS], a1k[CP_ITEMS], a2k[CP_ITEMS];
    load_ord8(ord, i0, cnt, (int)T0, it.o);          // tile-local position = point index
    if (l2 < LV_LOGTILE) prefetch_ord8(ord + g.n, i0, cnt);   // ord3[(l1, l2 + 1)] follows
#pragma unroll
    for (int k = 0; k < CP_ITEMS; ++k) {
      const int i = i0 + k;
      const int q = it.o[k];
      const int mid2 = ((i >> l2) << l2) + (1 << (l2 - 1));
      const bool act = q >= 0 && T0 + mid2 < g.n;
      y[k] = q >= 0 ? Pt.t3[q] : (k > 0 ? y[k - 1] : 0.0);
      it.u[k] = q >= 0 ? Pt.u[q] : 0.0;
      a1k[k] = act ? fabs(Pt.t1[q] - m1) : 0.0;
      a2k[k] = act ? fabs(Pt.t2[q] - Pt.t2[mid2]) : 0.0;
      it.a[k] = a1k[k] + a2k[k];
      it.ch[k] = act ? 2 * ((Pt.o2[q] >> (l1 - 1)) & 1) + ((q >> (l2 - 1)) & 1) : -1;
    }
    const bool nstart = (i0 & ((1 << l2) - 1)) == 0;
    const double ypre = (!nstart && i0 <= cnt) ? Pt.t3[__ldg(ord + i0 - 1) - (int)T0] : 0.0;
    titems_gaps(it, y, ypre, nstart, sc.tab);
    double of[CP_ITEMS];
    level_apply<A>(it, a1k, a2k, l2, of, sc);
#pragma unroll
    for (int k = 0; k < CP_ITEMS; ++k) if (it.o[k] >= 0) Pt.acc[it.o[k]] += of[k];
  }
  __syncthreads();
#pragma unroll 4
  for (int i = tid; i < LV_TILE; i += CP_BLOCK) if (i < cnt) slot[Pt.o2[i]] = Pt.acc[i];   // own slot: summed in order by the epilogue
}

// ---- one pass whose segments span several tiles (mode 1: aggregates, 2: apply)
struct Elem {
  double y, u, a, a2;   // a: the x1 split offset (d = 2: the only one), a2: the x2 split offset
  int r, ch;
};

__device__ __forceinline__ Elem lv_elem(const LvArgs& g, int64_t pos) {
  Elem el;
  if (g.mode == 2) {
    const int l = g.lseg;
    const int r = __ldg(g.ord + pos);
    const int64_t mid = ((pos >> l) << l) + (int64_t(1) << (l - 1));
    const Pt4 p = g.pts[r];
    el.a = fabs(p.t1 - __ldg(g.t1 + mid));
    el.a2 = 0.0;
    el.ch = (r >> (l - 1)) & 1;
    el.y = p.t2;
    el.u = p.u;
    el.r = r;
  } else {
    const int l1 = g.l1, l2 = g.lseg;
    const int q = __ldg(g.ord + pos);
    const int r = __ldg(g.ord2l1 + q);
    const int64_t mid1 = ((int64_t)(q >> l1) << l1) + (int64_t(1) << (l1 - 1));
    const int64_t mid2 = ((pos >> l2) << l2) + (int64_t(1) << (l2 - 1));
    const Pt4 p = g.pts[r];
    el.a = fabs(p.t1 - __ldg(g.t1 + mid1));
    el.a2 = fabs(p.t2 - __ldg(g.t2 + __ldg(g.ord2l1 + mid2)));
    el.ch = 2 * ((r >> (l1 - 1)) & 1) + ((q >> (l2 - 1)) & 1);
    el.y = p.t3;
    el.u = p.u;
    el.r = r;
  }
  return el;
}

__device__ __forceinline__ double lv_y(const LvArgs& g, int64_t pos) {
  if (g.mode == 2) return g.pts[__ldg(g.ord + pos)].t2;
  return g.pts[__ldg(g.ord2l1 + __ldg(g.ord + pos))].t3;
}

// Structure of one carried (multi-tile) pass, precomputed at setup (it does not depend on
// v): per position the gap to the previous position of its node, the split offset alpha,
// the rank and the channel: 20 B per position, read coalesced.  e^{-gap} and e^{-alpha}
// are recomputed per tile in k_cp (two branch-free fexp_neg per position and launch: the
// same values bit for bit, 16 B per position less DRAM traffic -- config 4 moves 2.1 GB of
// staged structure per apply at 36 B per position).
struct HpView {
  const double* d;
  const double* a;      // split offset (d = 3 L1: alpha1 + alpha2; P3: alpha1)
  const double* a2;     // P3 (d = 3 product form) only: alpha2, 28 B per position
  const unsigned* rc;   // rank | channel << 30; CP_NONE: padding
};
constexpr unsigned CP_RMASK = 0x3FFFFFFFu;
constexpr unsigned CP_NONE = 0xFFFFFFFFu;   // rank field CP_RMASK: no point (n < 2^30)
// Padded to whole tiles; within a tile, position i is stored at cpz(i) (the k_cp shared
// layout), padding positions are identities (no gap, no source, no target).
__host__ __device__ inline int64_t hp_padded(int64_t nact) {
  return (nact + LV_TILE - 1) / LV_TILE * LV_TILE;
}
__host__ __device__ inline size_t hp_bytes(int64_t nact, bool p3) {
  return ((size_t)hp_padded(nact) * (p3 ? 28 : 20) + 255) & ~size_t(255);
}
__host__ __device__ inline HpView hp_view(const unsigned char* base, int64_t nact, bool p3) {
  const int64_t np = hp_padded(nact);
  HpView v;
  v.d = reinterpret_cast<const double*>(base);
  v.a = v.d + np;
  v.a2 = p3 ? v.a + np : nullptr;
  v.rc = reinterpret_cast<const unsigned*>(v.a + (p3 ? 2 : 1) * np);
  return v;
}

#if GPM_LEVEL_PART == 0
__global__ void k_hp_prep(LvArgs g, unsigned char* base, bool p3) {
  HpView v = hp_view(base, g.n_act, p3);
  double* d = const_cast<double*>(v.d);
  double* a = const_cast<double*>(v.a);
  double* a2 = const_cast<double*>(v.a2);
  unsigned* rc = const_cast<unsigned*>(v.rc);
  const int64_t smask = (int64_t(1) << g.lseg) - 1;
  const int64_t np = hp_padded(g.n_act);
  for (int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pos < np;
       pos += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = (pos & ~int64_t(LV_TILE - 1)) | cpz((int)(pos & (LV_TILE - 1)));
    if (pos < g.n_act) {
      const Elem el = lv_elem(g, pos);
      const double dl = (pos & smask) == 0 ? 0.0 : el.y - lv_y(g, pos - 1);
      d[w] = dl;
      a[w] = p3 ? el.a : el.a + el.a2;
      if (p3) a2[w] = el.a2;
      rc[w] = (unsigned)el.r | ((unsigned)el.ch << 30);
    } else {   // identity: no gap; alpha = 800 makes e^{-alpha} exactly 0 (fexp_neg: d >= 708)
      d[w] = 0.0; a[w] = 800.0; rc[w] = CP_NONE;
      if (p3) a2[w] = 0.0;
    }
  }
}

#endif   // GPM_LEVEL_PART == 0

// one carried pass (flattened work items item0 .. item0 + ntiles - 1 of k_cp)
struct HpDesc {
  int64_t off;      // byte offset of the staged structure in hpbuf
  int64_t nact;     // active positions
  int lseg, ntiles;
  int item0, pad;
};

// ---------------------------------------------------------------------------
// Carried passes (k_cp).  A carried pass's nodes span whole 1024-position tiles, so no
// node boundary falls inside a tile: the tile scan needs no flags.  The structure of every
// carried pass is staged at setup (k_hp_prep) tile by tile in the exact shared-memory
// layout below, padded to whole tiles with identity positions, so one tile arrives as six
// 1-D bulk copies.  The kernel is persistent: each CTA walks the flattened (pass, tile)
// list with a two-stage bulk-copy pipeline (tile k + 2 loads while tile k computes), and
// processes every right-hand side of a tile from the staged copy; the gather of the next
// (tile, column)'s sources is in flight during the current one.  Per tile and column:
// 128 threads x 8 consecutive positions; per-thread aggregates in the direct form
// (Alg::inject_at), warp scans, block carry, apply loops.
//   MODE 1: tile aggregates (forward, backward) -> aggs;
//   MODE 2: apply, with the tile carries folded from MODE 1's aggregates of the node.
template <bool P3>
struct CpStageT {
  double d[LV_TILE], a[LV_TILE];
  unsigned rc[LV_TILE];   // rank | channel << 30
};
template <>
struct CpStageT<true> {   // d = 3 product form: both split offsets
  double d[LV_TILE], a[LV_TILE], a2[LV_TILE];
  unsigned rc[LV_TILE];
};
template <bool P3>
struct CpSmemT {
  CpStageT<P3> st[2];
};

// Tile carries of every node, once per (column, pass, direction): an exclusive scan of the
// tile aggregates of k_cp<1> (forward: tiles in order; backward: reversed), one warp per
// node, 32 tiles per step (Kogge-Stone with the same combine as the tile scans).  k_cp<2>
// then loads one record per direction instead of folding up to #tiles aggregates per column.
constexpr int CC_WARPS = 8;   // k_cp_carry: 8 warps x 32 tiles per step
template <class A>
__global__ void __launch_bounds__(32 * CC_WARPS) k_cp_carry(LvRecFor<A::NS>* aggs,
                                                            LvRecFor<A::NS>* carr,
                                                            const HpDesc* descs, int npass,
                                                            int max_tiles) {
  using S = CSt<A::NS>;
  using Rec = LvRecFor<A::NS>;
  __shared__ S wtot[CC_WARPS];
  const int p = blockIdx.y;
  const int c = blockIdx.z >> 1, dir = blockIdx.z & 1;
  const HpDesc hd = descs[p];
  const int tps = 1 << (hd.lseg - LV_LOGTILE);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t base = ((int64_t)c * npass + p) * 2 * max_tiles;
  const Rec* ag = aggs + base;
  Rec* cr = carr + base;
  if (tps <= 32) {   // short nodes: one warp per node, one step, no block barrier
    const int first = (blockIdx.x * CC_WARPS + warp) * tps;
    if (first >= hd.ntiles) return;
    const int last = min(first + tps, hd.ntiles) - 1;
    const int t = dir == 0 ? first + lane : last - lane;
    const bool in = lane <= last - first;
    S x = in ? cs_get<A::NS>(ag + 2 * t + dir) : cs_id<A>();
#pragma unroll 1
    for (int off = 1; off < tps; off <<= 1) {
      const S y = cs_shfl<A::NS>(x, off, true);
      if (lane >= off) x = dir == 0 ? cs_fw<A>(y, x) : cs_bw<A>(x, y);
    }
    S ex = cs_shfl<A::NS>(x, 1, true);
    if (lane == 0) ex = cs_id<A>();
    if (in) cs_put<A::NS>(cr + 2 * t + dir, ex);
    return;
  }
  const int first = blockIdx.x * tps;   // long nodes: one CTA per node
  if (first >= hd.ntiles) return;
  const int last = min(first + tps, hd.ntiles) - 1;
  const int cnt = last - first + 1;
  S cin = cs_id<A>();   // fold of the tiles before this step (same value in every thread)
  // step: 256 tiles, tile index j (0 = first tile in scan order); forward scans first..last,
  // backward scans last..first with the mirrored combine
#pragma unroll 1
  for (int j0 = 0; j0 < cnt; j0 += 32 * CC_WARPS) {
    const int j = j0 + threadIdx.x;
    const int t = dir == 0 ? first + j : last - j;
    const bool in = j < cnt;
    const bool wact = j0 + 32 * warp < cnt;   // this warp has tiles (uniform per warp)
    S ex = cs_id<A>();
    if (wact) {
      S x = in ? cs_get<A::NS>(ag + 2 * t + dir) : cs_id<A>();
#pragma unroll 1
      for (int off = 1; off < 32; off <<= 1) {
        const S y = cs_shfl<A::NS>(x, off, true);
        if (lane >= off) x = dir == 0 ? cs_fw<A>(y, x) : cs_bw<A>(x, y);
      }
      if (lane == 31) wtot[warp] = x;
      ex = cs_shfl<A::NS>(x, 1, true);
      if (lane == 0) ex = cs_id<A>();
    }
    __syncthreads();
    if (wact) {
      S pre = cin;
#pragma unroll 1
      for (int w = 0; w < warp; ++w) pre = dir == 0 ? cs_fw<A>(pre, wtot[w]) : cs_bw<A>(wtot[w], pre);
      if (in) cs_put<A::NS>(cr + 2 * t + dir, dir == 0 ? cs_fw<A>(pre, ex) : cs_bw<A>(ex, pre));
    }
    if (j0 + 32 * CC_WARPS < cnt) {   // another step: carry the whole step's fold
#pragma unroll 1
      for (int w = 0; w < CC_WARPS; ++w) cin = dir == 0 ? cs_fw<A>(cin, wtot[w]) : cs_bw<A>(wtot[w], cin);
      __syncthreads();
    }
  }
}

// flattened work item -> pass: items are visited in increasing order, so each CTA keeps a
// running pass index
constexpr int CP_MAXDESC = 64;   // pass descriptors kept in k_cp's shared memory (2 KB)
__device__ __forceinline__ int cp_pass_at(const HpDesc* descs, int npass, int p, int item) {
  while (p + 1 < npass && descs[p + 1].item0 <= item) ++p;
  return p;
}

// thread 0: bulk-copy tile `item` of pass p into stage buffer st (20 / 28 KB on bar)
template <bool P3>
__device__ __forceinline__ void cp_issue(const unsigned char* hpbase, const HpDesc* descs, int p,
                                         int item, CpStageT<P3>& st, uint64_t* bar) {
  const HpDesc hd = descs[p];
  const int64_t T0 = (int64_t)(item - hd.item0) * LV_TILE;
  const HpView v = hp_view(hpbase + hd.off, hd.nact, P3);
  mbar_expect_tx(bar, (P3 ? 28u : 20u) * LV_TILE);
  tma_load_1d(st.d, v.d + T0, 8 * LV_TILE, bar);
  tma_load_1d(st.a, v.a + T0, 8 * LV_TILE, bar);
  if constexpr (P3) tma_load_1d(st.a2, v.a2 + T0, 8 * LV_TILE, bar);
  tma_load_1d(st.rc, v.rc + T0, 4 * LV_TILE, bar);
}

// staged split offsets as the engine sees them: L1 / mixed-moment product: the offset alpha
// and e^{-alpha}; separated forms: offset 0 (the split factors sit in the source weight and
// the target factor of the sub-pass), e^{-(alpha1+alpha2)}
template <class A>
__device__ __forceinline__ double cp_aoff(const CpStageT<A::ST2>& E, int z) {
  if constexpr (A::P3) return 0.0;
  else return E.a[z];
}
template <class A>
__device__ __forceinline__ double cp_a2(const CpStageT<A::ST2>& E, int z) {
  if constexpr (A::ST2) return E.a2[z];
  else return 0.0;
}

template <class A, int MODE>
__global__ void __launch_bounds__(CP_BLOCK, GPM_CP_MINB) k_cp(LvArgs g, const unsigned char* hpbase,
                                                   const HpDesc* descs_g, int npass, int total,
                                                   int max_tiles, int nrhs, int64_t carr_off,
                                                   int item_lo) {
  // items [item_lo, total) of the flattened (pass, tile) list (a sharded apply's share)
  const int b0 = item_lo + (int)blockIdx.x;
  using S = CSt<A::NS>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using Stage = CpStageT<A::ST2>;
  CpSmemT<A::ST2>& SM = *reinterpret_cast<CpSmemT<A::ST2>*>(smem_raw);
  __shared__ CpScratch<A> sc;
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ double s_tab[64];
  // the pass descriptors in shared memory (every item looks its pass up; the global copy
  // misses L1 behind the streamed tiles): up to CP_MAXDESC passes, else the global array
  __shared__ HpDesc s_desc[CP_MAXDESC];
  const HpDesc* descs = npass <= CP_MAXDESC ? s_desc : descs_g;
  if (npass <= CP_MAXDESC)
    for (int i = threadIdx.x; i < npass; i += CP_BLOCK) s_desc[i] = descs_g[i];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int i0 = tid * CP_ITEMS;
  const int G = gridDim.x;
  int p_iss = 0;   // pass of the last issued tile (thread 0)
  fexp_table_init(s_tab);
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0) {
    if (b0 < total) {
      p_iss = cp_pass_at(descs, npass, p_iss, b0);
      cp_issue(hpbase, descs, p_iss, b0, SM.st[0], &bar[0]);
    }
    if (b0 + G < total) {
      p_iss = cp_pass_at(descs, npass, p_iss, b0 + G);
      cp_issue(hpbase, descs, p_iss, b0 + G, SM.st[1], &bar[1]);
    }
  }
  // sources of the first (tile, column)
  double un[CP_ITEMS];
  if (b0 < total) {
    mbar_wait(&bar[0], 0);
#pragma unroll
    for (int k = 0; k < CP_ITEMS; ++k) {
      const unsigned r = SM.st[0].rc[cpz(i0 + k)] & CP_RMASK;
      un[k] = r != CP_RMASK ? __ldcg(&g.pts[r].u) : 0.0;
    }
  }
  int j = 0, p = 0;
#pragma unroll 1
  for (int item = b0; item < total; item += G, ++j) {
    const int sidx = j & 1;
    Stage& E = SM.st[sidx];
    mbar_wait(&bar[sidx], (j >> 1) & 1);
    p = cp_pass_at(descs, npass, p, item);
    const HpDesc hd = descs[p];
    const int t = item - hd.item0;
    const int tps = 1 << (hd.lseg - LV_LOGTILE);    // tiles per node
    const int first = t & ~(tps - 1);
    const int last = min(first + tps, hd.ntiles) - 1;
    // e^{-gap}, e^{-alpha} of my positions (not staged: recomputed, shared by the columns)
    double ek[CP_ITEMS], eak[CP_ITEMS];
#pragma unroll
    for (int k = 0; k < CP_ITEMS; ++k) {
      const int z = cpz(i0 + k);
      ek[k] = fexp_neg(E.d[z], s_tab);
      eak[k] = fexp_neg(E.a[z] + cp_a2<A>(E, z), s_tab);
    }
    // separated product forms: every column runs NAB sub-passes (a, b) with sources
    // re-weighted by alpha1^a alpha2^b and the sub-pass's target factor (algebra.cuh); each
    // sub-pass has its own tile aggregates / carries (index cc), the outputs are summed
    double ur[CP_ITEMS], tot[CP_ITEMS];
#pragma unroll 1
    for (int cc = 0; cc < nrhs * A::NAB; ++cc) {
      const int c = cc / A::NAB, ab = cc - c * A::NAB;
      LvRecFor<A::NS>* aggs =
          reinterpret_cast<LvRecFor<A::NS>*>(g.aggs) + ((int64_t)cc * npass + p) * 2 * max_tiles;
      double uc[CP_ITEMS], of[CP_ITEMS];
      if (ab == 0) {
#pragma unroll
      for (int k = 0; k < CP_ITEMS; ++k) { ur[k] = un[k]; tot[k] = 0.0; }
      // prefetch the sources of the next (tile, column)
      if (c + 1 < nrhs) {
        const Pt4* pn = g.pts + (int64_t)(c + 1) * g.n;
#pragma unroll
        for (int k = 0; k < CP_ITEMS; ++k) {
          const unsigned r = E.rc[cpz(i0 + k)] & CP_RMASK;
          un[k] = r != CP_RMASK ? __ldcg(&pn[r].u) : 0.0;
        }
      } else if (item + G < total) {
        Stage& En = SM.st[sidx ^ 1];
        mbar_wait(&bar[sidx ^ 1], ((j + 1) >> 1) & 1);
#pragma unroll
        for (int k = 0; k < CP_ITEMS; ++k) {
          const unsigned r = En.rc[cpz(i0 + k)] & CP_RMASK;
          un[k] = r != CP_RMASK ? __ldcg(&g.pts[r].u) : 0.0;
        }
      }
      }
#pragma unroll
      for (int k = 0; k < CP_ITEMS; ++k) {
        if constexpr (A::P3) {
          const int z = cpz(i0 + k);
          uc[k] = ur[k] * A::srcw(E.a[z], cp_a2<A>(E, z), ab);
        } else {
          uc[k] = ur[k];
        }
      }
      // tile carries (k_cp_carry): loaded into registers now, stored to shared memory just
      // before the barrier that precedes their first use (the load's latency hides behind
      // the thread aggregates and the warp scan)
      double cvf = 0.0, cvb = 0.0;
      if (MODE == 2) {
        const double* cr = reinterpret_cast<const double*>(aggs + carr_off + 2 * t);
        if (tid < A::NS + 2) cvf = __ldcg(cr + tid);
        if (tid >= 32 && tid < 32 + A::NS + 2)
          cvb = __ldcg(cr + sizeof(LvRecFor<A::NS>) / 8 + tid - 32);
      }
      if constexpr (MODE == 1) {
        // ---- tile aggregates only: each thread's aggregates (direct form) shifted to the
        // tile's reference points and summed (a fixed-order reduction: no scan of the
        // (span, moments) pairs needed -- the spans are prefix sums of scalars)
        S XF, XB;
        double D = 0.0, Ee = 1.0, Db = 0.0, Eb = 1.0;
#pragma unroll
        for (int q = 0; q < A::NS; ++q) XF.M[q] = XB.M[q] = 0.0;
#pragma unroll
        for (int k = CP_ITEMS - 1; k >= 0; --k) {    // forward: reference at item 7
          const int z = cpz(i0 + k);
          A::inject_at(XF.M, E.rc[z] >> 30, uc[k], cp_aoff<A>(E, z), eak[k], D, Ee);
          D += E.d[z];
          Ee *= ek[k];
        }
#pragma unroll
        for (int k = 0; k < CP_ITEMS; ++k) {         // backward: reference before item 0
          const int z = cpz(i0 + k);
          Db += E.d[z];
          Eb *= ek[k];
          A::inject_at(XB.M, E.rc[z] >> 30, uc[k], cp_aoff<A>(E, z), eak[k], Db, Eb);
        }
        // spans after my last position / before my first one within the tile
        double incl = D;   // inclusive prefix sum of the thread spans (warp)
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const double y = __shfl_up_sync(0xffffffffu, incl, off);
          if (lane >= off) incl += y;
        }
        if (lane == 31) sc.wsp[warp] = incl;
        __syncthreads();
        double before = incl - D, wtot = 0.0, tot = 0.0;
#pragma unroll
        for (int w = 0; w < CP_WARPS; ++w) {
          const double sw = sc.wsp[w];
          if (w < warp) wtot += sw;
          tot += sw;
        }
        before = fmax(before + wtot, 0.0);
        const double after = tot - before - D;
        A::advance_all(XF.M, fmax(after, 0.0), fexp_neg(fmax(after, 0.0), s_tab));
        A::advance_all(XB.M, before, fexp_neg(before, s_tab));
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
#pragma unroll
          for (int q = 0; q < A::NS; ++q) {
            XF.M[q] += __shfl_xor_sync(0xffffffffu, XF.M[q], off);
            XB.M[q] += __shfl_xor_sync(0xffffffffu, XB.M[q], off);
          }
        if (lane == 0) {
          sc.wf[warp] = XF;
          sc.wb[warp] = XB;
        }
        __syncthreads();
        if (tid == 0) {
          S TF = sc.wf[0], TB = sc.wb[0];
#pragma unroll 1
          for (int w = 1; w < CP_WARPS; ++w)
#pragma unroll
            for (int q = 0; q < A::NS; ++q) {
              TF.M[q] += sc.wf[w].M[q];
              TB.M[q] += sc.wb[w].M[q];
            }
          TF.D = TB.D = tot;
          TF.E = TB.E = fexp_neg(tot, s_tab);
          cs_put<A::NS>(aggs + 2 * t, TF);
          cs_put<A::NS>(aggs + 2 * t + 1, TB);
        }
      } else {
      // ---- forward: per-thread aggregate (direct form), warp scan, block carry, apply.
      {
        S X;
        double D = 0.0, Ee = 1.0;
#pragma unroll
        for (int q = 0; q < A::NS; ++q) X.M[q] = 0.0;
#pragma unroll
        for (int k = CP_ITEMS - 1; k >= 0; --k) {    // reference at item 7
          const int z = cpz(i0 + k);
          A::inject_at(X.M, E.rc[z] >> 30, uc[k], cp_aoff<A>(E, z), eak[k], D, Ee);
          D += E.d[z];
          Ee *= ek[k];
        }
        X.D = D; X.E = Ee;
#pragma unroll 1
        for (int off = 1; off < 32; off <<= 1) {
          const S Y = cs_shfl<A::NS>(X, off, true);
          if (lane >= off) X = cs_fw<A>(Y, X);
        }
        if (lane == 31) sc.wf[warp] = X;
        S ex = cs_shfl<A::NS>(X, 1, true);
        if (lane == 0) ex = cs_id<A>();
        if (MODE == 2) {
          if (tid < A::NS + 2) reinterpret_cast<double*>(&sc.cf)[tid] = cvf;
          if (tid >= 32 && tid < 32 + A::NS + 2) reinterpret_cast<double*>(&sc.cb)[tid - 32] = cvb;
        }
        __syncthreads();
        if (MODE == 1) {
          if (tid == 0) {
            S T = sc.wf[0];
#pragma unroll 1
            for (int w = 1; w < CP_WARPS; ++w) T = cs_fw<A>(T, sc.wf[w]);
            cs_put<A::NS>(aggs + 2 * t, T);
          }
        } else {
          S C = sc.cf;
#pragma unroll 1
          for (int w = 0; w < warp; ++w) C = cs_fw<A>(C, sc.wf[w]);
          C = cs_fw<A>(C, ex);
          double M[A::NS];
#pragma unroll
          for (int q = 0; q < A::NS; ++q) M[q] = C.M[q];
#pragma unroll
          for (int k = 0; k < CP_ITEMS; ++k) {
            const int z = cpz(i0 + k);
            A::advance_all(M, E.d[z], ek[k]);
            const int ch = E.rc[z] >> 30;
            const double a = cp_aoff<A>(E, z), ea = eak[k];
            of[k] = A::read(M, A::NCH - 1 - ch, a, ea);
            A::inject(M, ch, uc[k], a, ea);
          }
        }
      }
      // ---- backward
      {
        S X;
        double D = 0.0, Ee = 1.0;
#pragma unroll
        for (int q = 0; q < A::NS; ++q) X.M[q] = 0.0;
#pragma unroll
        for (int k = 0; k < CP_ITEMS; ++k) {         // reference just before item 0
          const int z = cpz(i0 + k);
          D += E.d[z];
          Ee *= ek[k];
          A::inject_at(X.M, E.rc[z] >> 30, uc[k], cp_aoff<A>(E, z), eak[k], D, Ee);
        }
        X.D = D; X.E = Ee;
#pragma unroll 1
        for (int off = 1; off < 32; off <<= 1) {
          const S Y = cs_shfl<A::NS>(X, off, false);
          if (lane + off < 32) X = cs_bw<A>(X, Y);
        }
        if (lane == 0) sc.wb[warp] = X;
        S ex = cs_shfl<A::NS>(X, 1, false);
        if (lane == 31) ex = cs_id<A>();
        __syncthreads();
        if (MODE == 1) {
          if (tid == 0) {
            S T = sc.wb[CP_WARPS - 1];
#pragma unroll 1
            for (int w = CP_WARPS - 2; w >= 0; --w) T = cs_bw<A>(sc.wb[w], T);
            cs_put<A::NS>(aggs + 2 * t + 1, T);
          }
        } else {
          S C = sc.cb;
#pragma unroll 1
          for (int w = CP_WARPS - 1; w > warp; --w) C = cs_bw<A>(sc.wb[w], C);
          C = cs_bw<A>(ex, C);
          double M[A::NS];
#pragma unroll
          for (int q = 0; q < A::NS; ++q) M[q] = C.M[q];
          double* slot = g.part + (int64_t)c * g.part_stride + (int64_t)p * g.n;
#pragma unroll
          for (int k = CP_ITEMS - 1; k >= 0; --k) {
            const int z = cpz(i0 + k);
            const unsigned rcz = E.rc[z];
            const int ch = rcz >> 30;
            const double a = cp_aoff<A>(E, z), ea = eak[k];
            const double val = of[k] + A::read(M, A::NCH - 1 - ch, a, ea);
            A::inject(M, ch, uc[k], a, ea);
            A::advance_all(M, E.d[z], ek[k]);
            const unsigned r = rcz & CP_RMASK;
            if constexpr (A::P3) {
              tot[k] = fma(val, A::tgtw(E.a[z], cp_a2<A>(E, z), ab), tot[k]);
              if (ab == A::NAB - 1 && r != CP_RMASK) slot[r] = tot[k];
            } else {
              if (r != CP_RMASK) slot[r] = val;
            }
          }
        }
      }
      }
      __syncthreads();                               // scratch reuse by the next column
    }
    // stage sidx is free: load tile item + 2G into it
    if (tid == 0 && item + 2 * G < total) {
      fence_proxy_async_smem();
      p_iss = cp_pass_at(descs, npass, p_iss, item + 2 * G);
      cp_issue(hpbase, descs, p_iss, item + 2 * G, E, &bar[sidx]);
    }
  }
}

// ---------------------------------------------------------------------------
// Host side.
static size_t lv_smem_fused() { return sizeof(LvPoints); }

template <class A>
static cudaError_t lv_set_attrs() {
  cudaError_t e;
  const int fused = (int)lv_smem_fused();
  if constexpr (A::NCH == 2) {   // d = 2
    if ((e = cudaFuncSetAttribute(k_low2<A>, cudaFuncAttributeMaxDynamicSharedMemorySize, fused)))
      return e;
  } else {                       // d = 3
    if ((e = cudaFuncSetAttribute(k_low3<A>, cudaFuncAttributeMaxDynamicSharedMemorySize, fused)))
      return e;
    if ((e = cudaFuncSetAttribute(k_mid3<A>, cudaFuncAttributeMaxDynamicSharedMemorySize, fused)))
      return e;
  }
  if ((e = cudaFuncSetAttribute(k_cp<A, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(CpSmemT<A::ST2>))))
    return e;
  return cudaFuncSetAttribute(k_cp<A, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)sizeof(CpSmemT<A::ST2>));
}

#if GPM_LEVEL_PART == 0
// The carried passes of a plan, in apply order: (ord, ord2l1, lseg, l1, n_act).
struct HPass {
  const int* ord;
  const int* ord2l1;
  int lseg, l1;
  int64_t nact;
};
static std::vector<HPass> high_passes(const Plan& pl) {
  std::vector<HPass> v;
  const int64_t n = pl.n;
  for (int l1 = LV_LOGTILE + 1; l1 <= pl.L; ++l1) {
    const int64_t b_last = (n - 1) >> l1;
    const int64_t mid1 = (b_last << l1) + (int64_t(1) << (l1 - 1));
    const int64_t nact1 = mid1 >= n ? (b_last << l1) : n;
    if (pl.d == 2) {
      if (nact1 > 0) v.push_back({pl.ord2.as<int>() + (size_t)(l1 - 1) * n, nullptr, l1, l1, nact1});
    } else {
      for (int l2 = LV_LOGTILE + 1; l2 <= l1; ++l2) {
        const int64_t c_last = (n - 1) >> l2;
        const int64_t mid2 = (c_last << l2) + (int64_t(1) << (l2 - 1));
        int64_t nact = nact1;
        if (mid2 >= n) nact = std::min(nact, c_last << l2);
        if (nact > 0)
          v.push_back({pl.ord3.as<int>() + ((size_t)(l1 - 1) * l1 / 2 + (l2 - 1)) * n,
                       pl.ord2.as<int>() + (size_t)(l1 - 1) * n, l2, l1, nact});
      }
    }
  }
  return v;
}

// d = 3 product form with nu >= 3/2: the (a, b) sub-passes of algebra.cuh (P3)
bool level_p3(const Plan& pl) { return pl.d == 3 && pl.form == GP_FORM_PRODUCT && pl.P > 0; }
// most sub-passes per column over the plan's applies (value and gradient runs): sizes aggs
int level_nab(const Plan& pl) {
  if (pl.form != GP_FORM_PRODUCT || pl.d < 2) return 1;
  return pl.d == 3 ? (pl.P + 2) * (pl.P + 2) : pl.P + 2;
}
// runs per apply whose outputs the epilogue sums: the separated gradients take two
int level_phases(const Plan& pl, int kind) {
  if (kind == 0 || pl.form != GP_FORM_PRODUCT) return 1;
  return (pl.d == 3 && pl.P > 0) || (pl.d == 2 && pl.P > 3) ? 2 : 1;
}

static LvArgs lv_base_args(const Plan& pl) {
  LvArgs g{};
  const int64_t n = pl.n;
  g.ord2 = pl.ord2.as<int>();
  g.ord3 = pl.ord3.as<int>();
  g.t1 = pl.t.as<double>();
  g.t2 = pl.t.as<double>() + n;
  g.t3 = pl.d == 3 ? pl.t.as<double>() + 2 * n : nullptr;
  g.n = n;
  g.L = pl.L;
  g.mode = pl.d;
  return g;
}

// setup: stage the structure of every carried pass (lv_elem reads t through pts, which
// the caller packs first)
gp_status level_setup(Plan& pl, cudaStream_t s) {
  if (pl.d < 2) return GP_OK;
  if (!pl.s2) {
    GPM_CUDA(cudaStreamCreateWithFlags(&pl.s2, cudaStreamNonBlocking));
    GPM_CUDA(cudaEventCreateWithFlags(&pl.ev_fork, cudaEventDisableTiming));
    GPM_CUDA(cudaEventCreateWithFlags(&pl.ev_join, cudaEventDisableTiming));
    GPM_CUDA(cudaStreamCreateWithFlags(&pl.s3, cudaStreamNonBlocking));
    GPM_CUDA(cudaEventCreateWithFlags(&pl.ev_join3, cudaEventDisableTiming));
  }
  const std::vector<HPass> hp = high_passes(pl);
  const bool p3 = level_p3(pl);
  size_t total = 0;
  for (const HPass& h : hp) total += hp_bytes(h.nact, p3);
  if (total == 0) return GP_OK;
  GPM_TRY(pl.hpbuf.alloc(total));
  {
    std::vector<HpDesc> dv;
    size_t o = 0;
    int mt = 0;
    int items = 0;
    for (const HPass& h : hp) {
      const int nt = (int)((h.nact + LV_TILE - 1) / LV_TILE);
      dv.push_back({(int64_t)o, h.nact, h.lseg, nt, items, 0});
      o += hp_bytes(h.nact, p3);
      mt = std::max(mt, nt);
      items += nt;
    }
    pl.hp_items = items;
    pl.hp_tail.clear();
    for (const HPass& h : hp) pl.hp_tail.push_back(h.nact < pl.n ? 1 : 0);
    GPM_TRY(pl.hpdesc.alloc(sizeof(HpDesc) * dv.size()));
    GPM_CUDA(cudaMemcpy(pl.hpdesc.ptr, dv.data(), sizeof(HpDesc) * dv.size(), cudaMemcpyHostToDevice));
    pl.hp_npass = (int)dv.size();
    pl.hp_maxtiles = mt;
  }
  LvArgs g = lv_base_args(pl);
  g.pts = reinterpret_cast<const Pt4*>(pl.pts.ptr);
  size_t off = 0;
  for (const HPass& h : hp) {
    g.ord = h.ord;
    g.ord2l1 = h.ord2l1;
    g.lseg = h.lseg;
    g.l1 = h.l1;
    g.n_act = h.nact;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((hp_padded(h.nact) + 255) / 256, 148 * 8));
    k_hp_prep<<<grid, 256, 0, s>>>(g, pl.hpbuf.as<unsigned char>() + off, p3);
    GPM_CUDA(cudaGetLastError());
    off += hp_bytes(h.nact, p3);
  }
  pl.struct_bytes += (int64_t)total;
  return GP_OK;
}


// Sharded applies (gp_kmvm_partial): shard `shard` of `nshards` runs the
// tiles [T lo, T hi) of the tile kernels (k_low*, k_mid3) and the items [I lo, I hi) of the
// carried-pass apply (k_cp<2>); the carried-pass aggregates and carries (k_cp<1>,
// k_cp_carry) run whole on every shard.  Every pair lies in exactly one tile or item, so
// the shards' partial outputs sum to K v.
int64_t hp_item_count(int64_t n, int d) {
  int L = 0;
  while ((int64_t(1) << L) < n) ++L;
  int64_t items = 0;
  for (int l1 = LV_LOGTILE + 1; l1 <= L; ++l1) {
    const int64_t b_last = (n - 1) >> l1;
    const int64_t mid1 = (b_last << l1) + (int64_t(1) << (l1 - 1));
    const int64_t nact1 = mid1 >= n ? (b_last << l1) : n;
    if (d == 2) {
      if (nact1 > 0) items += (nact1 + LV_TILE - 1) / LV_TILE;
    } else {
      for (int l2 = LV_LOGTILE + 1; l2 <= l1; ++l2) {
        const int64_t c_last = (n - 1) >> l2;
        const int64_t mid2 = (c_last << l2) + (int64_t(1) << (l2 - 1));
        int64_t nact = nact1;
        if (mid2 >= n) nact = std::min(nact, c_last << l2);
        if (nact > 0) items += (nact + LV_TILE - 1) / LV_TILE;
      }
    }
  }
  return items;
}
void shard_ranges(int64_t n, int d, int shard, int nshards, int64_t* r) {
  const int64_t tiles = (n + LV_TILE - 1) / LV_TILE;
  const int64_t items = hp_item_count(n, d);
  r[0] = tiles * shard / nshards;
  r[1] = tiles * (shard + 1) / nshards;
  r[2] = items * shard / nshards;
  r[3] = items * (shard + 1) / nshards;
}

#endif   // GPM_LEVEL_PART == 0

template <class A>
static gp_status lv_run(Plan& pl, int nrhs, cudaStream_t s, int* launches) {
  static bool attr = false;
  if (!attr) {
    GPM_CUDA(lv_set_attrs<A>());
    attr = true;
  }
  const int64_t n = pl.n;
  const int L = pl.L;
  LvArgs g{};
  g.ord2 = pl.ord2.as<int>();
  g.ord3 = pl.ord3.as<int>();
  g.t1 = pl.t.as<double>();
  g.t2 = pl.t.as<double>() + n;
  g.t3 = pl.d == 3 ? pl.t.as<double>() + 2 * n : nullptr;
  g.u = nullptr;
  g.pts = reinterpret_cast<const Pt4*>(pl.pts.ptr);
  g.lb = pl.d == 2 ? pl.near_lb2 : pl.near_lb3;
  const bool multi2 = A::NCH == 2 && nrhs >= 2 && !getenv("GPM_LOW2_PERCOL");
  g.lb2 = pl.near_lb3m;
  g.acc = pl.acc.as<double>();
  g.aggs = pl.aggs.as<LvAgg>();
  g.n = n;
  g.L = L;
  g.mode = pl.d;
  const int tiles = (int)((n + LV_TILE - 1) / LV_TILE);
  g.agg_stride = 2 * (int64_t)tiles * std::max(1, pl.hp_npass);
  g.part = pl.part.as<double>();
  g.npass = pl.hp_npass;
  g.part_stride = (int64_t)level_nparts(pl) * n;
  int64_t sr[4] = {0, tiles, 0, pl.hp_items};   // tile range, carried-pass item range
  if (pl.nshards > 1) {
    shard_ranges(n, pl.d, pl.shard, pl.nshards, sr);
    if (sr[3] - sr[2] != 0 && pl.hp_items != hp_item_count(n, pl.d))
      return fail(GP_ERR_CUDA, "internal: carried-pass item count mismatch");
    // points outside this shard's tiles / items get no contribution: start from zero
    GPM_CUDA(cudaMemsetAsync(g.acc, 0, sizeof(double) * n * nrhs, s));
    if (level_nparts(pl) > 0)
      GPM_CUDA(cudaMemsetAsync(g.part, 0, sizeof(double) * g.part_stride * nrhs, s));
  }
  g.tile0 = (int)sr[0];
  const int tiles_run = (int)(sr[1] - sr[0]);
  const int nlow_alloc = low_parts(pl.d, pl.d == 2 ? pl.near_lb2 : pl.near_lb3, L);   // level_nparts
  const int nlow = low_parts(pl.d, g.lb, L);
  // trailing part slots this apply leaves unwritten (the epilogue skips them)
  pl.low_unused = nlow_alloc - nlow;
  g.low_slot0 = pl.hp_npass + (pl.d == 3 ? std::max(0, L - LV_LOGTILE) : 0);
  const dim3 gt(tiles_run, nrhs, nlow);
  const bool hp = pl.hp_npass > 0;
  const HpDesc* dd = pl.hpdesc.as<HpDesc>();
  static int grid1 = 0, grid2 = 0;   // persistent k_cp: as many CTAs as fit (per instantiation)
  if (hp && !grid1) {
    int dev = 0, sms = 0, o1 = 0, o2 = 0;
    GPM_CUDA(cudaGetDevice(&dev));
    GPM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    GPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_cp<A, 1>, CP_BLOCK, sizeof(CpSmemT<A::ST2>)));
    GPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_cp<A, 2>, CP_BLOCK, sizeof(CpSmemT<A::ST2>)));
    grid1 = std::max(1, o1) * sms;
    grid2 = std::max(1, o2) * sms;
  }
  if (hp) {
    // ranks past a pass's active range are never written: zero those slots once per buffer
    for (int c = pl.part_zero_cols; c < nrhs; ++c)
      for (int p = 0; p < pl.hp_npass; ++p)
        if (pl.hp_tail[p])
          GPM_CUDA(cudaMemsetAsync(g.part + c * g.part_stride + (int64_t)p * n, 0,
                                   sizeof(double) * n, s));
    pl.part_zero_cols = std::max(pl.part_zero_cols, nrhs);
    // the carried-pass tile aggregates do not depend on the low levels: side stream
    GPM_CUDA(cudaEventRecord(pl.ev_fork, s));
    GPM_CUDA(cudaStreamWaitEvent(pl.s2, pl.ev_fork, 0));
    const int64_t carr_off = (int64_t)g.agg_stride * nrhs * A::NAB;   // carries after the aggregates
    k_cp<A, 1><<<std::min(pl.hp_items, grid1), CP_BLOCK, sizeof(CpSmemT<A::ST2>), pl.s2>>>(
        g, pl.hpbuf.as<unsigned char>(), dd, pl.hp_npass, pl.hp_items, pl.hp_maxtiles, nrhs,
        carr_off, 0);
    GPM_CUDA(cudaGetLastError());
    LvRecFor<A::NS>* recs = reinterpret_cast<LvRecFor<A::NS>*>(g.aggs);
    // grid.x covers the level-11 nodes (two tiles each, CC_WARPS nodes per CTA)
    k_cp_carry<A><<<dim3((pl.hp_maxtiles + 2 * CC_WARPS - 1) / (2 * CC_WARPS), pl.hp_npass,
                         2 * nrhs * A::NAB),
                    32 * CC_WARPS, 0, pl.s2>>>(
        recs, recs + carr_off, dd, pl.hp_npass, pl.hp_maxtiles);
    GPM_CUDA(cudaGetLastError());
    // the carried-pass apply follows on the side stream too (it only needs the aggregates
    // and carries): its tail overlaps the tile kernels' (config 4 2.02 -> 1.99 ms;
    // GPM_CP2_SIDE=0 puts it back on the main stream after the tile kernels)
    static const int cp2_side = getenv("GPM_CP2_SIDE") ? atoi(getenv("GPM_CP2_SIDE")) : 1;
    if (cp2_side) {
      const int nit = (int)(sr[3] - sr[2]);
      if (nit > 0) {
        k_cp<A, 2><<<std::min(nit, grid2), CP_BLOCK, sizeof(CpSmemT<A::ST2>), pl.s2>>>(
            g, pl.hpbuf.as<unsigned char>(), dd, pl.hp_npass, (int)sr[3], pl.hp_maxtiles, nrhs,
            (int64_t)g.agg_stride * nrhs * A::NAB, (int)sr[2]);
        *launches += 1;
        GPM_CUDA(cudaGetLastError());
      }
    }
    GPM_CUDA(cudaEventRecord(pl.ev_join, pl.s2));
    *launches += 2;
  }
  // fused low levels (writes acc for every point of its tiles)
  if (tiles_run <= 0) {
    // this shard has no tiles
  } else if constexpr (A::NCH == 2) {
    if (multi2) {   // columns share the v-independent work
#ifndef GPM_LOW2M_NC
#define GPM_LOW2M_NC 4
#endif
      constexpr int NC = GPM_LOW2M_NC;
      static bool attr = false;
      if (!attr) {
        GPM_CUDA(cudaFuncSetAttribute(k_low2m<A, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)sizeof(LvPointsM<NC>)));
        attr = true;
      }
      // two CTAs per SM (80 KB of staged columns each): the parts only pay while the grid
      // leaves SMs empty
      const int groups = (nrhs + NC - 1) / NC;
      const bool msplit = (int64_t)tiles_run * groups < 148;
      if (!msplit) pl.low_unused = nlow_alloc - 1;
      k_low2m<A, NC><<<dim3(tiles_run, groups, msplit ? nlow : 1), CP_BLOCK, sizeof(LvPointsM<NC>), s>>>(
          g, nrhs);
    } else {
      k_low2<A><<<gt, CP_BLOCK, lv_smem_fused(), s>>>(g);
    }
    *launches += 1;
    GPM_CUDA(cudaGetLastError());
  } else {
    k_low3<A><<<gt, CP_BLOCK, lv_smem_fused(), s>>>(g);
    *launches += 1;
    GPM_CUDA(cudaGetLastError());
    if (L > LV_LOGTILE) {   // d = 3: every outer level l1 > 10 (inner l2 <= 10)
      g.l1 = LV_LOGTILE + 1;
      // k_mid3 does not depend on k_low3: while the grids are small (up to two waves of tiles)
      // it runs beside it on a stream of its own (d = 3, n = 2^14: 108 -> 67 us; at config 4's
      // size the kernels fill the GPU either way).  GPM_MID3_SIDE = 0 / 1 forces it off / on.
      static const int mid_env = getenv("GPM_MID3_SIDE") ? atoi(getenv("GPM_MID3_SIDE")) : -1;
      const bool mid_side = mid_env >= 0 ? mid_env != 0 : tiles_run <= 296;
      cudaStream_t sm = s;
      if (mid_side && hp && pl.s3) {   // (ev_fork is recorded on s whenever hp)
        GPM_CUDA(cudaStreamWaitEvent(pl.s3, pl.ev_fork, 0));
        sm = pl.s3;
      }
      k_mid3<A><<<dim3(tiles_run, nrhs, L - LV_LOGTILE), CP_BLOCK, lv_smem_fused(), sm>>>(g);
      *launches += 1;
      GPM_CUDA(cudaGetLastError());
      if (sm != s) {
        GPM_CUDA(cudaEventRecord(pl.ev_join3, pl.s3));
        GPM_CUDA(cudaStreamWaitEvent(s, pl.ev_join3, 0));
      }
    }
  }
  if (hp) {   // carried-pass apply (needs the aggregates)
    GPM_CUDA(cudaStreamWaitEvent(s, pl.ev_join, 0));
    static const int cp2_side = getenv("GPM_CP2_SIDE") ? atoi(getenv("GPM_CP2_SIDE")) : 1;
    const int nit = cp2_side ? 0 : (int)(sr[3] - sr[2]);
    if (nit > 0) {
      k_cp<A, 2><<<std::min(nit, grid2), CP_BLOCK, sizeof(CpSmemT<A::ST2>), s>>>(
          g, pl.hpbuf.as<unsigned char>(), dd, pl.hp_npass, (int)sr[3], pl.hp_maxtiles, nrhs,
          (int64_t)g.agg_stride * nrhs * A::NAB, (int)sr[2]);
      *launches += 1;
      GPM_CUDA(cudaGetLastError());
    }
  }
  return GP_OK;
}

#if GPM_LEVEL_PART == 0
// per-pass contribution slots: carried passes, then (d = 3) one per outer level l1 > 10, then
// the parts 1.. of the fused low kernels
int level_nparts(const Plan& pl) {
  return pl.hp_npass + (pl.d == 3 ? std::max(0, pl.L - LV_LOGTILE) : 0) +
         low_parts(pl.d, pl.d == 2 ? pl.near_lb2 : pl.near_lb3, pl.L) - 1;
}

// pack the rank-order point records (t1, t2, t3, u) used by every level kernel
__global__ void k_pack(const double* __restrict__ t, int64_t n, int d,
                       const int* __restrict__ perm, const double* __restrict__ v, int64_t n_src,
                       int64_t vstride, Pt4* __restrict__ pts) {
  v += blockIdx.y * vstride;
  pts += blockIdx.y * n;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    Pt4 p;
    p.t1 = t[r];
    p.t2 = t[n + r];
    p.t3 = d == 3 ? t[2 * n + r] : 0.0;
    if (perm) {
      const int i = __ldg(perm + r);
      p.u = i < n_src ? __ldcg(v + i) : 0.0;
    } else {
      p.u = v[r];
    }
    pts[r] = p;
  }
}

gp_status level_pack(Plan& pl, const double* v, int nrhs, bool user_order, cudaStream_t s) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((pl.n + 255) / 256, 148 * 8));
  const int64_t vstride = user_order ? pl.n_src : pl.n;
  k_pack<<<dim3(grid, nrhs), 256, 0, s>>>(pl.t.as<double>(), pl.n, pl.d,
                                          user_order ? pl.perm.as<int>() : nullptr, v,
                                          user_order ? pl.n_src : pl.n, vstride,
                                          reinterpret_cast<Pt4*>(pl.pts.ptr));
  GPM_CUDA(cudaGetLastError());
  return GP_OK;
}
size_t level_pt_bytes() { return sizeof(Pt4); }

#endif   // GPM_LEVEL_PART == 0

// Dispatch on the algebra.  Every part defines its own share of the instantiations.
#if GPM_LEVEL_PART == 0
gp_status level_passes(Plan& pl, int nrhs, cudaStream_t s, int* launches, int kind, int phase) {
  const bool prod = pl.form == GP_FORM_PRODUCT;
  const int P = pl.P;
#ifdef GPM_FEW   // experiment builds (build.py GPM_EXTRA_FLAGS): the three bench algebras only
  if (kind == 0 && pl.d == 2 && P == 1 && !prod) return lv_run<Alg<1, 2, false>>(pl, nrhs, s, launches);
  if (kind == 0 && pl.d == 2 && P == 1 && prod) return lv_run<Alg<1, 2, true>>(pl, nrhs, s, launches);
  if (kind == 0 && pl.d == 3 && P == 2 && !prod) return level_passes_p2(pl, nrhs, s, launches, kind, phase);
  return fail(GP_ERR_UNSUPPORTED, "GPM_FEW experiment build");
#else
  if (pl.d == 3) return kind != 0 ? level_passes_p3(pl, nrhs, s, launches, kind, phase)
                                  : level_passes_p2(pl, nrhs, s, launches, kind, phase);
  if (kind != 0) return level_passes_p1(pl, nrhs, s, launches, kind, phase);
  if (!prod) {
    switch (P) {
      case 0: return lv_run<Alg<0, 2, false>>(pl, nrhs, s, launches);
      case 1: return lv_run<Alg<1, 2, false>>(pl, nrhs, s, launches);
      case 2: return lv_run<Alg<2, 2, false>>(pl, nrhs, s, launches);
      case 3: return lv_run<Alg<3, 2, false>>(pl, nrhs, s, launches);
      default: return lv_run<Alg<4, 2, false>>(pl, nrhs, s, launches);
    }
  }
  if (P == 0) return lv_run<Alg<0, 2, true>>(pl, nrhs, s, launches);
  if (P == 1) return lv_run<Alg<1, 2, true>>(pl, nrhs, s, launches);
  if (P == 2) return lv_run<Alg<2, 2, true>>(pl, nrhs, s, launches);
  if (P == 3) return lv_run<Alg<3, 2, true>>(pl, nrhs, s, launches);
  return lv_run<Alg<4, 2, true>>(pl, nrhs, s, launches);
#endif
}
#elif GPM_LEVEL_PART == 1
// d = 2 lengthscale gradients: moment order p + 1
gp_status level_passes_p1(Plan& pl, int nrhs, cudaStream_t s, int* launches, int kind, int phase) {
#ifdef GPM_FEW
  return fail(GP_ERR_UNSUPPORTED, "GPM_FEW experiment build");
#else
  const bool prod = pl.form == GP_FORM_PRODUCT;
  const int P = pl.P;
  if (prod && level_phases(pl, kind) == 2)
    // separated product-form gradient (algebra.cuh SEP 2 / SEP 3) at nu = 9/2, whose
    // mixed-moment state would need 2 x 36 doubles
    return phase == 0 ? lv_run<Alg<4, 2, false, 0, 2>>(pl, nrhs, s, launches)
                      : lv_run<Alg<5, 2, false, 1, 3>>(pl, nrhs, s, launches);
  if (prod) {        // product form, nu <= 7/2 ((p+2)^2 moments per channel)
    if (P == 0) return lv_run<Alg<1, 2, true, 1>>(pl, nrhs, s, launches);
    if (P == 1) return lv_run<Alg<2, 2, true, 1>>(pl, nrhs, s, launches);
    if (P == 2) return lv_run<Alg<3, 2, true, 1>>(pl, nrhs, s, launches);
    return lv_run<Alg<4, 2, true, 1>>(pl, nrhs, s, launches);
  }
  switch (P) {
    case 0: return lv_run<Alg<1, 2, false, 1>>(pl, nrhs, s, launches);
    case 1: return lv_run<Alg<2, 2, false, 1>>(pl, nrhs, s, launches);
    case 2: return lv_run<Alg<3, 2, false, 1>>(pl, nrhs, s, launches);
    case 3: return lv_run<Alg<4, 2, false, 1>>(pl, nrhs, s, launches);
    default: return lv_run<Alg<5, 2, false, 1>>(pl, nrhs, s, launches);
  }
#endif
}
#elif GPM_LEVEL_PART == 2
// d = 3 values: the L1 form, and the product form by the separated sub-passes (SEP 1)
gp_status level_passes_p2(Plan& pl, int nrhs, cudaStream_t s, int* launches, int kind, int phase) {
  const int P = pl.P;
#ifdef GPM_FEW
  if (P == 2 && !level_p3(pl)) return lv_run<Alg<2, 4, false>>(pl, nrhs, s, launches);
  return fail(GP_ERR_UNSUPPORTED, "GPM_FEW experiment build");
#else
  if (level_p3(pl)) {   // product form (nu = 1/2 is the L1 kernel)
    switch (P) {
      case 1: return lv_run<Alg<1, 4, false, 0, 1>>(pl, nrhs, s, launches);
      case 2: return lv_run<Alg<2, 4, false, 0, 1>>(pl, nrhs, s, launches);
      case 3: return lv_run<Alg<3, 4, false, 0, 1>>(pl, nrhs, s, launches);
      default: return lv_run<Alg<4, 4, false, 0, 1>>(pl, nrhs, s, launches);
    }
  }
  switch (P) {
    case 0: return lv_run<Alg<0, 4, false>>(pl, nrhs, s, launches);
    case 1: return lv_run<Alg<1, 4, false>>(pl, nrhs, s, launches);
    case 2: return lv_run<Alg<2, 4, false>>(pl, nrhs, s, launches);
    case 3: return lv_run<Alg<3, 4, false>>(pl, nrhs, s, launches);
    default: return lv_run<Alg<4, 4, false>>(pl, nrhs, s, launches);
  }
#endif
}
#else
// d = 3 lengthscale gradients: L1 with one more moment; product form in two separated runs
gp_status level_passes_p3(Plan& pl, int nrhs, cudaStream_t s, int* launches, int kind, int phase) {
#ifdef GPM_FEW
  return fail(GP_ERR_UNSUPPORTED, "GPM_FEW experiment build");
#else
  const int P = pl.P;
  if (level_phases(pl, kind) == 2) {
    switch (P) {
      case 1: return phase == 0 ? lv_run<Alg<1, 4, false, 0, 2>>(pl, nrhs, s, launches)
                                : lv_run<Alg<2, 4, false, 1, 3>>(pl, nrhs, s, launches);
      case 2: return phase == 0 ? lv_run<Alg<2, 4, false, 0, 2>>(pl, nrhs, s, launches)
                                : lv_run<Alg<3, 4, false, 1, 3>>(pl, nrhs, s, launches);
      case 3: return phase == 0 ? lv_run<Alg<3, 4, false, 0, 2>>(pl, nrhs, s, launches)
                                : lv_run<Alg<4, 4, false, 1, 3>>(pl, nrhs, s, launches);
      default: return phase == 0 ? lv_run<Alg<4, 4, false, 0, 2>>(pl, nrhs, s, launches)
                                 : lv_run<Alg<5, 4, false, 1, 3>>(pl, nrhs, s, launches);
    }
  }
  switch (P) {
    case 0: return lv_run<Alg<1, 4, false, 1>>(pl, nrhs, s, launches);
    case 1: return lv_run<Alg<2, 4, false, 1>>(pl, nrhs, s, launches);
    case 2: return lv_run<Alg<3, 4, false, 1>>(pl, nrhs, s, launches);
    case 3: return lv_run<Alg<4, 4, false, 1>>(pl, nrhs, s, launches);
    default: return lv_run<Alg<5, 4, false, 1>>(pl, nrhs, s, launches);   // 4 x 6 moments (LvRec<24>)
  }
#endif
}
#endif

#if GPM_LEVEL_PART == 0
int64_t level_tiles(int64_t n) { return (n + LV_TILE - 1) / LV_TILE; }
#endif   // GPM_LEVEL_PART == 0

}  // namespace gpm
