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
// Kernel layout: tile = 2048 positions per 256-thread CTA; element data
// staged in shared memory (padded, conflict-free); per-thread sequential recurrences,
// warp-shuffle block scans with segment flags; segments longer than a tile get carries
// from a tile-aggregate kernel (a reduce-then-scan across the tiles of one segment).
#include <algorithm>

#include "algebra.cuh"
#include "internal.h"

namespace gpm {

__device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t lmax(int64_t a, int64_t b) { return a > b ? a : b; }

constexpr int LV_BLOCK = 256;
constexpr int LV_ITEMS = 8;
constexpr int LV_LOGTILE = 11;
constexpr int LV_TILE = 1 << LV_LOGTILE;  // == LV_BLOCK * LV_ITEMS
constexpr int LV_WARPS = LV_BLOCK / 32;
__host__ __device__ constexpr int lvpad(int i) { return i + (i >> 3); }
constexpr int LV_PADN = LV_TILE + LV_TILE / 8;

struct PassDesc {
  const int* ord;      // this pass's order (positions [0, n_act))
  const int* ord2l1;   // d = 3: ord2[l1] (position -> rank); d = 2: unused
  const double* t1;
  const double* t2;
  const double* t3;
  const double* u;     // rank-order input
  double* acc;         // rank-order accumulator
  LvAgg* aggs;         // [2 * tiles]
  int64_t n, n_act;
  int mode;            // 2 or 3
  int lseg;            // log2 of the segment (node) size of this pass
  int l1;              // d = 3: outer level
  int ntiles;
};

struct LvSmem {
  double d[LV_PADN];   // last coordinate y, then the gap Delta to the previous position
  double e[LV_PADN];   // e^{-Delta}
  double u[LV_PADN];   // source weight
  double a[LV_PADN];   // alpha = distance to the split reference(s)
  double ea[LV_PADN];  // e^{-alpha}
  int r[LV_TILE];      // rank of the point (output slot)
  signed char ch[LV_TILE];
};

template <int NS>
struct LSt {
  double D, E;
  double M[NS];
  int f;
};

template <class A>
__device__ __forceinline__ LSt<A::NS> lid() {
  LSt<A::NS> s;
  s.D = 0.0; s.E = 1.0; s.f = 0;
#pragma unroll
  for (int i = 0; i < A::NS; ++i) s.M[i] = 0.0;
  return s;
}

// forward (X left of Y): a segment start inside Y cuts X off
template <class A>
__device__ __forceinline__ LSt<A::NS> lcf(const LSt<A::NS>& X, const LSt<A::NS>& Y) {
  if (Y.f) return Y;
  LSt<A::NS> R;
#pragma unroll
  for (int i = 0; i < A::NS; ++i) R.M[i] = X.M[i];
  A::advance_all(R.M, Y.D, Y.E);
#pragma unroll
  for (int i = 0; i < A::NS; ++i) R.M[i] += Y.M[i];
  R.D = X.D + Y.D; R.E = X.E * Y.E; R.f = X.f;
  return R;
}
// backward (X left of Y): a segment end inside X cuts Y off
template <class A>
__device__ __forceinline__ LSt<A::NS> lcb(const LSt<A::NS>& X, const LSt<A::NS>& Y) {
  if (X.f) return X;
  LSt<A::NS> R;
#pragma unroll
  for (int i = 0; i < A::NS; ++i) R.M[i] = Y.M[i];
  A::advance_all(R.M, X.D, X.E);
#pragma unroll
  for (int i = 0; i < A::NS; ++i) R.M[i] += X.M[i];
  R.D = X.D + Y.D; R.E = X.E * Y.E; R.f = Y.f;
  return R;
}

template <int NS>
__device__ __forceinline__ LSt<NS> lshfl(const LSt<NS>& s, int off, bool up) {
  LSt<NS> r;
  if (up) {
    r.D = __shfl_up_sync(0xffffffffu, s.D, off);
    r.E = __shfl_up_sync(0xffffffffu, s.E, off);
    r.f = __shfl_up_sync(0xffffffffu, s.f, off);
#pragma unroll
    for (int i = 0; i < NS; ++i) r.M[i] = __shfl_up_sync(0xffffffffu, s.M[i], off);
  } else {
    r.D = __shfl_down_sync(0xffffffffu, s.D, off);
    r.E = __shfl_down_sync(0xffffffffu, s.E, off);
    r.f = __shfl_down_sync(0xffffffffu, s.f, off);
#pragma unroll
    for (int i = 0; i < NS; ++i) r.M[i] = __shfl_down_sync(0xffffffffu, s.M[i], off);
  }
  return r;
}

template <int NS>
__device__ __forceinline__ void agg_put(LvAgg* g, const LSt<NS>& s) {
  g->D = s.D; g->E = s.E; g->flag = s.f;
#pragma unroll
  for (int i = 0; i < NS; ++i) g->M[i] = s.M[i];
}
template <int NS>
__device__ __forceinline__ LSt<NS> agg_get(const LvAgg* g) {
  LSt<NS> s;
  s.D = __ldcg(&g->D); s.E = __ldcg(&g->E); s.f = __ldcg(&g->flag);
#pragma unroll
  for (int i = 0; i < NS; ++i) s.M[i] = __ldcg(&g->M[i]);
  return s;
}

// Block-wide exclusive scan in one direction (FWD: threads < me; else threads > me),
// plus the tile total.  Uses shared warp totals; ends with a barrier.
template <class A, bool FWD>
__device__ __forceinline__ void lv_block_scan(const LSt<A::NS>& mine, LSt<A::NS>& excl,
                                              LSt<A::NS>& tot, LSt<A::NS>* s_w,
                                              LSt<A::NS>* s_wx, LSt<A::NS>* s_tot) {
  using S = LSt<A::NS>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  S x = mine;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    if (FWD) {
      S l = lshfl<A::NS>(x, off, true);
      if (lane >= off) x = lcf<A>(l, x);
    } else {
      S r = lshfl<A::NS>(x, off, false);
      if (lane + off < 32) x = lcb<A>(x, r);
    }
  }
  if (FWD && lane == 31) s_w[warp] = x;
  if (!FWD && lane == 0) s_w[warp] = x;
  S ex = lshfl<A::NS>(x, 1, FWD);
  if ((FWD && lane == 0) || (!FWD && lane == 31)) ex = lid<A>();
  __syncthreads();
  if (warp == 0) {
    S y = lane < LV_WARPS ? s_w[lane] : lid<A>();
#pragma unroll
    for (int off = 1; off < LV_WARPS; off <<= 1) {
      if (FWD) {
        S l = lshfl<A::NS>(y, off, true);
        if (lane >= off) y = lcf<A>(l, y);
      } else {
        S r = lshfl<A::NS>(y, off, false);
        if (lane + off < 32) y = lcb<A>(y, r);
      }
    }
    S ye = lshfl<A::NS>(y, 1, FWD);
    if ((FWD && lane == 0) || (!FWD && lane >= LV_WARPS - 1)) ye = lid<A>();
    if (lane < LV_WARPS) s_wx[lane] = ye;
    if (FWD && lane == LV_WARPS - 1) *s_tot = y;
    if (!FWD && lane == 0) *s_tot = y;
  }
  __syncthreads();
  excl = FWD ? lcf<A>(s_wx[warp], ex) : lcb<A>(ex, s_wx[warp]);
  tot = *s_tot;
  __syncthreads();
}

// Element of a pass at position pos: scan coordinate y, weight u, split offset alpha,
// channel, rank.
struct Elem {
  double y, u, a;
  int r, ch;
};

__device__ __forceinline__ Elem lv_elem(const PassDesc& pd, int64_t pos) {
  Elem el;
  if (pd.mode == 2) {
    const int l = pd.lseg;
    const int r = __ldg(pd.ord + pos);
    const int64_t mid = ((pos >> l) << l) + (int64_t(1) << (l - 1));
    const double m = __ldg(pd.t1 + mid);
    el.a = fabs(__ldg(pd.t1 + r) - m);
    el.ch = (r >> (l - 1)) & 1;
    el.y = __ldg(pd.t2 + r);
    el.u = __ldg(pd.u + r);
    el.r = r;
  } else {
    const int l1 = pd.l1, l2 = pd.lseg;
    const int q = __ldg(pd.ord + pos);
    const int r = __ldg(pd.ord2l1 + q);
    const int64_t mid1 = ((int64_t)(q >> l1) << l1) + (int64_t(1) << (l1 - 1));
    const int64_t mid2 = ((pos >> l2) << l2) + (int64_t(1) << (l2 - 1));
    const double m1 = __ldg(pd.t1 + mid1);
    const double m2 = __ldg(pd.t2 + __ldg(pd.ord2l1 + mid2));
    el.a = fabs(__ldg(pd.t1 + r) - m1) + fabs(__ldg(pd.t2 + r) - m2);
    el.ch = 2 * ((r >> (l1 - 1)) & 1) + ((q >> (l2 - 1)) & 1);
    el.y = __ldg(pd.t3 + r);
    el.u = __ldg(pd.u + r);
    el.r = r;
  }
  return el;
}

__device__ __forceinline__ double lv_y(const PassDesc& pd, int64_t pos) {
  if (pd.mode == 2) return __ldg(pd.t2 + __ldg(pd.ord + pos));
  return __ldg(pd.t3 + __ldg(pd.ord2l1 + __ldg(pd.ord + pos)));
}

// KMODE 0: apply (segments fit in a tile), 1: tile aggregates only, 2: apply with carries
template <class A, int KMODE>
__global__ void __launch_bounds__(LV_BLOCK) k_level(PassDesc pd) {
  using S = LSt<A::NS>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LvSmem& sm = *reinterpret_cast<LvSmem*>(smem_raw);
  __shared__ S s_w[LV_WARPS], s_wx[LV_WARPS], s_tot;
  __shared__ double s_carry[2][A::NS];

  const int tid = threadIdx.x;
  const int64_t T0 = (int64_t)blockIdx.x * LV_TILE;
  const int cnt = (int)lmin(LV_TILE, pd.n_act - T0);
  const int64_t smask = (int64_t(1) << pd.lseg) - 1;

  // ---- tile carries (from the aggregate kernel), warp 0 forward / warp 1 backward
  if (KMODE == 2) {
    const int lane = tid & 31, warp = tid >> 5;
    if (warp < 2) {
      const int tps = 1 << (pd.lseg - LV_LOGTILE);
      const int t = blockIdx.x;
      const int first = t & ~(tps - 1);
      const int last = min(first + tps, pd.ntiles) - 1;
      const int lo = warp == 0 ? first : t + 1;
      const int hi = warp == 0 ? t : last + 1;
      const int cntc = max(0, hi - lo);
      const int per = (cntc + 31) / 32;
      S X = lid<A>();
      for (int k = 0; k < per; ++k) {
        const int j = lo + lane * per + k;
        if (j < hi) {
          S g = agg_get<A::NS>(pd.aggs + 2 * j + warp);
          X = warp == 0 ? lcf<A>(X, g) : lcb<A>(X, g);
        }
      }
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        S Y = lshfl<A::NS>(X, off, false);
        if (lane + off < 32) X = warp == 0 ? lcf<A>(X, Y) : lcb<A>(X, Y);
      }
      if (lane == 0) {
#pragma unroll
        for (int i = 0; i < A::NS; ++i) s_carry[warp][i] = X.M[i];
      }
    }
  }

  // ---- phase 0: element data into shared memory (coalesced over positions)
  for (int i = tid; i < cnt; i += LV_BLOCK) {
    const Elem el = lv_elem(pd, T0 + i);
    const int pi = lvpad(i);
    sm.d[pi] = el.y;
    sm.u[pi] = el.u;
    sm.a[pi] = el.a;
    sm.ea[pi] = exp(-el.a);
    sm.r[i] = el.r;
    sm.ch[i] = (signed char)el.ch;
  }
  __syncthreads();
  const int i0 = tid * LV_ITEMS;
  double yprev = 0.0;
  if (i0 < cnt) {
    const int64_t pos0 = T0 + i0;
    if ((pos0 & smask) == 0) yprev = sm.d[lvpad(i0)];
    else if (i0 > 0) yprev = sm.d[lvpad(i0 - 1)];
    else yprev = lv_y(pd, pos0 - 1);
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < LV_ITEMS; ++k) {
    const int i = i0 + k;
    if (i < cnt) {
      const int pi = lvpad(i);
      const double y = sm.d[pi];
      const double dl = (((T0 + i) & smask) == 0) ? 0.0 : y - yprev;
      yprev = y;
      sm.d[pi] = dl;
      sm.e[pi] = exp(-dl);
    }
  }
  __syncthreads();

  auto is_start = [&](int i) { return ((T0 + i) & smask) == 0; };
  auto is_end = [&](int i) { return (((T0 + i + 1) & smask) == 0) || (T0 + i == pd.n_act - 1); };

  // ---- forward direction
  S Fx, Ft;
  {
    S X = lid<A>();
#pragma unroll
    for (int k = 0; k < LV_ITEMS; ++k) {
      const int i = i0 + k;
      if (i < cnt) {
        const int pi = lvpad(i);
        if (is_start(i)) {
          X = lid<A>();
          X.f = 1;
        } else {
          A::advance_all(X.M, sm.d[pi], sm.e[pi]);
          X.D += sm.d[pi];
          X.E *= sm.e[pi];
        }
        A::inject(X.M, sm.ch[i], sm.u[pi], sm.a[pi], sm.ea[pi]);
      }
    }
    lv_block_scan<A, true>(X, Fx, Ft, s_w, s_wx, &s_tot);
  }
  if (KMODE == 1) {
    if (tid == 0) agg_put<A::NS>(pd.aggs + 2 * blockIdx.x, Ft);
  }
  double rf[LV_ITEMS];
  if (KMODE != 1) {
    S C = lid<A>();
    if (KMODE == 2) {
#pragma unroll
      for (int i = 0; i < A::NS; ++i) C.M[i] = s_carry[0][i];
    }
    const S Cin = lcf<A>(C, Fx);
    double M[A::NS];
#pragma unroll
    for (int i = 0; i < A::NS; ++i) M[i] = Cin.M[i];
#pragma unroll
    for (int k = 0; k < LV_ITEMS; ++k) {
      const int i = i0 + k;
      rf[k] = 0.0;
      if (i < cnt) {
        const int pi = lvpad(i);
        if (is_start(i)) {
#pragma unroll
          for (int j = 0; j < A::NS; ++j) M[j] = 0.0;
        } else {
          A::advance_all(M, sm.d[pi], sm.e[pi]);
        }
        const int c = sm.ch[i];
        rf[k] = A::read(M, A::NCH - 1 - c, sm.a[pi], sm.ea[pi]);
        A::inject(M, c, sm.u[pi], sm.a[pi], sm.ea[pi]);
      }
    }
  }

  // ---- backward direction
  S Bx, Bt;
  {
    S X = lid<A>();
#pragma unroll
    for (int k = LV_ITEMS - 1; k >= 0; --k) {
      const int i = i0 + k;
      if (i < cnt) {
        const int pi = lvpad(i);
        if (is_end(i)) {
          X = lid<A>();
          X.f = 1;
        }
        A::inject(X.M, sm.ch[i], sm.u[pi], sm.a[pi], sm.ea[pi]);
        A::advance_all(X.M, sm.d[pi], sm.e[pi]);
        X.D += sm.d[pi];
        X.E *= sm.e[pi];
      }
    }
    lv_block_scan<A, false>(X, Bx, Bt, s_w, s_wx, &s_tot);
  }
  if (KMODE == 1) {
    if (tid == 0) agg_put<A::NS>(pd.aggs + 2 * blockIdx.x + 1, Bt);
    return;
  }
  {
    S C = lid<A>();
    if (KMODE == 2) {
#pragma unroll
      for (int i = 0; i < A::NS; ++i) C.M[i] = s_carry[1][i];
    }
    const S Cin = lcb<A>(Bx, C);
    double M[A::NS];
#pragma unroll
    for (int i = 0; i < A::NS; ++i) M[i] = Cin.M[i];
#pragma unroll
    for (int k = LV_ITEMS - 1; k >= 0; --k) {
      const int i = i0 + k;
      if (i < cnt) {
        const int pi = lvpad(i);
        if (is_end(i)) {
#pragma unroll
          for (int j = 0; j < A::NS; ++j) M[j] = 0.0;
        }
        const int c = sm.ch[i];
        const double val = rf[k] + A::read(M, A::NCH - 1 - c, sm.a[pi], sm.ea[pi]);
        A::inject(M, c, sm.u[pi], sm.a[pi], sm.ea[pi]);
        A::advance_all(M, sm.d[pi], sm.e[pi]);
        const int r = sm.r[i];
        pd.acc[r] += val;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Host side: pass list and launches.

template <class A>
static cudaError_t lv_set_attr() {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k_level<A, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(LvSmem))))
    return e;
  if ((e = cudaFuncSetAttribute(k_level<A, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(LvSmem))))
    return e;
  return cudaFuncSetAttribute(k_level<A, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)sizeof(LvSmem));
}

template <class A>
static gp_status lv_launch_pass(PassDesc pd, cudaStream_t s, int* launches) {
  static bool attr = false;
  if (!attr) {
    GPM_CUDA(lv_set_attr<A>());
    attr = true;
  }
  const int tiles = (int)((pd.n_act + LV_TILE - 1) / LV_TILE);
  pd.ntiles = tiles;
  if (pd.lseg <= LV_LOGTILE) {
    k_level<A, 0><<<tiles, LV_BLOCK, sizeof(LvSmem), s>>>(pd);
    *launches += 1;
  } else {
    k_level<A, 1><<<tiles, LV_BLOCK, sizeof(LvSmem), s>>>(pd);
    k_level<A, 2><<<tiles, LV_BLOCK, sizeof(LvSmem), s>>>(pd);
    *launches += 2;
  }
  GPM_CUDA(cudaGetLastError());
  return GP_OK;
}

template <class A>
static gp_status lv_all_passes(Plan& pl, const double* u_rank, cudaStream_t s, int* launches) {
  const int64_t n = pl.n;
  const int L = pl.L;
  PassDesc pd;
  pd.t1 = pl.t.as<double>();
  pd.t2 = pl.t.as<double>() + n;
  pd.t3 = pl.d == 3 ? pl.t.as<double>() + 2 * n : nullptr;
  pd.u = u_rank;
  pd.acc = pl.acc.as<double>();
  pd.aggs = pl.aggs.as<LvAgg>();
  pd.n = n;
  pd.mode = pl.d;
  for (int l1 = 1; l1 <= L; ++l1) {
    // outer node activity: the last node has cross pairs only if its mid < n
    const int64_t b_last = (n - 1) >> l1;
    const int64_t mid1 = (b_last << l1) + (int64_t(1) << (l1 - 1));
    const int64_t nact1 = mid1 >= n ? (b_last << l1) : n;
    if (pl.d == 2) {
      if (nact1 <= 0) continue;
      pd.ord = pl.ord2.as<int>() + (size_t)(l1 - 1) * n;
      pd.ord2l1 = nullptr;
      pd.lseg = l1;
      pd.l1 = l1;
      pd.n_act = nact1;
      GPM_TRY(lv_launch_pass<A>(pd, s, launches));
    } else {
      for (int l2 = 1; l2 <= l1; ++l2) {
        const int64_t c_last = (n - 1) >> l2;
        const int64_t mid2 = (c_last << l2) + (int64_t(1) << (l2 - 1));
        int64_t nact = nact1;
        if (mid2 >= n) nact = std::min(nact, c_last << l2);
        if (nact <= 0) continue;
        pd.ord = pl.ord3.as<int>() + ((size_t)(l1 - 1) * l1 / 2 + (l2 - 1)) * n;
        pd.ord2l1 = pl.ord2.as<int>() + (size_t)(l1 - 1) * n;
        pd.lseg = l2;
        pd.l1 = l1;
        pd.n_act = nact;
        GPM_TRY(lv_launch_pass<A>(pd, s, launches));
      }
    }
  }
  return GP_OK;
}

gp_status level_passes(Plan& pl, const double* u_rank, cudaStream_t s, int* launches) {
  const bool prod = pl.form == GP_FORM_PRODUCT;
  if (pl.d == 2) {
    if (!prod) {
      if (pl.P == 0) return lv_all_passes<Alg<0, 2, false>>(pl, u_rank, s, launches);
      if (pl.P == 1) return lv_all_passes<Alg<1, 2, false>>(pl, u_rank, s, launches);
      return lv_all_passes<Alg<2, 2, false>>(pl, u_rank, s, launches);
    }
    if (pl.P == 0) return lv_all_passes<Alg<0, 2, true>>(pl, u_rank, s, launches);
    if (pl.P == 1) return lv_all_passes<Alg<1, 2, true>>(pl, u_rank, s, launches);
    return lv_all_passes<Alg<2, 2, true>>(pl, u_rank, s, launches);
  }
  if (pl.P == 0) return lv_all_passes<Alg<0, 4, false>>(pl, u_rank, s, launches);
  if (pl.P == 1) return lv_all_passes<Alg<1, 4, false>>(pl, u_rank, s, launches);
  return lv_all_passes<Alg<2, 4, false>>(pl, u_rank, s, launches);
}

int64_t level_tiles(int64_t n) { return (n + LV_TILE - 1) / LV_TILE; }

}  // namespace gpm
