// apply_d1_big.cu -- the d = 1 path above the single-chunk capacity of apply_d1.cu
// (N > #SMs x BLOCK x ITEMS of k_d1_lpc): a reduce-then-scan in three plain launches,
// same method and algebra (P:314-340 [eq fast_exact_decomposition_1d, §2.1]).
#include <algorithm>
#include <climits>
#include <cstdlib>

#include <algorithm>

#include "algebra.cuh"
#include "fexp.cuh"
#include "internal.h"
#include "tma.cuh"


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
      uu[k] = pi < a.n_src ? __ldcg(a.v + pi) : 0.0;   // no reuse: L2 only
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


}  // namespace gpm
