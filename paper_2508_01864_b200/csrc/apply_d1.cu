// apply_d1.cu -- the d = 1 hot path: K.v over the stored sort in
// ONE cooperative launch when the sorted points fit one shared-memory chunk per CTA
// (N <= #SMs x BLOCK x ITEMS; every BASELINE.json d = 1 config).  Method: the weighted
// ECDF / survival-function decomposition of P:314-325 [eq fast_exact_decomposition_1d]
// evaluated by "fast sum updating" over the presorted data (P:326-340 [§2.1]) in the
// overflow-free moment basis of algebra.cuh (reading R5).
//
// B200 structure (k_d1_lpc, "local pass + correction"):
//   0. the chunk's sorted t (+ perm, user order) arrive by 1-D bulk copies issued before
//      griddepcontrol.wait (plan data); the gaps and e^{-gap} are computed into registers
//      while v is still in flight;
//   1. rank order: v by bulk copies; user order: the gathers v[perm] (after a 1/G-slice L2
//      prefetch of v per CTA);
//   2. LOCAL pass: each thread runs the forward and backward recurrences over its ITEMS
//      consecutive points starting from zero state (two independent chains), keeping
//      loc_j = self u_j + read_F + read_B in registers; the final states are the thread's
//      aggregates;
//   3. chunk aggregate = fixed-order plain sum of the thread aggregates shifted to the
//      chunk's reference points (all shifts forward: e^{-x}, x >= 0), published as a
//      self-validating record (every 8-byte word = 32 data bits + a 32-bit column tag,
//      "LL" words: no fence, no flag, no barrier);
//   4. while the other chunks publish: the block scan of the thread aggregates (warp
//      shuffles) -> each thread's exclusive prefix / suffix inside the chunk;
//   5. each thread folds the records it needs (one record per thread, poll until every
//      word carries this column's tag; plain sums of forward shifts, fixed order);
//   6. CORRECTION pass: the carry entering a thread adds e^{-D} sum_r beta_r D^r at a
//      point D past the thread's reference (P + 3 FLOPs per point and direction);
//      out = os2 (loc + both corrections), written back coalesced (rank order) or
//      scattered to out[perm] (user order).
// Determinism: every sum has a fixed order (no atomics on data), so repeated applies are
// bitwise identical.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "algebra.cuh"
#include "fexp.cuh"
#include "internal.h"
#include "tma.cuh"

namespace gpm {

namespace lpc {

constexpr int NPART = 4;    // bulk-copy pipeline depth (parts of the chunk)
constexpr int LL_W = 32;    // 8-byte words per record slot (<= 2 x 2 x 6 moments x 2 halves)

struct Args {
  const double* ts;    // sorted scaled coordinates (plan)
  const double* ends;  // chunk ends: t_0, t[min(b chunk, n) - 1] for b = 1..G (plan, padded)
  const double* e1;    // e^{-gap} per rank (plan, padded with 1)
  const int* perm;     // rank -> user index (plan, padded)
  const double* v;     // input columns: user order or rank order
  double* out;         // output columns: user order (targets only) or rank order
  int64_t n, n_src, tgt_off, chunk;
  int nrhs;
  int prefetch;        // user order: L2 prefetch of a 1/G slice of v per CTA
  int cap;             // user order: shared-memory array capacity (multiple of 4, >= chunk + items)
  int64_t vstride, ostride;
  double os2;
  unsigned long long* rec;   // [2 parities][G][LL_W] LL words
  unsigned* ep;              // [G]: columns published by CTA b over the plan's life
  unsigned long long* dbg;   // optional phase timestamps [G][16] (GPM_D1_TIMING)
  int knob;                  // debug: skip phases (GPM_D1_KNOB; timing experiments only)
  double cg_s2;              // CG epilogue (rank order): out = K u + cg_s2 u ...
  double* cg_part;           // ... and the CTA's partial u . out -> cg_part[col * G + cta]
};

// SM cycle counter (per SM; phase stamps are compared within a warp)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %clock64;" : "=l"(t));
  return t;
}
// per-warp phase timestamps (lane 0 of every warp): dbg[(cta * 32 + warp) * 16 + slot]
#define LPC_STAMP(k)                                                                      \
  do {                                                                                    \
    if (a.dbg && (threadIdx.x & 31) == 0)                                                 \
      a.dbg[(blockIdx.x * 32 + (threadIdx.x >> 5)) * 16 + (k)] = gtimer();                \
  } while (0)

// LL words: 32 data bits in the low half, the column tag in the high half; each 8-byte
// access is single-copy atomic, so a word with the expected tag carries valid data.
__device__ __forceinline__ void st_ll2(unsigned long long* p, unsigned long long a,
                                       unsigned long long b) {
  asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b)
               : "memory");
}
__device__ __forceinline__ void ld_ll2(const unsigned long long* p, unsigned long long& a,
                                       unsigned long long& b) {
  asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p)
               : "memory");
}
__device__ __forceinline__ unsigned long long ll_word(unsigned tag, unsigned data) {
  return ((unsigned long long)tag << 32) | data;
}

// scan element: span D, E = e^{-D}, NQ moments
template <int NQ>
struct Mon {
  double D, E, M[NQ];
};
template <int NQ>
__device__ __forceinline__ Mon<NQ> mon_id() {
  Mon<NQ> r;
  r.D = 0.0;
  r.E = 1.0;
#pragma unroll
  for (int q = 0; q < NQ; ++q) r.M[q] = 0.0;
  return r;
}
// forward (A left of B): S(B.D) A + B
template <int NQ>
__device__ __forceinline__ Mon<NQ> mon_f(const Mon<NQ>& A, const Mon<NQ>& B) {
  Mon<NQ> r;
#pragma unroll
  for (int q = 0; q < NQ; ++q) r.M[q] = A.M[q];
  advance<NQ - 1>(r.M, B.D, B.E);
#pragma unroll
  for (int q = 0; q < NQ; ++q) r.M[q] += B.M[q];
  r.D = A.D + B.D;
  r.E = A.E * B.E;
  return r;
}
// backward (A left of B): A + S(A.D) B
template <int NQ>
__device__ __forceinline__ Mon<NQ> mon_b(const Mon<NQ>& A, const Mon<NQ>& B) {
  Mon<NQ> r;
#pragma unroll
  for (int q = 0; q < NQ; ++q) r.M[q] = B.M[q];
  advance<NQ - 1>(r.M, A.D, A.E);
#pragma unroll
  for (int q = 0; q < NQ; ++q) r.M[q] += A.M[q];
  r.D = A.D + B.D;
  r.E = A.E * B.E;
  return r;
}
template <int NQ>
__device__ __forceinline__ Mon<NQ> mon_shfl(const Mon<NQ>& s, int off, bool up) {
  Mon<NQ> r;
  if (up) {
    r.D = __shfl_up_sync(0xffffffffu, s.D, off);
    r.E = __shfl_up_sync(0xffffffffu, s.E, off);
#pragma unroll
    for (int q = 0; q < NQ; ++q) r.M[q] = __shfl_up_sync(0xffffffffu, s.M[q], off);
  } else {
    r.D = __shfl_down_sync(0xffffffffu, s.D, off);
    r.E = __shfl_down_sync(0xffffffffu, s.E, off);
#pragma unroll
    for (int q = 0; q < NQ; ++q) r.M[q] = __shfl_down_sync(0xffffffffu, s.M[q], off);
  }
  return r;
}
template <int NQ>
__device__ __forceinline__ void mon_st(double* p, const Mon<NQ>& s) {
  p[0] = s.D;
  p[1] = s.E;
#pragma unroll
  for (int q = 0; q < NQ; ++q) p[2 + q] = s.M[q];
}
template <int NQ>
__device__ __forceinline__ Mon<NQ> mon_ld(const double* p) {
  Mon<NQ> s;
  s.D = p[0];
  s.E = p[1];
#pragma unroll
  for (int q = 0; q < NQ; ++q) s.M[q] = p[2 + q];
  return s;
}

// read(S(D) C) = e^{-D} sum_r beta_r D^r with beta_r = sum_{q >= r} c_q C(q, q - r) C_{q-r}
template <int P, int KIND>
__device__ __forceinline__ void carry_beta(const double* C, double* beta) {
#pragma unroll
  for (int r = 0; r <= P; ++r) {
    double br = 0.0;
#pragma unroll
    for (int q = r; q <= P; ++q)
      if (rcoef(P, KIND, q) != 0.0) br = fma(rcoef(P, KIND, q) * binom(q, q - r), C[q - r], br);
    beta[r] = br;
  }
}

constexpr int pow2_at_least(int x) { return x <= 1 ? 1 : 2 * pow2_at_least((x + 1) / 2); }

// Warp sum of NV values by a reduce-scatter butterfly (NP = NV rounded up to a power of
// two): each round halves the values a lane keeps, so a warp moves NP - 1 + log2(32/NP)
// doubles per lane instead of 5 NV.  Returns the warp total of value *idx (same on every
// lane of a group of 32/NP lanes); fixed order, hence deterministic.
template <int NV>
__device__ __forceinline__ double warp_sum_scatter(const double* in, int lane, int* idx) {
  constexpr int NP = pow2_at_least(NV);
  static_assert(NP <= 32, "at most 32 values");
  double v[NP];
#pragma unroll
  for (int i = 0; i < NP; ++i) v[i] = i < NV ? in[i] : 0.0;
  int id = 0;
#pragma unroll
  for (int r = 0, cur = NP; r < 5; ++r) {
    const int o = 16 >> r;
    if (cur > 1) {
      const int half = cur / 2;
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < half; ++i) {
        const double keep = up ? v[i + half] : v[i];
        const double send = up ? v[i] : v[i + half];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
      if (up) id += half;
      cur = half;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    }
  }
  *idx = id;
  return v[0];
}

// One scan element of a run of points (forward moments MF referenced at the run's last
// point, backward moments MB referenced at the point before its first point, span D from
// that point to the last point, E = e^{-D}).
template <int NQ>
struct Run {
  double D, E, MF[NQ], MB[NQ];
};

// u buffers: two in rank order (the next column's v lands while this one computes) when
// t, e^{-gap} and 2 u fit the 227 KB carve-out, else one
constexpr int lpc_nub(bool user, int sub) { return (!user && (4 * sub + 18) * 8 <= 221 * 1024) ? 2 : 1; }

// P: moment order (KIND 0: nu = P + 1/2; KIND 1: the lengthscale gradient of nu = P - 1/2)
template <int P, int KIND, int BLOCK, int SEGS, int SL, bool USER>
__global__ void __launch_bounds__(BLOCK, 1) k_d1_lpc(Args a) {
  constexpr int ITEMS = SEGS * SL;    // my points: SEGS segments of SL consecutive points
  constexpr int NQ = P + 1;
  constexpr int SUB = BLOCK * ITEMS;
  constexpr int NW = BLOCK / 32;
  constexpr int PT = BLOCK / NPART;   // threads per load part
  constexpr int PSZ = PT * ITEMS;     // points per load part
  constexpr int NV = 2 * NQ;          // record values: forward + backward moments
  constexpr int NUB = lpc_nub(USER, SUB);   // rank order: u double-buffered across columns
  static_assert(PSZ % 4 == 0, "load parts must stay 16-byte aligned");
  static_assert(2 * NV <= LL_W, "record slot too small");
  static_assert(NW <= 32 && BLOCK >= 64 + 160, "warp roles: 2 totals warps, fold threads for G <= 160");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* s_t = reinterpret_cast<double*>(smem_raw) + 2;   // [-2, SUB + 8): t (clamped past
                                                           // the end; s_t[-1] = t[c0 - 1])
  // Array capacity: SUB, or (user order, default shape) a.cap = the chunk's points + one
  // thread's items, so that a 10^6-point plan stays in the 164 KB shared-memory class (more
  // L1 for the random gathers).  Threads wholly past the chunk all use the last ITEMS slots
  // (window base jb), which hold the neutral tail values.
  constexpr bool RTCAP = USER && ITEMS == 27;   // the default shape only: the larger shapes sit
                                                // at the register cap and lose more to the
                                                // run-time strides than the L1 gives them
  const int CAP = RTCAP ? a.cap : SUB;
  double* s_e = s_t + CAP + 8;                         // CAP + 8: e^{-gap} (1 past the end)
  double* s_ub = s_e + CAP + 8;                        // NUB x CAP: u, then out (rank order)
  // user order: the chunk's perm (SUB + 8 ints) lives in the upper half of the one u buffer
  // (28 KB less shared memory: the 3x10 shape stays below the largest carve-out, whose small L1
  // halves the gather rate -- profiles/r02_notes.md).  It is read before u is written (one block barrier) and
  // bulk-copied again after the local pass, for the scatter.
  int* s_pi = reinterpret_cast<int*>(s_ub + CAP / 2);
  __shared__ uint64_t mbar[NPART], mbar_v[NUB][NPART], mbar_tab, mbar_pi;
  __shared__ __align__(16) double s_tab[64];
  __shared__ double s_wf[NW][NQ + 2], s_wb[NW][NQ + 2];   // warp totals of the block scan
  __shared__ double s_red[NW][NV];                        // warp partials of the chunk sum
  __shared__ double s_pq[NW];                             // CG epilogue: warp partials of p . q
  __shared__ __align__(16) double s_tl[160 + 2];         // chunk-end t: s_tl[b + 1], s_tl[0] = t_0

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, c = blockIdx.x;
  const int64_t c0 = (int64_t)c * a.chunk;
  const int cnt = (int)min(a.chunk, a.n - c0);   // >= 1 (host: every CTA owns points)
  const int j0 = tid * ITEMS;
  const int jb = (RTCAP && j0 >= cnt) ? a.cap - ITEMS : j0;   // shared-memory window of my items
  const int mypart = tid / PT;
  const bool part_live = mypart * PSZ < cnt;
  const bool v_bulk = !USER && ((reinterpret_cast<uintptr_t>(a.v + c0) & 15) == 0) &&
                      (a.vstride % 2 == 0 || a.nrhs == 1);
  const bool o_bulk = !USER && ((reinterpret_cast<uintptr_t>(a.out + c0) & 15) == 0) &&
                      (a.ostride % 2 == 0 || a.nrhs == 1);
  // rank order: a column of v by bulk copies into u buffer col % NUB (thread 0 owns the
  // barriers)
  auto issue_v = [&](int col) {
    double* dst = s_ub + (col % NUB) * CAP;
#pragma unroll 1
    for (int p = 0; p < NPART; ++p) {
      const int lo = p * PSZ, hi = min(cnt, lo + PSZ);
      if (lo < hi) {
        const unsigned nu = (unsigned)((hi - lo) & ~1);   // never over-read v
        mbar_expect_tx(&mbar_v[col % NUB][p], nu * 8);
        if (nu) tma_load_1d(dst + lo, a.v + col * a.vstride + c0 + lo, nu * 8, &mbar_v[col % NUB][p]);
      }
    }
  };
  auto prefetch_v = [&](int col) {   // user order: this CTA's 1/G slice of v into L2
    const int64_t per = (a.n_src + G - 1) / G;
    const int64_t lo = min((int64_t)c * per, a.n_src);
    const int64_t hi = min(lo + per, a.n_src);
    if (hi > lo) prefetch_l2_range(a.v + col * a.vstride + lo, (size_t)(hi - lo) * 8);
  };

  LPC_STAMP(0);
  // ---- prologue.  Thread 0 initialises the barriers; after one __syncthreads it issues
  // the plan-data bulk copies while the others go on.  Boundary coordinates come from the
  // copied t (scalar global loads would queue behind the bulk traffic at the L2).
  if (tid == 0) {
    for (int p = 0; p < NPART; ++p) {
      mbar_init(&mbar[p], 1);
      for (int ub = 0; ub < NUB; ++ub) mbar_init(&mbar_v[ub][p], 1);
    }
    mbar_init(&mbar_tab, 1);
    mbar_init(&mbar_pi, 1);
    mbar_fence_init();
  }
  __syncthreads();   // barrier initialisation visible
  if (tid == 0) {   // plan data: before griddepcontrol.wait
    const unsigned nend = (unsigned)((G + 2) & ~1);   // chunk ends (padded plan array)
    mbar_expect_tx(&mbar_tab, 64 * 8 + nend * 8);
    tma_load_1d(s_tab, g_fexp_tab, 64 * 8, &mbar_tab);
    tma_load_1d(s_tl, a.ends, nend * 8, &mbar_tab);
#pragma unroll 1
    for (int p = 0; p < NPART; ++p) {
      const int lo = p * PSZ, hi = min(cnt, lo + PSZ);
      if (lo < hi) {
        // part 0 of chunks c > 0 starts two points early (16-byte aligned): s_t[-1] is
        // the chunk's reference point
        const int lo2 = (p == 0 && c > 0) ? lo - 2 : lo;
        const unsigned nt = (unsigned)(((hi - lo2) + 1) & ~1);   // padded plan arrays
        const unsigned np = (unsigned)(((hi - lo) + 3) & ~3);
        const unsigned ne = (unsigned)(((hi - lo) + 1) & ~1);
        mbar_expect_tx(&mbar[p], nt * 8 + ne * 8 + (USER ? np * 4 : 0));
        tma_load_1d(s_t + lo2, a.ts + c0 + lo2, nt * 8, &mbar[p]);
        tma_load_1d(s_e + lo, a.e1 + c0 + lo, ne * 8, &mbar[p]);
        if (USER) tma_load_1d(s_pi + lo, a.perm + c0 + lo, np * 4, &mbar[p]);
      }
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");   // v, records and ep of earlier launches
  asm volatile("griddepcontrol.launch_dependents;");
  LPC_STAMP(8);
  if (tid == 0 && v_bulk) {
    issue_v(0);
    if (NUB > 1 && a.nrhs > 1) issue_v(1);
  }
  if (USER && a.prefetch && tid == 32) prefetch_v(0);
  const unsigned base = __ldcg(a.ep + c);   // columns published so far (L2: the previous grid)
  mbar_wait(&mbar_tab, 0);
  LPC_STAMP(7);
#pragma unroll 1
  for (int p = 0; p < NPART; ++p)   // every live part: boundary points may lie in any
    if (p * PSZ < cnt) mbar_wait(&mbar[p], 0);
  LPC_STAMP(9);
  // boundary coordinates (clamped to the chunk): the chunk's reference point (the point
  // before its first point; t_0 for chunk 0: its first gap is 0), the point before my
  // first point, the last points of my segments, the chunk's last point
  const double tref0 = c > 0 ? s_t[-1] : s_t[0];
  const double tlast = s_t[cnt - 1];
  // (true index: the first thread past the chunk, j0 == cnt, still reads the chunk's last point)
  const double tprev = j0 == 0 ? tref0 : (j0 - 1 < cnt ? s_t[j0 - 1] : tlast);
  double tseg[SEGS];   // the last point of each of my segments
#pragma unroll
  for (int sg = 0; sg < SEGS; ++sg) tseg[sg] = s_t[min(j0 + (sg + 1) * SL, cnt) - 1];
  if (j0 >= cnt) {
#pragma unroll
    for (int sg = 0; sg < SEGS; ++sg) tseg[sg] = tlast;
  }
  const double tmye = tseg[SEGS - 1];
  __syncthreads();   // every thread's boundary reads before the tails are clamped
  // ---- neutral tails (once per launch): t clamped to the last point (gap 0), weight 1,
  // u = 0 (rank order: the bulk copies stop at cnt), no source index (user order)
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const int j = j0 + k, js = jb + k;
    if (j >= cnt) {
      s_t[js] = tlast;
      s_e[js] = 1.0;
      if (!USER) {   // user order: every thread writes all its u slots per column
#pragma unroll
        for (int ub = 0; ub < NUB; ++ub) s_ub[ub * CAP + js] = 0.0;
      }
    }
    if (USER && j >= ((cnt + 3) & ~3)) s_pi[js] = INT_MAX;
  }
  // v-independent shifts, once per launch: my element's span, the chunk-sum shifts (my
  // last point -> chunk last point, chunk reference -> my t_prev)
  const double Dme = tmye - tprev, Eme = fexp_neg(Dme, s_tab);
  const double dF = tlast - tmye, eF = fexp_neg(dF, s_tab);
  const double dB = tprev - tref0, eB = fexp_neg(dB, s_tab);
  LPC_STAMP(1);

#pragma unroll 1
  for (int col = 0; col < a.nrhs; ++col) {
    const double* vcol = a.v + col * a.vstride;
    double* ocol = a.out + col * a.ostride;
    double* s_u = s_ub + (col % NUB) * CAP;
    const unsigned tag = base + (unsigned)col + 1u;
    unsigned long long* recp = a.rec + (size_t)(col & 1) * G * LL_W;
    // ---- u of my points into s_u (own items only: no block barrier needed)
    if (USER) {
      double uu[ITEMS];
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        const int pi = s_pi[jb + k];
        uu[k] = (j0 + k < cnt && pi < a.n_src) ? __ldcg(vcol + pi) : 0.0;   // no reuse: L2 only (gs_variants.cu)
      }
      if (a.prefetch && tid == 32 && col + 1 < a.nrhs) prefetch_v(col + 1);
      __syncthreads();   // perm shares the u buffer: every thread's perm reads precede the u writes
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) s_u[jb + k] = uu[k];
    } else if (v_bulk) {
      if (part_live) mbar_wait(&mbar_v[col % NUB][mypart], (unsigned)((col / NUB) & 1));
      const int lo = mypart * PSZ, hi = min(cnt, lo + PSZ);
      if (lo < hi && ((hi - lo) & 1) && tid == (hi - 1) / ITEMS)   // odd tail element
        s_u[hi - 1] = __ldg(vcol + c0 + hi - 1);
    } else {
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) s_u[jb + k] = j0 + k < cnt ? __ldg(vcol + c0 + j0 + k) : 0.0;
    }
    LPC_STAMP(2);
    // ---- local pass from zero state: the forward recurrence over all my points and the
    // backward one, interleaved (two chains), continuous across my segments; a phase
    // stages the forward chain's segment and the backward chain's segment (t, e^{-gap},
    // u, once each from shared memory); loc_j = u_j (self term) + read_F + read_B, all
    // scaled by os2 through the injected weights (u' = os2 u)
    double loc[ITEMS];
    double F[NQ], B[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) F[q] = B[q] = 0.0;
#pragma unroll
    for (int ph = 0; ph < SEGS; ++ph) {
      const int sf = ph, sb = SEGS - 1 - ph;       // forward / backward segment
      const int f0 = sf * SL, b0 = sb * SL;
      double tf[SL + 1], ef[SL], uf[SL], tb[SL + 1], eb[SL + 1], ub[SL];
      tf[0] = sf ? s_t[jb + f0 - 1] : tprev;
#pragma unroll
      for (int k = 0; k < SL; ++k) {
        tf[k + 1] = s_t[jb + f0 + k];
        ef[k] = s_e[jb + f0 + k];
        uf[k] = a.os2 * s_u[jb + f0 + k];
      }
#pragma unroll
      for (int k = 0; k < SL; ++k) {   // the backward segment's t, e^{-gap} of the next point
        tb[k] = sf == sb ? tf[k + 1] : s_t[jb + b0 + k];
        ub[k] = sf == sb ? uf[k] : a.os2 * s_u[jb + b0 + k];
        eb[k] = k == 0 ? 0.0 : (sf == sb ? ef[k] : s_e[jb + b0 + k]);
      }
      tb[SL] = sb + 1 < SEGS ? s_t[jb + b0 + SL] : 0.0;
      eb[SL] = sb + 1 < SEGS ? s_e[jb + b0 + SL] : 1.0;
#pragma unroll
      for (int k = 0; k < SL; ++k) {
        const int i = f0 + k;              // forward point
        if (i > 0) advance<P>(F, tf[k + 1] - tf[k], ef[k]);
        const double rf = KIND == 0 ? (i > 0 ? uf[k] + readc0<P, KIND>(F) : uf[k])
                                    : (i > 0 ? readc0<P, KIND>(F) : 0.0);
        F[0] += uf[k];
        const int kb = SL - 1 - k, ib = b0 + kb;   // backward point
        if (ib < ITEMS - 1) advance<P>(B, tb[kb + 1] - tb[kb], eb[kb + 1]);
        const double rb = ib < ITEMS - 1 ? readc0<P, KIND>(B) : 0.0;
        B[0] += ub[kb];
        // first touch assigns: point i meets the forward chain at step i and the backward
        // chain at step ITEMS-1-i (the middle point: both in one step, forward first)
        if (i <= ITEMS - 1 - i) loc[i] = rf; else loc[i] += rf;
        if (ITEMS - 1 - ib < ib) loc[ib] = rb; else loc[ib] += rb;
      }
    }
    {   // backward aggregate -> my t_prev
      const double t0 = s_t[jb];
      advance<P>(B, t0 - tprev, s_e[jb]);
    }
    Run<NQ> me;   // my scan element: span t_prev -> my last point
    me.D = Dme;
    me.E = Eme;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      me.MF[q] = F[q];
      me.MB[q] = B[q];
    }
    LPC_STAMP(3);
    // ---- chunk aggregate = fixed-order sum of the shifted thread aggregates -> record
    {
      double m[NV];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        m[q] = me.MF[q];
        m[NQ + q] = me.MB[q];
      }
      advance<P>(m, dF, eF);
      advance<P>(m + NQ, dB, eB);
      int id;
      const double sw = warp_sum_scatter<NV>(m, lane, &id);
      if ((lane & (32 / pow2_at_least(NV) - 1)) == 0 && id < NV) s_red[warp][id] = sw;
    }
    __syncthreads();   // #1: chunk-sum partials
    if (USER && tid == 0) {   // u is consumed: perm back into its upper half for the scatter
      fence_proxy_async_smem();
      const unsigned np = (unsigned)((cnt + 3) & ~3);
      mbar_expect_tx(&mbar_pi, np * 4);
      tma_load_1d(s_pi, a.perm + c0, np * 4, &mbar_pi);
    }
    if (tid < NV) {    // one value per thread, warps summed in order, published as 2 words
      double s = 0.0;
#pragma unroll 1
      for (int w = 0; w < NW; ++w) s += s_red[w][tid];
      st_ll2(recp + (size_t)c * LL_W + 2 * tid, ll_word(tag, (unsigned)__double2loint(s)),
             ll_word(tag, (unsigned)__double2hiint(s)));
    }
    LPC_STAMP(4);
    // ---- block scan of the thread elements (overlaps the other chunks' publication):
    // forward inclusive prefix / backward inclusive suffix per warp -> the warp totals
    Mon<NQ> fe, be;
    {
      Mon<NQ> fi, bi;
      fi.D = bi.D = me.D;
      fi.E = bi.E = me.E;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        fi.M[q] = me.MF[q];
        bi.M[q] = me.MB[q];
      }
#pragma unroll 1
      for (int off = 1; off < 32; off <<= 1) {
        const Mon<NQ> l = mon_shfl<NQ>(fi, off, true);
        const Mon<NQ> r = mon_shfl<NQ>(bi, off, false);
        if (lane >= off) fi = mon_f<NQ>(l, fi);
        if (lane + off < 32) bi = mon_b<NQ>(bi, r);
      }
      if (lane == 31) mon_st<NQ>(s_wf[warp], fi);
      if (lane == 0) mon_st<NQ>(s_wb[warp], bi);
      fe = mon_shfl<NQ>(fi, 1, true);    // exclusive within the warp
      be = mon_shfl<NQ>(bi, 1, false);
      if (lane == 0) fe = mon_id<NQ>();
      if (lane == 31) be = mon_id<NQ>();
    }
    LPC_STAMP(10);
    __syncthreads();   // #2: warp totals
    LPC_STAMP(5);
    if (warp < 2) {    // warp 0: exclusive forward prefix of the warp totals; warp 1: suffix
      const bool fw = warp == 0;
      Mon<NQ> xw = lane < NW ? mon_ld<NQ>(fw ? s_wf[lane] : s_wb[lane]) : mon_id<NQ>();
#pragma unroll 1
      for (int off = 1; off < NW; off <<= 1) {
        const Mon<NQ> y = mon_shfl<NQ>(xw, off, fw);
        if (fw && lane >= off) xw = mon_f<NQ>(y, xw);
        if (!fw && lane + off < 32) xw = mon_b<NQ>(xw, y);
      }
      Mon<NQ> xe = mon_shfl<NQ>(xw, 1, fw);
      if ((fw && lane == 0) || (!fw && lane >= NW - 1)) xe = mon_id<NQ>();
      __syncwarp();
      if (lane < NW) mon_st<NQ>(fw ? s_wf[lane] : s_wb[lane], xe);
    } else if (tid >= 64 && tid < 64 + 32 * ((G + 31) / 32)) {
      // ---- fold the other chunks' records, one per thread (threads 64 .. 64 + G - 1): poll
      // until every word carries this column's tag; forward moments of earlier chunks
      // shifted from their last point to my chunk's reference, backward moments of later
      // chunks from their reference to my chunk's last point; warp sums in fixed order
      double fm[NV];
#pragma unroll
      for (int q = 0; q < NV; ++q) fm[q] = 0.0;
      const int b = tid - 64;
      if (b < G && b != c) {
        const int o = b < c ? 0 : NQ;
        const unsigned long long* w = recp + (size_t)b * LL_W + 2 * o;
        unsigned long long x[2 * NQ];
        bool ok;
        do {
          ok = true;
#pragma unroll
          for (int i = 0; i < NQ; ++i) {
            ld_ll2(w + 2 * i, x[2 * i], x[2 * i + 1]);
            ok &= (unsigned)(x[2 * i] >> 32) == tag && (unsigned)(x[2 * i + 1] >> 32) == tag;
          }
        } while (!ok);
        double mv[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q)
          mv[q] = __hiloint2double((int)(unsigned)x[2 * q + 1], (int)(unsigned)x[2 * q]);
        const double D = b < c ? s_tl[c] - s_tl[b + 1] : s_tl[b] - s_tl[c + 1];
        advance<P>(mv, D, fexp_neg(D, s_tab));
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          fm[q] = b < c ? mv[q] : 0.0;
          fm[NQ + q] = b < c ? 0.0 : mv[q];
        }
      }
      LPC_STAMP(11);
      int id;
      const double sw = warp_sum_scatter<NV>(fm, lane, &id);
      if ((lane & (32 / pow2_at_least(NV) - 1)) == 0 && id < NV) s_red[warp - 2][id] = sw;
    }
    __syncthreads();   // #3: exclusive warp totals, fold partials
    LPC_STAMP(13);
    // ---- my carries: X = forward state entering my first point (earlier threads and
    // chunks), Y = backward state entering my last point; a carry C seen from a point D
    // further on reads e^{-D} sum_r beta_r D^r (carry_beta)
    double bX[NQ], bY[NQ];
    {
      const Mon<NQ> wf = mon_ld<NQ>(s_wf[warp]), wb = mon_ld<NQ>(s_wb[warp]);
      const Mon<NQ> Fx = mon_f<NQ>(wf, fe);   // threads before me, referenced at my t_prev
      const Mon<NQ> Bx = mon_b<NQ>(be, wb);   // threads after me, referenced at my last point
      double g[NQ], y[NQ];   // the chunk carries: fold partials summed in order
#pragma unroll
      for (int q = 0; q < NQ; ++q) g[q] = y[q] = 0.0;
#pragma unroll 1
      for (int w = 0; w < (G + 31) / 32; ++w) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          g[q] += s_red[w][q];
          y[q] += s_red[w][NQ + q];
        }
      }
      advance<P>(g, Fx.D, Fx.E);   // chunk reference -> my t_prev
      advance<P>(y, Bx.D, Bx.E);   // chunk last point -> my last point
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        g[q] += Fx.M[q];
        y[q] += Bx.M[q];
      }
      advance<P>(g, s_t[jb] - tprev, s_e[jb]);   // -> my first point
      carry_beta<P, KIND>(g, bX);
      carry_beta<P, KIND>(y, bY);
    }
    LPC_STAMP(14);
    // ---- correction pass (forward and backward chains interleaved, staged per phase as
    // the local pass), then the output
    {
      double Ef = 1.0, Eb = 1.0;
      const double tfirst = s_t[jb], tmyl = s_t[jb + ITEMS - 1];
#pragma unroll
      for (int ph = 0; ph < SEGS; ++ph) {
        const int f0 = ph * SL, b0 = (SEGS - 1 - ph) * SL;
        double tf[SL], ef[SL], tb[SL], eb[SL + 1];
#pragma unroll
        for (int k = 0; k < SL; ++k) {
          tf[k] = s_t[jb + f0 + k];
          ef[k] = s_e[jb + f0 + k];
          tb[k] = f0 == b0 ? tf[k] : s_t[jb + b0 + k];
          eb[k] = k == 0 ? 0.0 : (f0 == b0 ? ef[k] : s_e[jb + b0 + k]);
        }
        eb[SL] = b0 + SL < ITEMS ? s_e[jb + b0 + SL] : 1.0;
#pragma unroll
        for (int k = 0; k < SL; ++k) {
          const int i = f0 + k, kb = SL - 1 - k, ib = b0 + kb;
          if (i > 0) Ef *= ef[k];
          if (ib < ITEMS - 1) Eb *= eb[kb + 1];
          const double Df = tf[k] - tfirst, Db = tmyl - tb[kb];
          double hf = bX[P], hb = bY[P];
#pragma unroll
          for (int r = P - 1; r >= 0; --r) {
            hf = fma(hf, Df, bX[r]);
            hb = fma(hb, Db, bY[r]);
          }
          loc[i] = fma(Ef, hf, loc[i]);
          loc[ib] = fma(Eb, hb, loc[ib]);
        }
      }
    }
    if (USER) {
      mbar_wait(&mbar_pi, (unsigned)(col & 1));
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        const int j = j0 + k;
        const int pi = s_pi[jb + k];
        if (j < cnt && pi >= a.tgt_off) ocol[pi - a.tgt_off] = loc[k];
      }
    } else if (!a.cg_part) {
#pragma unroll
      for (int k = 0; k < ITEMS; ++k)
        if (j0 + k < cnt) s_u[jb + k] = loc[k];   // the tail stays 0 for a later column
    } else {   // CG epilogue: q = K p + s2 p, partial p . q (the tail has p = 0)
      double pq = 0.0;
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        const double pk = s_u[jb + k];
        const double qk = fma(a.cg_s2, pk, loc[k]);
        pq = fma(pk, qk, pq);
        if (j0 + k < cnt) s_u[jb + k] = qk;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) pq += __shfl_xor_sync(0xffffffffu, pq, off);
      if (lane == 0) s_pq[warp] = pq;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
#pragma unroll 1
        for (int w = 0; w < NW; ++w) t += s_pq[w];
        a.cg_part[(size_t)col * G + c] = t;
      }
    }
    LPC_STAMP(12);
    if (!USER) {   // this warp's contiguous outputs, coalesced 16-byte stores (+ an odd tail)
      __syncwarp();
      const int wb = warp * 32 * ITEMS;
      const int we = min(cnt, wb + 32 * ITEMS);
      if (o_bulk) {
        const int np2 = (we - wb) >> 1;
        const double2* src = reinterpret_cast<const double2*>(s_u + wb);
        double2* dst = reinterpret_cast<double2*>(ocol + c0 + wb);
#pragma unroll 4
        for (int k = lane; k < np2; k += 32) dst[k] = src[k];
        if (((we - wb) & 1) && lane == 0) ocol[c0 + we - 1] = s_u[we - 1];
      } else {
#pragma unroll 4
        for (int j = wb + lane; j < we; j += 32) ocol[c0 + j] = s_u[j];
      }
    }
    LPC_STAMP(6);
    if (col + 1 < a.nrhs) {
      // the u buffer of this column is the v destination of column col + NUB: every
      // thread's generic accesses precede the copy
      fence_proxy_async_smem();
      __syncthreads();   // s_u, s_red, s_C, s_wf / s_wb of this column consumed
      if (!USER && v_bulk && tid == 0 && col + NUB < a.nrhs) issue_v(col + NUB);
    }
  }   // column loop
  if (tid == 0) a.ep[c] = base + (unsigned)a.nrhs;
}

// e1[r] = e^{-(t_r - t_{r-1})} (e1[0] = 1; padding 1): the v-independent exponentials of
// the scan, precomputed once per plan (plan data, read by bulk copies beside t: one
// e^{-x} per point per apply saved for 8 bytes per point of L2-resident plan traffic)
__global__ void k_d1_e_build(const double* __restrict__ t, int64_t n, double* __restrict__ e1) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n + 16;
       r += (int64_t)gridDim.x * blockDim.x)
    e1[r] = (r > 0 && r < n) ? exp(-(t[r] - t[r - 1])) : 1.0;
}

// chunk ends of a chunking (plan data for the fold's shift distances): ends[0] = t_0,
// ends[b] = t[min(b chunk, n) - 1] for b = 1..G (ends[G + 1] padding)
__global__ void k_d1_ends(const double* __restrict__ t, int64_t n, int64_t chunk, int G,
                          double* __restrict__ ends) {
  for (int b = threadIdx.x; b <= G + 1; b += blockDim.x)
    ends[b] = b == 0 ? t[0] : t[min((int64_t)min(b, G) * chunk, n) - 1];
}

}  // namespace lpc

// ---------------------------------------------------------------------------
// Host side.
gp_status db_launch(Plan& pl, const double* v, double* out, int nrhs, bool user_order,
                    cudaStream_t s, int kind);
int db_capacity_sub();

namespace {

// shapes (threads x points per thread); ITEMS odd: conflict-free 8-byte strided smem reads
struct Shape {
  int block, items;
  const void* fn[2][10];   // [user order][KIND * 5 + P]
  size_t smem[2];
};

template <int BLOCK, int SEGS, int SL, bool USER>
void shape_fns(const void** f) {
  f[0] = (const void*)lpc::k_d1_lpc<0, 0, BLOCK, SEGS, SL, USER>;
  f[1] = (const void*)lpc::k_d1_lpc<1, 0, BLOCK, SEGS, SL, USER>;
  f[2] = (const void*)lpc::k_d1_lpc<2, 0, BLOCK, SEGS, SL, USER>;
  f[3] = (const void*)lpc::k_d1_lpc<3, 0, BLOCK, SEGS, SL, USER>;
  f[4] = (const void*)lpc::k_d1_lpc<4, 0, BLOCK, SEGS, SL, USER>;
  f[5] = (const void*)lpc::k_d1_lpc<1, 1, BLOCK, SEGS, SL, USER>;
  f[6] = (const void*)lpc::k_d1_lpc<2, 1, BLOCK, SEGS, SL, USER>;
  f[7] = (const void*)lpc::k_d1_lpc<3, 1, BLOCK, SEGS, SL, USER>;
  f[8] = (const void*)lpc::k_d1_lpc<4, 1, BLOCK, SEGS, SL, USER>;
  f[9] = (const void*)lpc::k_d1_lpc<5, 1, BLOCK, SEGS, SL, USER>;
}
template <int BLOCK, int SEGS, int SL>
Shape make_shape() {
  Shape s;
  s.block = BLOCK;
  s.items = SEGS * SL;
  shape_fns<BLOCK, SEGS, SL, false>(s.fn[0]);
  shape_fns<BLOCK, SEGS, SL, true>(s.fn[1]);
  const size_t sub = (size_t)BLOCK * SEGS * SL;
  s.smem[0] = sizeof(double) * ((2 + lpc::lpc_nub(false, (int)sub)) * sub + 18);   // t, e, u buffers
  s.smem[1] = sizeof(double) * (3 * sub + 18 + 8);   // t, e, u (perm shares u's upper half)
  return s;
}

constexpr int NSHAPE = 3;
Shape g_shapes[NSHAPE];
int g_ready = 0;
int g_default = 0;

gp_status shapes_init() {
  if (g_ready) return GP_OK;
  g_shapes[0] = make_shape<256, 3, 9>();
  g_shapes[1] = make_shape<256, 3, 10>();   // #SMs x 7680 points: N = 2^20 in one chunk each
  g_shapes[2] = make_shape<256, 4, 7>();
  for (auto& s : g_shapes)
    for (int u = 0; u < 2; ++u)
      for (int p = 0; p < 10; ++p)
        GPM_CUDA(cudaFuncSetAttribute(s.fn[u][p], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)s.smem[u]));
  if (const char* e = getenv("GPM_D1_SHAPE")) g_default = std::max(0, std::min(NSHAPE - 1, atoi(e)));
  g_ready = 1;
  return GP_OK;
}

}  // namespace

gp_status d1_prepare(Plan& pl) {
  GPM_TRY(shapes_init());
  int dev = 0, nsm = 0, coop = 0;
  GPM_CUDA(cudaGetDevice(&dev));
  GPM_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  GPM_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  if (!coop) return fail(GP_ERR_UNSUPPORTED, "device does not support cooperative launch");
  // shape: the requested one, or (auto) the default and, above its capacity, the larger
  // ones (shape 1: #SMs x 7680 points, N = 2^20 in one chunk per CTA)
  const int first = pl.d1_shape >= 0 && pl.d1_shape < NSHAPE ? pl.d1_shape : g_default;
  const int last = pl.d1_shape >= 0 && pl.d1_shape < NSHAPE ? pl.d1_shape : NSHAPE - 1;
  for (int shp = first; shp <= last && pl.d1_force != 3; ++shp) {
    if (pl.d1_shape < 0 && shp != first && shp == 2) break;   // auto: shapes 0 and 1 only
    const Shape& sh = g_shapes[shp];
    int occ = 0;
    GPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sh.fn[1][2], sh.block, sh.smem[1]));
    const int64_t cap = (int64_t)sh.block * sh.items;
    const int gmax = std::min(occ * nsm, 160);   // s_tl holds 161 chunk ends
    if (gmax <= 0) continue;
    // grid: #SMs CTAs, fewer for small n (>= 1024 points per chunk); chunk a multiple of 4
    int64_t g = std::min<int64_t>(gmax, std::max<int64_t>(1, (pl.n + 1023) / 1024));
    int64_t chunk = ((pl.n + g - 1) / g + 3) & ~int64_t(3);
    g = (pl.n + chunk - 1) / chunk;   // every CTA owns >= 1 point
    if (chunk <= cap && g <= gmax) {
      pl.d1_shape_used = shp;
      pl.d1_grid = (int)g;
      pl.d1_chunk = chunk;
      pl.d1_path = 1;
      GPM_TRY(pl.aggs.alloc(sizeof(unsigned long long) * lpc::LL_W * 2 * (size_t)g));
      GPM_CUDA(cudaMemset(pl.aggs.ptr, 0, pl.aggs.bytes));
      GPM_TRY(pl.bar.alloc(sizeof(unsigned) * (size_t)g));
      GPM_CUDA(cudaMemset(pl.bar.ptr, 0, pl.bar.bytes));
      // plan data of the d = 1 path: e^{-gap} per rank (once) and the chunk ends
      if (pl.d1e.bytes < sizeof(double) * (size_t)(pl.n + 16)) {
        GPM_TRY(pl.d1e.alloc(sizeof(double) * (size_t)(pl.n + 16)));
        lpc::k_d1_e_build<<<148 * 4, 256>>>(pl.t.as<double>(), pl.n, pl.d1e.as<double>());
      }
      GPM_TRY(pl.d1ends.alloc(sizeof(double) * (size_t)(g + 2)));
      lpc::k_d1_ends<<<1, 256>>>(pl.t.as<double>(), pl.n, chunk, (int)g, pl.d1ends.as<double>());
      GPM_CUDA(cudaGetLastError());
      GPM_CUDA(cudaDeviceSynchronize());
      if (getenv("GPM_D1_TIMING")) {
        GPM_TRY(pl.dbg.alloc(sizeof(unsigned long long) * 16 * 32 * (size_t)g));
        GPM_CUDA(cudaMemset(pl.dbg.ptr, 0, pl.dbg.bytes));
      }
      return GP_OK;
    }
  }
  // path 3: reduce-then-scan over sub-tiles in three plain launches (apply_d1_big.cu), any N
  const int64_t nsub = (pl.n + db_capacity_sub() - 1) / db_capacity_sub();
  if (nsub > (int64_t)1 << 30) return fail(GP_ERR_UNSUPPORTED, "d=1 problem too large");
  pl.d1_grid = (int)nsub;
  pl.d1_chunk = db_capacity_sub();
  pl.d1_path = 3;
  GPM_TRY(pl.aggs.alloc(128 * 2 * (size_t)nsub));   // sub-tile records + carries
  return GP_OK;
}

gp_status d1_launch(Plan& pl, const double* v, double* out, int nrhs, bool user_order,
                    cudaStream_t s, int kind, double cg_s2, double* cg_part) {
  if (pl.d1_path == 3) {
    if (cg_part) return fail(GP_ERR_INVALID_ARG, "internal: no CG epilogue on the d=1 path 3");
    return db_launch(pl, v, out, nrhs, user_order, s, kind);
  }
  const Shape& sh = g_shapes[pl.d1_shape_used];
  lpc::Args a;
  a.ts = pl.t.as<double>();
  a.ends = pl.d1ends.as<double>();
  a.e1 = pl.d1e.as<double>();
  a.perm = pl.perm.as<int>();
  a.v = v;
  a.out = out;
  a.n = pl.n;
  a.n_src = user_order ? pl.n_src : pl.n;
  a.tgt_off = user_order ? pl.tgt_off : 0;
  a.chunk = pl.d1_chunk;
  a.nrhs = nrhs;
  a.prefetch = pl.d1_prefetch;
  a.vstride = user_order ? pl.n_src : pl.n;
  a.ostride = user_order ? pl.n - pl.tgt_off : pl.n;
  a.os2 = pl.os2;
  a.rec = pl.aggs.as<unsigned long long>();
  a.ep = pl.bar.as<unsigned>();
  a.dbg = pl.dbg.bytes ? pl.dbg.as<unsigned long long>() : nullptr;
  a.cg_s2 = cg_s2;
  a.cg_part = user_order ? nullptr : cg_part;
  static const int knob = getenv("GPM_D1_KNOB") ? atoi(getenv("GPM_D1_KNOB")) : 0;
  a.knob = knob;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.d1_grid);
  cfg.blockDim = dim3(sh.block);
  // user order: arrays sized by the chunk (+ one thread's items for the neutral tail window)
  a.cap = (int)std::min<int64_t>((int64_t)sh.block * sh.items,
                                 ((pl.d1_chunk + 3) & ~int64_t(3)) + ((sh.items + 3) & ~3));
  cfg.dynamicSmemBytes = (user_order && sh.items == 27) ? sizeof(double) * (3 * (size_t)a.cap + 18 + 8)
                                                          : sh.smem[user_order ? 1 : 0];
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  static const int nocoop = getenv("GPM_D1_NOCOOP") ? atoi(getenv("GPM_D1_NOCOOP")) : 0;   // timing experiment
  cfg.attrs = nocoop ? at + 1 : at;
  cfg.numAttrs = nocoop ? (pl.d1_pdl ? 1 : 0) : (pl.d1_pdl ? 2 : 1);
  void* args[] = {&a};
  GPM_CUDA(cudaLaunchKernelExC(&cfg, sh.fn[user_order ? 1 : 0][kind * 5 + pl.P], args));
  return GP_OK;
}

}  // namespace gpm
