// algebra.cuh -- the overflow-free moment algebra behind the ECDF decomposition.
//
// The paper writes K.v as weighted ECDFs of v with global weights
// y_i (delta.x_i)^p exp(sqrt(2nu)/l delta.x_i)   (P:598-602 [eq matern_weights]),
// which overflow for |t| > 709 and cancel catastrophically.  We carry the SAME sums
// referenced at the current scan position instead (reading R5):
//
//   moment state   M_q = sum_{i in S} u_i s_i^q e^{-s_i},  q = 0..P,  s_i >= 0 the
//                  distance of source i from the current position;
//   advance by D   M'_q = e^{-D} sum_{m<=q} C(q,m) D^{q-m} M_m        (all terms >= 0)
//   inject source  M_q += u alpha^q e^{-alpha}   (alpha = offset from a split reference)
//   read target    e^{-beta} sum_q a_q sum_{m<=q} C(q,m) beta^{q-m} M_m
//
// with the profile k(s) = sum_q a_q s^q e^{-s} of nu = P + 1/2 in scaled coordinates
// (P:1282 [eq matern_explicit]: a = [1], [1,1], [1,1,1/3], ...).  Advances compose,
// S(a)S(b) = S(a+b), so (span, moments) is an associative scan monoid; this is the
// "fast sum updating" of P:326-337 [§2.1] evaluated in a numerically safe basis.
//
// Product form: the state is M[m][q] = sum u alpha^m e^{-alpha} s^q e^{-s};
// the scan advance acts on q, the split offset on m.
#pragma once
#include <cstdint>

namespace gpm {

// Small exact tables (literal constants, no loops or divisions at run time: every use sits
// in a fully unrolled loop, so each call folds to one immediate).
// Binomial C(q, m), q <= 6.
__host__ __device__ __forceinline__ constexpr double binom(int q, int m) {
  return (m < 0 || m > q) ? 0.0
         : (m == 0 || m == q) ? 1.0
         : (m == 1 || m == q - 1) ? double(q)
         : q == 4 ? 6.0
         : q == 5 ? 10.0
         : (m == 3 ? 20.0 : 15.0);   // q == 6
}
// Matern coefficients of nu = p + 1/2 in scaled distance s = sqrt(2p+1) |u| (P:1282
// [eq matern_explicit]: a_q = C(p,q) (2p-q)! / (2p)! 2^q), p <= 4: [1], [1,1], [1,1,1/3],
// [1,1,2/5,1/15], [1,1,3/7,2/21,1/105]; zero outside 0..p.
__host__ __device__ __forceinline__ constexpr double mcoef(int p, int q) {
  return (q < 0 || q > p) ? 0.0
         : q <= 1 ? 1.0
         : p == 2 ? 1.0 / 3.0
         : p == 3 ? (q == 2 ? 2.0 / 5.0 : 1.0 / 15.0)
         : (q == 2 ? 3.0 / 7.0 : q == 3 ? 2.0 / 21.0 : 1.0 / 105.0);   // p == 4
}

// Advance a (P+1)-moment vector by D (E = e^{-D}).  In place, high q first.
template <int P>
__device__ __forceinline__ void advance(double* M, double D, double E) {
  if constexpr (P > 3) {
    // M'_q = E sum_{m<=q} C(q,m) D^{q-m} M_m, Horner in D; q descending keeps M_m (m < q)
#pragma unroll
    for (int q = P; q >= 0; --q) {
      double acc = M[0];
#pragma unroll
      for (int m = 1; m <= q; ++m) acc = fma(acc, D, binom(q, m) * M[m]);
      M[q] = E * acc;
    }
  } else if constexpr (P == 3) {
    // M3 + 3D M2 + 3D^2 M1 + D^3 M0 = M3 + D (3 M2 + D (3 M1 + D M0))
    const double a = fma(D, M[0], M[1]);
    const double b = fma(D, fma(D, M[0], 3.0 * M[1]), 3.0 * M[2]);
    M[3] = E * fma(D, b, M[3]);
    M[2] = E * fma(D, M[1] + a, M[2]);
    M[1] = E * a;
    M[0] = E * M[0];
  } else if constexpr (P == 2) {
    // M2 + 2D M1 + D^2 M0 = M2 + D (M1 + (M1 + D M0)):  6 FP64 ops
    const double a = fma(D, M[0], M[1]);
    M[2] = E * fma(D, M[1] + a, M[2]);
    M[1] = E * a;
    M[0] = E * M[0];
  } else if constexpr (P == 1) {
    M[1] = E * fma(D, M[0], M[1]);
    M[0] = E * M[0];
  } else {
    M[0] = E * M[0];
  }
}

// out = S(D) A + B  (elementwise on P+1 moments)
template <int P>
__device__ __forceinline__ void advance_add(double* A, double D, double E, const double* B) {
  advance<P>(A, D, E);
#pragma unroll
  for (int q = 0; q <= P; ++q) A[q] += B[q];
}

// sum_q a_q sum_{m<=q} C(q,m) beta^{q-m} R_m   (without the e^{-beta} factor)
template <int P>
__device__ __forceinline__ double read_poly(const double* R, double beta) {
  if constexpr (P > 2) {
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q <= P; ++q) {
      double t = 0.0, bp = 1.0;
#pragma unroll
      for (int m = q; m >= 0; --m) {
        t = fma(binom(q, m) * bp, R[m], t);
        bp *= beta;
      }
      acc = fma(mcoef(P, q), t, acc);
    }
    return acc;
  } else if constexpr (P == 2) {
    // a0 R0 + a1 (R1 + b R0) + a2 (R2 + 2 b R1 + b^2 R0)
    const double b = beta;
    return R[0] + (R[1] + b * R[0]) + (1.0 / 3.0) * fma(b * b, R[0], fma(2.0 * b, R[1], R[2]));
  } else if constexpr (P == 1) {
    return R[0] + fma(beta, R[0], R[1]);
  } else {
    return R[0];
  }
}

// sum_q a_q R_q  (beta = 0)
template <int P>
__device__ __forceinline__ double read0(const double* R) {
  if constexpr (P > 2) {
    double acc = 0.0;
#pragma unroll
    for (int q = P; q >= 0; --q) acc = fma(mcoef(P, q), R[q], acc);
    return acc;
  } else if constexpr (P == 2) return fma(1.0 / 3.0, R[2], R[0] + R[1]);
  else if constexpr (P == 1) return R[0] + R[1];
  else return R[0];
}

// ---------------------------------------------------------------------------
// Read profiles.  KIND 0: the Matern profile k(s) = sum_q a_q s^q e^{-s} of nu = PM + 1/2
// (moments q <= PM).  KIND 1: the lengthscale-gradient profile of nu = PM - 1/2,
//   g(s) = -s k'(s) = sum_m b_m s^m e^{-s},  b_m = a_{m-1} - m a_m   (moments m <= PM),
// so that dK/d(log l) = varsigma^2 g(s): P:1309 [eq dkernel_dl] with the closed forms
// P:1321-1323 (nu=1/2: s e^{-s}; 3/2: s^2 e^{-s}; 5/2: (s^2 + s^3)/3 e^{-s}).
// KIND 0: a_q of nu = PM + 1/2; KIND 1: b_q = a_{q-1} - q a_q of nu = PM - 1/2 (g = -s k'(s))
__host__ __device__ __forceinline__ constexpr double rcoef(int PM, int KIND, int q) {
  return KIND == 0 ? mcoef(PM, q) : mcoef(PM - 1, q - 1) - q * mcoef(PM - 1, q);
}
// sum_q c_q R_q
template <int PM, int KIND>
__device__ __forceinline__ double readc0(const double* R) {
  if constexpr (KIND == 0) {
    return read0<PM>(R);
  } else {
    if constexpr (PM == 1) return R[1];
    else if constexpr (PM == 2) return R[2];
    else if constexpr (PM == 3) return (1.0 / 3.0) * (R[2] + R[3]);
    else {
      double acc = 0.0;
#pragma unroll
      for (int q = PM; q >= 0; --q)
        if (rcoef(PM, 1, q) != 0.0) acc = fma(rcoef(PM, 1, q), R[q], acc);
      return acc;
    }
  }
}
// sum_q c_q sum_{m<=q} C(q,m) beta^{q-m} R_m   (without e^{-beta})
template <int PM, int KIND>
__device__ __forceinline__ double readc_poly(const double* R, double beta) {
  if constexpr (KIND == 0) {
    return read_poly<PM>(R, beta);
  } else {
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q <= PM; ++q) {
      if (rcoef(PM, KIND, q) != 0.0) {
        double t = 0.0, bp = 1.0;
#pragma unroll
        for (int m = q; m >= 0; --m) {   // sum_m C(q,m) beta^{q-m} R_m
          t = fma(binom(q, m) * bp, R[m], t);
          bp *= beta;
        }
        acc = fma(rcoef(PM, KIND, q), t, acc);
      }
    }
    return acc;
  }
}

// x^e, small runtime e >= 0 (x^0 = 1 also at x = 0)
__device__ __forceinline__ double powi(double x, int e) {
  double r = 1.0;
  for (int i = 0; i < e; ++i) r *= x;
  return r;
}
// target factor of a separated split profile sum_q c_q s^q e^{-s} (c = rcoef(PM, KIND, .):
// k of nu = PM + 1/2, or g of nu = PM - 1/2): sum_{q=a..PM} c_q C(q,a) beta^{q-a}; runtime a,
// 0 for a > PM
template <int PM, int KIND>
__device__ __forceinline__ double tpoly(int a, double beta) {
  double acc = 0.0;
#pragma unroll
  for (int q = PM; q >= 0; --q)
    if (q >= a) acc = fma(acc, beta, rcoef(PM, KIND, q) * binom(q, a));
  return acc;
}

// ---------------------------------------------------------------------------
// Multi-channel algebra for the d >= 2 level passes.
//   NCH channels (2 for d = 2: side of the x1 split; 4 for d = 3: sides of the x1 and
//   inner x2 splits).  A source on channel c feeds targets on channel NCH-1-c.
//   NM moments per channel: P+1 (L1) or (P+1)^2 (product, d = 2).
//
// Product form, d = 3 (P3; P:414-416, P:487-509 [Prop 2]): each split factor separates,
//   k(a_s + a_t) = sum_{a<=P} [a_s^a e^{-a_s}] [e^{-a_t} sum_{q>=a} a_q C(q,a) a_t^{q-a}],
// so the pair sum over a node is sum_{a,b} T_a(alpha1_t) T_b(alpha2_t) times a scan along the
// last coordinate with source weights u alpha1^a alpha2^b e^{-alpha1-alpha2} and NO split
// offset: the L1 engine (P+1 moments per channel) run NAB = (P+1)^2 times per level with
// re-weighted sources and a target multiplier (tpoly), instead of a (P+1)^3-moment state.
//
// The same separation gives the lengthscale gradient of the product forms (product rule,
// P:1301-1327): with g(s) = -s k'(s) of order p+1, g(a_s + a_t) = sum_{a<=p+1} [a_s^a e^{-a_s}]
// Tg_a(a_t), in two runs summed by the epilogue:
//   SEP 2: scan profile k (engine order p, KIND 0), split factors g k + k g (d = 3: g1 k2 k3 +
//          k1 g2 k3), sub-passes (a, b) <= p+1, target factor Tg_a Tk_b + Tk_a Tg_b;
//   SEP 3: scan profile g (engine order p+1, KIND 1), split factors k (k1 k2 g3), target
//          factor Tk_a Tk_b with the order-p coefficients.
// SEP 1 is the value.  d = 2 (NCH = 2) has one split factor: b = 0, alpha2 = 0.
template <int P_, int NCH_, bool PROD_, int KIND_ = 0, int SEP_ = 0>
struct Alg {
  static constexpr int P = P_;          // moment order (gradient: nu - 1/2 + 1)
  static constexpr int NCH = NCH_;
  static constexpr bool PROD = PROD_;   // product form (mixed-moment state, d = 2)
  static constexpr int KIND = KIND_;
  static constexpr int SEP = SEP_;      // separated product form (sub-passes of the L1 engine)
  static constexpr bool P3 = SEP != 0;
  static constexpr bool ST2 = P3 && NCH == 4;   // staged structure holds alpha1 and alpha2
  static constexpr int NQ = P + 1;
  static constexpr int P0 = SEP == 3 ? P - 1 : P;             // nu - 1/2 of the kernel
  static constexpr int NA = !P3 ? 1 : (SEP == 2 ? P0 + 2 : P0 + 1);
  static constexpr int NB = NCH == 4 ? NA : 1;
  // SEP 2, d = 3: the last pair (p+1, p+1) has a zero target factor
  static constexpr int NAB = NA * NB - ((SEP == 2 && NCH == 4) ? 1 : 0);
  static constexpr int NM = PROD ? NQ * NQ : NQ;
  static constexpr int NS = NCH * NM;

  __device__ __forceinline__ static void advance_all(double* M, double D, double E) {
#pragma unroll
    for (int r = 0; r < NS / NQ; ++r) advance<P>(M + r * NQ, D, E);
  }

  // M[c] += injection of u at split offset alpha (ea = e^{-alpha}).  Branch-free: the
  // channel is a per-lane value (divergent), so every channel takes a masked FMA.
  __device__ __forceinline__ static void inject(double* M, int c, double u, double alpha,
                                                double ea) {
    double pw[NQ];
    pw[0] = u * ea;
#pragma unroll
    for (int q = 1; q < NQ; ++q) pw[q] = pw[q - 1] * alpha;
#pragma unroll
    for (int cc = 0; cc < NCH; ++cc) {
      const double msk = cc == c ? 1.0 : 0.0;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        if constexpr (!PROD) M[cc * NM + q] = fma(msk, pw[q], M[cc * NM + q]);
        else M[cc * NM + q * NQ + 0] = fma(msk, pw[q], M[cc * NM + q * NQ + 0]);
      }
    }
  }

  // M[c] += the injection of u at split offset alpha, shifted along the scan by a span D
  // (E = e^{-D}): the source's moments seen from a point D further on (direct form of
  // inject followed by advance(D), used by the reduce loops: no full-state advance).
  __device__ __forceinline__ static void inject_at(double* M, int c, double u, double alpha,
                                                   double ea, double D, double E) {
    if constexpr (!PROD) {
      inject(M, c, u * E, alpha + D, ea);
    } else {
      double pm[NM];
      double pa = u * ea * E;
#pragma unroll
      for (int m = 0; m < NQ; ++m) {
        double pq = pa;
#pragma unroll
        for (int q = 0; q < NQ; ++q) { pm[m * NQ + q] = pq; pq *= D; }
        pa *= alpha;
      }
#pragma unroll
      for (int cc = 0; cc < NCH; ++cc) {
        const double msk = cc == c ? 1.0 : 0.0;
#pragma unroll
        for (int i = 0; i < NM; ++i) M[cc * NM + i] = fma(msk, pm[i], M[cc * NM + i]);
      }
    }
  }

  // value contributed to a target on channel rc at split offset beta (eb = e^{-beta})
  // Branch-free: the channel's moments are selected first, then read once.
  __device__ __forceinline__ static double read(const double* M, int rc, double beta,
                                                double eb) {
    double Ms[NM];
#pragma unroll
    for (int i = 0; i < NM; ++i) Ms[i] = M[i];
#pragma unroll
    for (int cc = 1; cc < NCH; ++cc)
#pragma unroll
      for (int i = 0; i < NM; ++i) Ms[i] = cc == rc ? M[cc * NM + i] : Ms[i];
    double v;
    if constexpr (!PROD) {
      v = readc_poly<P, KIND>(Ms, beta);
    } else if constexpr (KIND == 0) {
      // k(alpha+beta) k(s): e^{-beta} sum_a a_a sum_{m<=a} C(a,m) beta^{a-m} (sum_q a_q M[m][q])
      double G[NQ];
#pragma unroll
      for (int m = 0; m < NQ; ++m) G[m] = read0<P>(Ms + m * NQ);
      v = read_poly<P>(G, beta);
    } else {
      // lengthscale gradient of k(r1) k(r2) (product rule): g(r1) k(r2) + k(r1) g(r2), with
      // k of order P - 1 (coefficients a) and g = -s k'(s) of order P (coefficients b)
      double Ga[NQ], Gb[NQ];
#pragma unroll
      for (int m = 0; m < NQ; ++m) {
        Ga[m] = readc0<P - 1, 0>(Ms + m * NQ);
        Gb[m] = readc0<P, 1>(Ms + m * NQ);
      }
      v = readc_poly<P, 1>(Ga, beta) + readc_poly<P - 1, 0>(Gb, beta);
    }
    return eb * v;
  }

  // separated forms: source weight and target factor of sub-pass ab = pa * NB + pb
  __device__ __forceinline__ static double srcw(double a1, double a2, int ab) {
    const int pa = ab / NB, pb = ab - pa * NB;
    return powi(a1, pa) * powi(a2, pb);
  }
  __device__ __forceinline__ static double tgtw(double a1, double a2, int ab) {
    const int pa = ab / NB, pb = ab - pa * NB;
    if constexpr (SEP == 2)
      return tpoly<P0 + 1, 1>(pa, a1) * tpoly<P0, 0>(pb, a2) +
             tpoly<P0, 0>(pa, a1) * tpoly<P0 + 1, 1>(pb, a2);
    else
      return tpoly<P0, 0>(pa, a1) * tpoly<P0, 0>(pb, a2);
  }
};

}  // namespace gpm
