// fexp.cuh -- branch-free e^{-d} for d >= 0 in float64 (~2 ulp), used for the e^{-gap}
// and e^{-alpha} factors of the moment scans.  d = (n/64) ln2 - r with a 64-entry table
// 2^{k/64} in shared memory and a degree-5 Taylor polynomial on |r| <= ln2/128
// (truncation 3.5e-17 relative).  One-FMA range reduction: the rounding of ln2/64 costs
// ~3e-17*d relative, negligible wherever e^{-d} is not (d <= 40).  The scale 2^m is added
// to the table value's exponent as an integer.  9 FP64 instructions; e^{-0} == 1 exactly
// (ties); d >= 708 -> 0.  Constants sit in the constant bank (DFMA c[] operands), unlike
// libdevice exp() whose 64-bit immediates cost UMOV pairs and a slow-path branch.
#pragma once

namespace gpm {

__constant__ double c_fexp[8] = {
    92.33248261689366,        // 64 / ln2
    6755399441055744.0,       // 1.5 * 2^52 (round-to-int magic)
    0.010830424696249145,     // ln2 / 64
    1.0, 1.0, 0.5, 0.16666666666666666, 0.041666666666666664,
};
__constant__ double c_fexp5 = 0.008333333333333333;   // 1/120

// 2^{k/64}, correctly rounded
__constant__ double c_fexp_tab[64] = {
1.0,
    1.0108892860517005,
    1.0218971486541166,
    1.0330248790212284,
    1.0442737824274138,
    1.0556451783605572,
    1.0671404006768237,
    1.0787607977571199,
    1.0905077326652577,
    1.102382583307841,
    1.1143867425958924,
    1.1265216186082418,
    1.1387886347566916,
    1.1511892299529827,
    1.1637248587775775,
    1.1763969916502812,
    1.189207115002721,
    1.202156731452703,
    1.215247359980469,
    1.22848053610687,
    1.241857812073484,
    1.255380757024691,
    1.2690509571917332,
    1.2828700160787783,
    1.2968395546510096,
    1.3109612115247644,
    1.3252366431597413,
    1.339667524053303,
    1.3542555469368927,
    1.3690024229745905,
    1.383909881963832,
    1.3989796725383112,
    1.4142135623730951,
    1.42961333839197,
    1.4451808069770467,
    1.460917794180647,
    1.4768261459394993,
    1.4929077282912648,
    1.5091644275934228,
    1.5255981507445384,
    1.5422108254079407,
    1.559004400237837,
    1.5759808451078865,
    1.593142151342267,
    1.6104903319492543,
    1.6280274218573478,
    1.645755478153965,
    1.6636765803267364,
    1.681792830507429,
    1.7001063537185235,
    1.718619298122478,
    1.7373338352737062,
    1.7562521603732995,
    1.7753764925265212,
    1.7947090750031072,
    1.8142521755003989,
    1.8340080864093424,
    1.8539791250833855,
    1.8741676341103,
    1.8945759815869656,
    1.9152065613971474,
    1.9360617934922943,
    1.9571441241754002,
    1.978456026387951};

__device__ __forceinline__ void fexp_table_init(double* tab) {
  for (int i = threadIdx.x; i < 64; i += blockDim.x) tab[i] = c_fexp_tab[i];
}

// e^{-d}, d >= 0 (tab = the shared table above)
__device__ __forceinline__ double fexp_neg(double d, const double* tab) {
  const double x = -d;
  const double t = fma(x, c_fexp[0], c_fexp[1]);
  const int n = __double2loint(t);            // rint(x * 64/ln2) (two's complement low word)
  const double nd = t - c_fexp[1];
  const double r = fma(-nd, c_fexp[2], x);
  double p = fma(c_fexp5, r, c_fexp[7]);
  p = fma(p, r, c_fexp[6]);
  p = fma(p, r, c_fexp[5]);
  p = fma(p, r, c_fexp[4]);
  p = fma(p, r, c_fexp[3]);
  const double tk = tab[n & 63];
  const int m = n >> 6;                        // floor(n / 64)
  const double T = __hiloint2double(__double2hiint(tk) + (m << 20), __double2loint(tk));
  return d < 708.0 ? p * T : 0.0;
}

}  // namespace gpm
