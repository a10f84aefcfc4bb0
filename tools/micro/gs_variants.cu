// gs_variants.cu -- cache-operator variants of the d = 1 user-order gather and scatter
// (one CTA per SM, 256 threads x 27 items, 162 KB of dynamic shared memory like k_d1_lpc's
// user-order launch at N = 10^6; 100 launches per CUDA graph, best of 5 replays; "L2" = one
// v / out pair, "HBM" = 64 pairs cycled).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gs_variants gs_variants.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

constexpr int ITEMS = 27, BLOCK = 256;

template <int V>
__device__ __forceinline__ double ld(const double* p) {
  if (V == 0) return __ldg(p);
  if (V == 1) return __ldcg(p);
  if (V == 2) return __ldcs(p);
  if (V == 3) return __ldlu(p);
  double x;
  asm volatile("ld.global.L1::no_allocate.f64 %0, [%1];" : "=d"(x) : "l"(p));
  return x;
}
template <int V>
__device__ __forceinline__ void st(double* p, double x) {
  if (V == 0) *p = x;
  else if (V == 1) __stcg(p, x);
  else if (V == 2) __stcs(p, x);
  else if (V == 3) __stwt(p, x);
  else asm volatile("st.global.L1::no_allocate.f64 [%0], %1;" ::"l"(p), "d"(x) : "memory");
}

template <int MODE, int V>
__global__ void __launch_bounds__(BLOCK, 1) k(const int* __restrict__ perm, const double* __restrict__ v,
                                              double* __restrict__ out, int n, int chunk) {
  extern __shared__ double sm[];
  const int c0 = blockIdx.x * chunk;
  const int j0 = c0 + threadIdx.x * ITEMS;
  int pi[ITEMS];
#pragma unroll
  for (int k2 = 0; k2 < ITEMS; ++k2) pi[k2] = (j0 + k2 < min(n, c0 + chunk)) ? __ldg(perm + j0 + k2) : -1;
  if (MODE == 0) {
    double u[ITEMS];
#pragma unroll
    for (int k2 = 0; k2 < ITEMS; ++k2) u[k2] = pi[k2] >= 0 ? ld<V>(v + pi[k2]) : 0.0;
    double s = 0.0;
#pragma unroll
    for (int k2 = 0; k2 < ITEMS; ++k2) s += u[k2];
    if (s == 12345.678) sm[threadIdx.x] = s, out[0] = sm[0];
  } else {
    const double x = (double)threadIdx.x;
#pragma unroll
    for (int k2 = 0; k2 < ITEMS; ++k2) if (pi[k2] >= 0) st<V>(out + pi[k2], x);
  }
}

using K = void (*)(const int*, const double*, double*, int, int);

int main() {
  const int n = 1000000, NV = 64, R = 100;
  std::vector<int> perm(n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  std::mt19937 rng(1);
  std::shuffle(perm.begin(), perm.end(), rng);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int chunk = ((n + nsm - 1) / nsm + 3) & ~3;
  int* dp;
  double *dv, *dout;
  cudaMalloc(&dp, 4 * n);
  cudaMalloc(&dv, 8ull * n * NV);
  cudaMalloc(&dout, 8ull * n * NV);
  cudaMemcpy(dp, perm.data(), 4 * n, cudaMemcpyHostToDevice);
  cudaMemset(dv, 0, 8ull * n * NV);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  K fns[2][5] = {{k<0, 0>, k<0, 1>, k<0, 2>, k<0, 3>, k<0, 4>}, {k<1, 0>, k<1, 1>, k<1, 2>, k<1, 3>, k<1, 4>}};
  const char* names[2][5] = {{"ld.nc (__ldg)", "ld.cg", "ld.cs", "ld.lu", "ld L1::no_allocate"},
                             {"st", "st.cg", "st.cs", "st.wt", "st L1::no_allocate"}};
  const int smem = 162 * 1024;
  for (int mode = 0; mode < 2; ++mode)
    for (int var = 0; var < 5; ++var) {
      K fn = fns[mode][var];
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      for (int hbm = 0; hbm < 2; ++hbm) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int r = 0; r < R; ++r) {
          const size_t off = hbm ? (size_t)(r % NV) * n : 0;
          fn<<<nsm, BLOCK, smem, s>>>(dp, dv + off, dout + off, n, chunk);
        }
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, s);
        cudaStreamSynchronize(s);
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
          cudaEventRecord(e0, s);
          cudaGraphLaunch(ge, s);
          cudaEventRecord(e1, s);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          best = std::min(best, ms);
        }
        printf("%-7s %-20s %-3s: %6.2f us per launch\n", mode ? "scatter" : "gather", names[mode][var],
               hbm ? "HBM" : "L2", best * 1e3 / R);
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
      }
    }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
