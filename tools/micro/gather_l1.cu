// gather_l1.cu -- how the L1 size left by the shared-memory carve-out bounds the random
// 8-byte gathers / scatters of the d = 1 user-order apply.  One CTA per SM, 256 threads x 27
// consecutive ranks per thread (the k_d1_lpc shape), 10^6 points; the kernel allocates `smem`
// bytes of dynamic shared memory (unused) so that the driver picks the matching carve-out.
//   gather : u[k] = v[perm[j0 + k]] (27 independent loads per thread), summed into a sink
//   scatter: out[perm[j0 + k]] = x
// 100 launches per CUDA graph, best of 5 replays.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_l1 gather_l1.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

constexpr int ITEMS = 27, BLOCK = 256;

template <int MODE>
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
    for (int k2 = 0; k2 < ITEMS; ++k2) u[k2] = pi[k2] >= 0 ? __ldg(v + pi[k2]) : 0.0;
    double s = 0.0;
#pragma unroll
    for (int k2 = 0; k2 < ITEMS; ++k2) s += u[k2];
    if (s == 12345.678) sm[threadIdx.x] = s, out[0] = sm[0];
  } else {
    const double x = (double)threadIdx.x;
#pragma unroll
    for (int k2 = 0; k2 < ITEMS; ++k2) if (pi[k2] >= 0) out[pi[k2]] = x;
  }
}

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
  const int smems[] = {0, 64 * 1024, 100 * 1024, 132 * 1024 - 2048, 164 * 1024 - 2048, 196 * 1024 - 2048, 220 * 1024};
  for (int mode = 0; mode < 2; ++mode) {
    auto fn = mode == 0 ? k<0> : k<1>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    for (int hbm = 0; hbm < 2; ++hbm)
      for (int smem : smems) {
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
        printf("%-7s %-3s dynamic smem %3d KB: %6.2f us per launch\n", mode ? "scatter" : "gather",
               hbm ? "HBM" : "L2", smem / 1024, best * 1e3 / R);
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
      }
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
