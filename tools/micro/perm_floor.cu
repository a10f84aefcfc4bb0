// perm_floor.cu -- the user-order floor of the d = 1 apply: what moving 10^6 doubles through
// a random permutation costs on this B200, with no arithmetic at all.
//   copy    o[i] = v[i]                      (coalesced reference: 8 MB in, 8 MB out)
//   gather  o[i] = v[p[i]]                   (the apply's input permutation)
//   scatter o[p[i]] = v[i]                   (the apply's output permutation)
//   both    u = v[p[i]]; o[p[i]] = 2u         (gather + scatter in one pass)
// Each kernel runs R times back to back in one CUDA graph (grid = #SMs x 8, 256 threads);
// "L2" rows reuse one v / o pair (L2-resident), "HBM" rows cycle 64 pairs (1 GB).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o perm_floor perm_floor.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

__global__ void k_copy(const int* __restrict__, const double* __restrict__ v, double* __restrict__ o, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) o[i] = v[i];
}
__global__ void k_gather(const int* __restrict__ p, const double* __restrict__ v, double* __restrict__ o, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) o[i] = __ldg(v + __ldg(p + i));
}
__global__ void k_scatter(const int* __restrict__ p, const double* __restrict__ v, double* __restrict__ o, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) o[__ldg(p + i)] = v[i];
}
__global__ void k_both(const int* __restrict__ p, const double* __restrict__ v, double* __restrict__ o, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int j = __ldg(p + i);
    o[j] = 2.0 * __ldg(v + j);
  }
}

int main(int argc, char**) {
  const int n = 1000000, NV = 64, R = 100;
  const bool ncu_mode = argc > 1;   // plain launches only (for an ncu capture)
  std::vector<int> perm(n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  std::mt19937 rng(1);
  std::shuffle(perm.begin(), perm.end(), rng);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
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
  using K = void (*)(const int*, const double*, double*, int);
  K ks[] = {k_copy, k_gather, k_scatter, k_both};
  const char* names[] = {"copy", "gather", "scatter", "gather+scatter"};
  for (int hbm = 0; hbm < (ncu_mode ? 0 : 2); ++hbm) {
    for (int kind = 0; kind < 4; ++kind) {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      for (int r = 0; r < R; ++r) {
        const size_t off = hbm ? (size_t)(r % NV) * n : 0;
        ks[kind]<<<nsm * 8, 256, 0, s>>>(dp, dv + off, dout + off, n);
      }
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, s);   // warm
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
      printf("%-4s %-15s : %7.2f us per launch (best of 5 graph replays of %d)\n", hbm ? "HBM" : "L2",
             names[kind], best * 1e3 / R, R);
      cudaGraphExecDestroy(ge);
      cudaGraphDestroy(g);
    }
  }
  // one plain launch of each for an ncu capture (argv[1] given; the L2-resident case after
  // a warming launch)
  for (int kind = 0; kind < 4; ++kind) ks[kind]<<<nsm * 8, 256, 0, s>>>(dp, dv, dout, n);
  for (int kind = 0; kind < 4; ++kind) ks[kind]<<<nsm * 8, 256, 0, s>>>(dp, dv, dout, n);
  cudaStreamSynchronize(s);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
