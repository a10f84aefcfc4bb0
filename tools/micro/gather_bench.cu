// Microbenchmark: cost of random 8-byte gather / scatter vs coalesced streams on B200.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void k_copy(const double* __restrict__ a, double* __restrict__ b, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void k_gather(const int* __restrict__ p, const double* __restrict__ v, double* __restrict__ o, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) o[i] = __ldg(v + __ldg(p + i));
}
__global__ void k_scatter(const int* __restrict__ p, const double* __restrict__ v, double* __restrict__ o, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) o[__ldg(p + i)] = v[i];
}
__global__ void k_gs(const int* __restrict__ p, const double* __restrict__ v, double* __restrict__ o, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) { int j = __ldg(p + i); o[j] = 2.0 * __ldg(v + j); }
}
int main() {
  const int n = 1000000, NV = 64;
  std::vector<int> perm(n); for (int i = 0; i < n; ++i) perm[i] = i;
  std::mt19937 rng(1); std::shuffle(perm.begin(), perm.end(), rng);
  int* dp; double *dv, *dout; cudaMalloc(&dp, 4 * n); cudaMalloc(&dv, 8ull * n * NV); cudaMalloc(&dout, 8ull * n * NV);
  cudaMemcpy(dp, perm.data(), 4 * n, cudaMemcpyHostToDevice);
  cudaMemset(dv, 0, 8ull * n * NV);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"copy", "gather", "scatter", "gather+scatter"};
  for (int kind = 0; kind < 4; ++kind) for (int bs : {256, 1024}) for (int gm : {1, 4, 16}) {
    int grid = 148 * gm * (1024 / bs);
    auto run = [&](int r) {
      const double* v = dv + (size_t)(r % NV) * n; double* o = dout + (size_t)(r % NV) * n;
      if (kind == 0) k_copy<<<grid, bs>>>(v, o, n);
      else if (kind == 1) k_gather<<<grid, bs>>>(dp, v, o, n);
      else if (kind == 2) k_scatter<<<grid, bs>>>(dp, v, o, n);
      else k_gs<<<grid, bs>>>(dp, v, o, n);
    };
    for (int r = 0; r < 10; ++r) run(r);
    cudaEventRecord(e0);
    const int R = 200;
    for (int r = 0; r < R; ++r) run(r);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-15s bs=%4d grid=%6d : %7.2f us/launch\n", names[kind], bs, grid, ms * 1e3 / R);
  }
  return 0;
}
