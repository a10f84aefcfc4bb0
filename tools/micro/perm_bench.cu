// Microbenchmark: grid-barrier cost and a two-phase "partition" permutation
// (u[r] = v[perm[r]]) that keeps global traffic coalesced and does the random part in smem.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ void gbar(unsigned* bar, unsigned nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vg = bar + 1;
    unsigned gen = *vg;
    __threadfence();
    if (atomicAdd(bar, 1u) == nb - 1) { atomicExch(bar, 0u); __threadfence(); atomicAdd(bar + 1, 1u); }
    else { unsigned cur; do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory"); } while (cur == gen); }
    __threadfence();
  }
  __syncthreads();
}

__global__ void k_barriers(unsigned* bar, int k) { for (int i = 0; i < k; ++i) gbar(bar, gridDim.x); }
__global__ void k_gridsync(int k) { cg::grid_group g = cg::this_grid(); for (int i = 0; i < k; ++i) g.sync(); }

// phase A+B in one cooperative kernel
__global__ void __launch_bounds__(1024, 1) k_part(const double* __restrict__ v, const unsigned short* __restrict__ lk,
    const int* __restrict__ gp, const unsigned short* __restrict__ bo, double* __restrict__ stg,
    double* __restrict__ u, int n, int C, unsigned* bar) {
  extern __shared__ double sm[];
  const int b = blockIdx.x, i0 = b * C, cnt = min(C, n - i0);
  for (int k = threadIdx.x; k < cnt; k += blockDim.x) sm[lk[i0 + k]] = __ldg(v + i0 + k);
  __syncthreads();
  for (int k = threadIdx.x; k < cnt; k += blockDim.x) stg[gp[i0 + k]] = sm[k];
  gbar(bar, gridDim.x);
  for (int k = threadIdx.x; k < cnt; k += blockDim.x) sm[k] = __ldcg(stg + i0 + k);
  __syncthreads();
  for (int k = threadIdx.x; k < cnt; k += blockDim.x) u[i0 + k] = sm[bo[i0 + k]];
}
__global__ void k_direct(const int* __restrict__ p, const double* __restrict__ v, double* __restrict__ u, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) u[i] = __ldg(v + __ldg(p + i));
}

int main() {
  const int n = 1000000, G = 148, C = (n + G - 1) / G, NV = 64;
  std::vector<int> perm(n); for (int i = 0; i < n; ++i) perm[i] = i;
  std::mt19937 rng(1); std::shuffle(perm.begin(), perm.end(), rng);
  std::vector<int> inv(n); for (int r = 0; r < n; ++r) inv[perm[r]] = r;
  // staging layout: bucket c at [c*C, ...), runs ordered by source slice b
  std::vector<unsigned short> lk(n), bo(n); std::vector<int> gp(n);
  std::vector<std::vector<int>> cnt(G, std::vector<int>(G, 0));
  for (int i = 0; i < n; ++i) cnt[inv[i] / C][i / C]++;
  std::vector<std::vector<int>> off(G, std::vector<int>(G, 0));
  for (int c = 0; c < G; ++c) { int o = 0; for (int b = 0; b < G; ++b) { off[c][b] = o; o += cnt[c][b]; } }
  std::vector<int> stpos(n);
  for (int b = 0; b < G; ++b) {
    int i0 = b * C, i1 = std::min(n, i0 + C);
    std::vector<int> idx; for (int i = i0; i < i1; ++i) idx.push_back(i);
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int c) { return inv[a] / C < inv[c] / C; });
    std::vector<int> fill(G, 0);
    for (int k = 0; k < (int)idx.size(); ++k) {
      int i = idx[k], c = inv[i] / C;
      lk[i] = (unsigned short)k;
      int sp = c * C + off[c][b] + fill[c]++;
      gp[i0 + k] = sp; stpos[i] = sp;
    }
  }
  for (int r = 0; r < n; ++r) bo[r] = (unsigned short)(stpos[perm[r]] - (r / C) * C);
  int *dp, *dgp; unsigned short *dlk, *dbo; double *dv, *du, *dst; unsigned* bar;
  cudaMalloc(&dp, 4 * n); cudaMalloc(&dgp, 4 * n); cudaMalloc(&dlk, 2 * n); cudaMalloc(&dbo, 2 * n);
  cudaMalloc(&dv, 8ull * n * NV); cudaMalloc(&du, 8ull * n * NV); cudaMalloc(&dst, 8ull * n); cudaMalloc(&bar, 64);
  cudaMemset(bar, 0, 64);
  cudaMemcpy(dp, perm.data(), 4 * n, cudaMemcpyHostToDevice); cudaMemcpy(dgp, gp.data(), 4 * n, cudaMemcpyHostToDevice);
  cudaMemcpy(dlk, lk.data(), 2 * n, cudaMemcpyHostToDevice); cudaMemcpy(dbo, bo.data(), 2 * n, cudaMemcpyHostToDevice);
  std::vector<double> hv(n); for (int i = 0; i < n; ++i) hv[i] = i;
  for (int r = 0; r < NV; ++r) cudaMemcpy(dv + (size_t)r * n, hv.data(), 8 * n, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto fn) {
    for (int r = 0; r < 5; ++r) fn(r);
    cudaEventRecord(e0); const int R = 200; for (int r = 0; r < R; ++r) fn(r);
    cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-34s %8.2f us  (%s)\n", name, ms * 1e3 / R, cudaGetErrorString(cudaGetLastError()));
  };
  for (int k : {0, 1, 4}) {
    char nm[64]; sprintf(nm, "coop empty kernel, %d barriers", k);
    timeit(nm, [&](int) { void* a[] = {&bar, &k}; cudaLaunchCooperativeKernel((void*)k_barriers, dim3(148), dim3(512), a, 0, 0); });
    sprintf(nm, "normal launch, %d barriers", k);
    timeit(nm, [&](int) { k_barriers<<<148, 512>>>(bar, k); });
    sprintf(nm, "cg grid.sync, %d syncs", k);
    timeit(nm, [&](int) { void* a[] = {&k}; cudaLaunchCooperativeKernel((void*)k_gridsync, dim3(148), dim3(512), a, 0, 0); });
  }
  cudaFuncSetAttribute(k_part, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * C + 64);
  timeit("direct gather", [&](int r) { k_direct<<<592, 1024>>>(dp, dv + (size_t)(r % NV) * n, du + (size_t)(r % NV) * n, n); });
  timeit("partition gather (coop)", [&](int r) {
    const double* v = dv + (size_t)(r % NV) * n; double* u = du + (size_t)(r % NV) * n; int nn = n, CC = C;
    void* a[] = {&v, &dlk, &dgp, &dbo, &dst, &u, &nn, &CC, &bar};
    cudaLaunchCooperativeKernel((void*)k_part, dim3(G), dim3(1024), a, 8 * C + 64, 0); });
  // verify
  std::vector<double> hu(n); cudaMemcpy(hu.data(), du + (size_t)((205 - 1) % NV) * n, 8 * n, cudaMemcpyDeviceToHost);
  int bad = 0; for (int r = 0; r < n; ++r) bad += hu[r] != (double)perm[r];
  printf("partition verify bad=%d\n", bad);
  return 0;
}
