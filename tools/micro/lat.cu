// Microbenchmark: latencies that set the d = 1 kernel's fixed costs on B200 (sm_100a):
// dependent DFMA / DADD chains, double SHFL chain, __syncthreads (768 thr),
// __threadfence after a store, cooperative grid.sync (148 x 768), L2-hit pointer chase.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a lat.cu -o lat
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_chain(double* out, long long* cyc, double b, double c) {
  double a = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a = fma(a, b, c);
  }
  long long t1 = clock64();
  double x = threadIdx.x;
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x = x + c;
  }
  long long t2 = clock64();
  double y = a + x;
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) y = __shfl_xor_sync(0xffffffffu, y, 1 + (k & 3)) + c;
  }
  long long t3 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
  out[threadIdx.x] = y;
}
__global__ void __launch_bounds__(768, 1) k_sync(double* out, long long* cyc, unsigned long long* gt) {
  long long t0 = clock64();
  for (int i = 0; i < 1000; ++i) __syncthreads();
  long long t1 = clock64();
  for (int i = 0; i < 100; ++i) {
    if (threadIdx.x == 0) { out[blockIdx.x * 64] = i; __threadfence(); }
    __syncthreads();
  }
  long long t2 = clock64();
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < 3; ++i) g.sync();
  unsigned long long a, b;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(a));
  for (int i = 0; i < 100; ++i) g.sync();
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(b));
  long long t3 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) { cyc[3] = t1 - t0; cyc[4] = t2 - t1; cyc[5] = t3 - t2; gt[0] = b - a; }
}
__global__ void k_chase(const int* __restrict__ nxt, long long* cyc, int* sink) {
  int p = 0;
  for (int i = 0; i < 64; ++i) p = __ldcg(nxt + p);   // warm
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) p = __ldcg(nxt + p);
  long long t1 = clock64();
  cyc[6] = t1 - t0;
  *sink = p;
}
int main() {
  double* out; long long* cyc; unsigned long long* gt; int *nxt, *sink;
  cudaMalloc(&out, 8 * 148 * 64 * 2); cudaMalloc(&cyc, 8 * 16); cudaMalloc(&gt, 8 * 4);
  const int M = 1 << 20;   // 4 MB ring, stride 4097 ints (16 KB hops)
  int* h = new int[M];
  for (int i = 0; i < M; ++i) h[i] = (int)((i + 4097ll * 33) % M);
  cudaMalloc(&nxt, 4 * M); cudaMalloc(&sink, 4);
  cudaMemcpy(nxt, h, 4 * M, cudaMemcpyHostToDevice);
  k_chain<<<1, 32>>>(out, cyc, 1.0000001, 1e-9);
  k_chain<<<1, 32>>>(out, cyc, 1.0000001, 1e-9);
  void* args[] = {&out, &cyc, &gt};
  cudaLaunchCooperativeKernel((void*)k_sync, 148, 768, args, 0, 0);
  k_chase<<<1, 1>>>(nxt, cyc, sink);
  k_chase<<<1, 1>>>(nxt, cyc, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long hc[8]; unsigned long long hg;
  cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
  cudaMemcpy(&hg, gt, 8, cudaMemcpyDeviceToHost);
  printf("err=%s\n", cudaGetErrorString(e));
  printf("DFMA dep chain: %.1f cyc/op\n", hc[0] / 2048.0);
  printf("DADD dep chain: %.1f cyc/op\n", hc[1] / 2048.0);
  printf("SHFL.f64+DADD chain: %.1f cyc/step\n", hc[2] / 2048.0);
  printf("__syncthreads (768 thr): %.1f cyc\n", hc[3] / 1000.0);
  printf("store+__threadfence+__syncthreads: %.1f cyc\n", hc[4] / 100.0);
  printf("grid.sync (148x768): %.1f cyc, %.1f ns\n", hc[5] / 103.0, hg / 100.0);
  printf("L2-hit pointer chase (ld.cg): %.1f cyc/hop\n", hc[6] / 256.0);
  return 0;
}
