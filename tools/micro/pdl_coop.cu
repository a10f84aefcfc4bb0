// Does the next launch's prologue overlap the previous launch's tail under PDL?
// mode 1: cooperative + cg grid.sync; mode 2: cooperative + PDL; mode 3: plain + PDL with a
// hand-written grid barrier (slot per launch parity).
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__device__ void gbar(unsigned* bar, unsigned nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned cur;
    do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory"); } while (cur < nb);
  }
  __syncthreads();
}
__global__ void k_work(double* out, int spin, int mode, unsigned* bars, int k) {
  extern __shared__ double s[];
  double acc = 0;
  for (int i = 0; i < spin; ++i) acc = fma(acc, 1.0000001, 0.5);   // prologue
  if (mode >= 2) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (mode == 3) {
    if (blockIdx.x == 0 && threadIdx.x == 0) bars[(k + 1) % 3] = 0;   // reset the slot of launch k+1
    gbar(bars + k % 3, gridDim.x);
  } else {
    cg::this_grid().sync();
  }
  for (int i = 0; i < spin; ++i) acc = fma(acc, 1.0000001, 0.25);
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
  if (mode >= 2) asm volatile("griddepcontrol.launch_dependents;");
}
int main() {
  double* out; cudaMalloc(&out, 8 * 4096);
  unsigned* bars; cudaMalloc(&bars, 64); cudaMemset(bars, 0, 64);
  cudaFuncSetAttribute(k_work, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
  cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int spin : {0, 2000, 8000})
  for (int mode = 1; mode <= 3; ++mode) {
    const int K = 200;
    int kk = 0;
    auto launch = [&]() {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(148); cfg.blockDim = dim3(768); cfg.dynamicSmemBytes = 200 << 10; cfg.stream = s;
      cudaLaunchAttribute at[2]; int na = 0;
      if (mode <= 2) { at[na].id = cudaLaunchAttributeCooperative; at[na].val.cooperative = 1; ++na; }
      if (mode >= 2) { at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[na].val.programmaticStreamSerializationAllowed = 1; ++na; }
      cfg.attrs = at; cfg.numAttrs = na;
      int k = kk++;
      return cudaLaunchKernelEx(&cfg, k_work, out, spin, mode, bars, k);
    };
    cudaMemset(bars, 0, 64); kk = 0;
    for (int k = 0; k < 5; ++k) launch();
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    for (int k = 0; k < K; ++k) launch();
    cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("spin %5d mode %d: %.2f us/launch (%s)\n", spin, mode, ms * 1e3 / K, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
