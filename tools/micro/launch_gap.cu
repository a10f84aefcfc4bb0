// Per-launch cost of back-to-back kernels in a CUDA graph vs dynamic smem size and
// cooperative attribute (148 CTAs x 768 threads, grid.sync or not).
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void k_empty(int* p) { extern __shared__ char s[]; if (threadIdx.x == 0 && p) s[0] = 1; }
__global__ void k_sync(int* p) { extern __shared__ char s[]; cg::this_grid().sync(); if (threadIdx.x == 0 && p) s[0] = 1; }
int main() {
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(k_sync, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int coop = 0; coop < 2; ++coop)
    for (int sync = 0; sync < 2; ++sync) {
      if (sync && !coop) continue;
      for (size_t smem : {0ul, 64ul << 10, 200ul << 10}) {
        const int K = 200;
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        for (int k = 0; k < K; ++k) {
          int* p = nullptr; void* args[] = {&p};
          void* fn = sync ? (void*)k_sync : (void*)k_empty;
          if (coop) cudaLaunchCooperativeKernel(fn, dim3(148), dim3(768), args, smem, st);
          else cudaLaunchKernel(fn, dim3(148), dim3(768), args, smem, st);
        }
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
        cudaEventRecord(e0, st); cudaGraphLaunch(ge, st); cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        // plain stream loop too
        cudaEventRecord(e0, st);
        for (int k = 0; k < K; ++k) {
          int* p = nullptr; void* args[] = {&p};
          void* fn = sync ? (void*)k_sync : (void*)k_empty;
          if (coop) cudaLaunchCooperativeKernel(fn, dim3(148), dim3(768), args, smem, st);
          else cudaLaunchKernel(fn, dim3(148), dim3(768), args, smem, st);
        }
        cudaEventRecord(e1, st); cudaEventSynchronize(e1);
        float ms2; cudaEventElapsedTime(&ms2, e0, e1);
        printf("coop=%d sync=%d smem=%6zu KB: graph %.2f us/launch, stream %.2f us/launch (%s)\n", coop, sync,
               smem >> 10, ms * 1e3 / K, ms2 * 1e3 / K, cudaGetErrorString(cudaGetLastError()));
        cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
      }
    }
  return 0;
}
