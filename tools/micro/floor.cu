// Floor of the d = 1 rank-order apply's launch structure on B200: one CTA per SM
// (148 x 768 threads, ~193 KB dynamic smem), bulk-copy t (8 MB plan array) and v (8 MB,
// one of 100 rotating vectors) into smem, optionally one grid.sync, write 8 MB out
// coalesced; 100 launches captured in a CUDA graph.  Variants: cooperative attribute,
// PDL attribute, grid sync on/off, 0 / 1 / 2 barriers of a cheap counter.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a floor.cu -o floor
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(768, 1) k(const double* __restrict__ t, const double* __restrict__ v,
                                            double* __restrict__ out, int n, int chunk, int mode) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t mb[2];
  double* st = reinterpret_cast<double*>(sm);
  double* su = st + chunk + 8;
  const int c0 = blockIdx.x * chunk, cnt = max(0, min(chunk, n - c0));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mb[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mb[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const unsigned bytes = ((cnt + 1) & ~1) * 8;
  if (threadIdx.x == 0 && cnt > 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mb[0])), "r"(bytes));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(st)),
                 "l"(t + c0), "r"(bytes), "r"(su32(&mb[0])) : "memory");
  }
  if (mode & 4) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && cnt > 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mb[1])), "r"(bytes));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(su)),
                 "l"(v + c0), "r"(bytes), "r"(su32(&mb[1])) : "memory");
  }
  for (int i = 0; i < 2; ++i) {
    unsigned ok = 0;
    while (cnt > 0 && !ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok) : "r"(su32(&mb[i])));
  }
  if (mode & 1) cg::this_grid().sync();
  for (int j = threadIdx.x; j < cnt; j += blockDim.x) out[c0 + j] = st[j] * su[j];
  if (mode & 4) asm volatile("griddepcontrol.launch_dependents;");
}

int main() {
  const int n = 1000000, NV = 100, grid = 148, chunk = ((n + grid - 1) / grid + 3) & ~3;
  double *t, *v, *o;
  cudaMalloc(&t, 8ull * (n + 64)); cudaMalloc(&v, 8ull * n * NV + 64); cudaMalloc(&o, 8ull * n * NV);
  cudaMemset(t, 0, 8ull * n); cudaMemset(v, 0, 8ull * n * NV);
  const size_t smem = 193 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  // mode bits: 1 grid.sync, 2 cooperative attribute, 4 PDL attribute (+ griddepcontrol)
  for (int mode : {0, 2, 3, 4, 6, 7}) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int r = 0; r < NV; ++r) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid); cfg.blockDim = dim3(768); cfg.dynamicSmemBytes = smem; cfg.stream = s;
      cudaLaunchAttribute at[2]; int na = 0;
      if (mode & 2) { at[na].id = cudaLaunchAttributeCooperative; at[na].val.cooperative = 1; ++na; }
      if (mode & 4) { at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[na].val.programmaticStreamSerializationAllowed = 1; ++na; }
      cfg.attrs = at; cfg.numAttrs = na;
      const double* vr = v + (size_t)r * n; double* orr = o + (size_t)r * n; int nn = n, ch = chunk, md = mode;
      cudaLaunchKernelEx(&cfg, k, (const double*)t, vr, orr, nn, ch, md);
    }
    cudaStreamEndCapture(s, &g);
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("mode %d: instantiate failed\n", mode); continue; }
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0, s); cudaGraphLaunch(ge, s); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
    }
    printf("mode %d (sync=%d coop=%d pdl=%d): %.2f us/launch (%s)\n", mode, mode & 1, (mode >> 1) & 1, (mode >> 2) & 1,
           best * 1e3 / NV, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
