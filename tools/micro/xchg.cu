// Microbenchmark: cost of one grid-wide exchange of per-CTA records (148 CTAs x 768 thr,
// cooperative launch), 100 rounds, ns per round (globaltimer):
//   0: cg grid.sync + __ldcg of all records
//   1: per-slot flags, ld.acquire.gpu polling (one lane per slot)
//   2: per-slot flags, ld.relaxed.gpu polling + fence.acq_rel.gpu, then __ldcg data
//   3: counter barrier: red.release.gpu.add + relaxed polling by thread 0 + fence, then loads
//   4: per-slot flags, ld.acquire.gpu polling with __nanosleep(32)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a xchg.cu -o xchg
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdio>
namespace cg = cooperative_groups;

struct __align__(128) Rec { double v[14]; unsigned long long flag, pad; };

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
  unsigned long long v; asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ unsigned long long ld_rlx(const unsigned long long* p) {
  unsigned long long v; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void st_rel(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
template <int MODE, int WORK>
__global__ void __launch_bounds__(768, 1) k(Rec* rec, unsigned long long* ctr, double* out, unsigned long long* ns, int rounds) {
  __shared__ double acc[8];
  const int b = blockIdx.x, G = gridDim.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double s = 0;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  for (int r = 1; r <= rounds; ++r) {
    if (threadIdx.x == 0) {
      for (int q = 0; q < 14; ++q) rec[(r & 1) * G + b].v[q] = r + b + q;
      if (MODE == 0) __threadfence();
      if (MODE == 1 || MODE == 2 || MODE == 4) st_rel(&rec[(r & 1) * G + b].flag, (unsigned long long)((r + 1) >> 1));
      if (MODE == 3 && !WORK) asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
    }
    if (MODE == 0) cg::this_grid().sync();
    if ((MODE >= 5 || (MODE == 3 && WORK)) && threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
    if (WORK) {   // split barrier: independent FP64 work between arrive and wait
      double w = threadIdx.x;
      for (int i = 0; i < WORK; ++i) w = fma(w, 1.0000001, 1e-9);
      s += w * 1e-30;
    }
    if (MODE == 3 || MODE == 5 || MODE == 6) {
      if (threadIdx.x == 0) {
        if (MODE == 3) { while (ld_rlx(ctr) < (unsigned long long)r * G) {} asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
        if (MODE == 5) { while (ld_rlx(ctr) < (unsigned long long)r * G) __nanosleep(64); asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
        if (MODE == 6) { while (ld_acq(ctr) < (unsigned long long)r * G) {} }
      }
      __syncthreads();
    }
    const int j = warp * 32 + lane;
    if (warp < 5 && j < G) {
      const Rec* o = rec + (r & 1) * G + j;
      const unsigned long long tg = (unsigned long long)((r + 1) >> 1);
      if (MODE == 1) while (ld_acq(&o->flag) < tg) {}
      if (MODE == 4) while (ld_acq(&o->flag) < tg) __nanosleep(32);
      if (MODE == 2) { while (ld_rlx(&o->flag) < tg) {} asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
      for (int q = 0; q < 5; ++q) s += __ldcg(&o->v[q]);
    }
    __syncthreads();
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) ns[b] = t1 - t0;
  if (s == 1.2345) out[0] = s;
}
template <int MODE, int WORK>
void run(Rec* rec, unsigned long long* ctr, double* out, unsigned long long* ns) {
  int rounds = 100;
  cudaMemset(rec, 0, sizeof(Rec) * 2 * 148);
  cudaMemset(ctr, 0, 8);
  void* args[] = {&rec, &ctr, &out, &ns, &rounds};
  cudaLaunchCooperativeKernel((void*)k<MODE, WORK>, 148, 768, args, 0, 0);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, ns, sizeof(h), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("mode %d work %4d: %8.1f ns/round (%s)\n", MODE, WORK, mx / 100.0, cudaGetErrorString(e));
}
int main() {
  Rec* rec; unsigned long long *ctr, *ns; double* out;
  cudaMalloc(&rec, sizeof(Rec) * 2 * 148); cudaMalloc(&ctr, 8); cudaMalloc(&ns, 8 * 148); cudaMalloc(&out, 8);
  for (int rep = 0; rep < 2; ++rep) {
    run<0, 0>(rec, ctr, out, ns); run<3, 0>(rec, ctr, out, ns); run<5, 0>(rec, ctr, out, ns); run<6, 0>(rec, ctr, out, ns);
    run<0, 256>(rec, ctr, out, ns); run<3, 256>(rec, ctr, out, ns); run<5, 256>(rec, ctr, out, ns); run<6, 256>(rec, ctr, out, ns);
  }
  return 0;
}
