// Microbenchmark: cost of executing K straight-line FP64 instructions ONCE per launch
// (cold instruction fetch) vs the same block executed a second time (warm), 148 CTAs x 768.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a icache.cu -o icache
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
template <int K>
__global__ void __launch_bounds__(768, 1) k(double* out, unsigned long long* st, int reps) {
  double a = threadIdx.x, d = 2.0; unsigned i0 = threadIdx.x, i1 = 1, i2 = 2, i3 = 3, i4 = 4, i5 = 5, i6 = 6, i7 = 7, c = reps;
  unsigned long long t0 = gt(), t1 = 0;
#pragma unroll 1
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < K; ++i) {
      asm volatile("add.u32 %0, %0, %1;" : "+r"(i0) : "r"(c));
      asm volatile("add.u32 %0, %0, %1;" : "+r"(i1) : "r"(c));
      asm volatile("add.u32 %0, %0, %1;" : "+r"(i2) : "r"(c));
      asm volatile("add.u32 %0, %0, %1;" : "+r"(i3) : "r"(c));
      asm volatile("add.u32 %0, %0, %1;" : "+r"(i4) : "r"(c));
      asm volatile("add.u32 %0, %0, %1;" : "+r"(i5) : "r"(c));
      asm volatile("add.u32 %0, %0, %1;" : "+r"(i6) : "r"(c));
      asm volatile("add.u32 %0, %0, %1;" : "+r"(i7) : "r"(c));
      c ^= i;
    }
    if (r == 0) t1 = gt();
  }
  __syncthreads();
  unsigned long long t2 = gt();
  if (threadIdx.x == 0) { st[blockIdx.x * 3] = t0; st[blockIdx.x * 3 + 1] = t1; st[blockIdx.x * 3 + 2] = t2; }
  if (i0 + i1 + i2 + i3 + i4 + i5 + i6 + i7 == 12345u) out[threadIdx.x] = a + d;
}
int NT = 768;
template <int K>
void run(double* out, unsigned long long* st, int reps) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 5; ++i) k<K><<<148, NT>>>(out, st, reps);
  cudaEventRecord(e0);
  const int R = 100;
  for (int i = 0; i < R; ++i) k<K><<<148, NT>>>(out, st, reps);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148 * 3];
  cudaMemcpy(h, st, sizeof(h), cudaMemcpyDeviceToHost);
  double first = 0, total = 0;
  for (int b = 0; b < 148; ++b) { first += h[b * 3 + 1] - h[b * 3]; total += h[b * 3 + 2] - h[b * 3]; }
  printf("K=%5d (x8 IADD) reps=%d: %7.2f us/launch, in-kernel first pass %7.2f us, total %7.2f us\n", K, reps,
         ms * 1e3 / R, first / 148 / 1e3, total / 148 / 1e3);
}
int main() {
  double* out; unsigned long long* st;
  cudaMalloc(&out, 8 * 1024); cudaMalloc(&st, 8 * 148 * 3);
  for (int nt : {32, 768}) for (int reps : {1, 2}) { NT = nt; printf("threads %d\n", nt);
    run<16>(out, st, reps); run<128>(out, st, reps); run<512>(out, st, reps); run<2048>(out, st, reps);
  }
  return 0;
}
