// Microbenchmark: random 8-byte gathers of 1e6 doubles, one chunk of ranks per CTA
// (the d = 1 user-order access pattern), by
//   0: LDG (one lane per element, L1TEX wavefront per line),
//   1: TMA tile::gather4 (2-D tensor map over v viewed as [N/2][2] doubles, 4 rows/instr),
//   2: cp.async.bulk 16 B per element (non-tensor bulk copy).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tma_gather.cu -o tma_gather -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

__device__ __forceinline__ unsigned su32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

template <int MODE>
__global__ void __launch_bounds__(256, 1)
    k(const CUtensorMap* __restrict__ tm, const int* __restrict__ perm, const double* __restrict__ v,
      double* __restrict__ out, int n, int chunk) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t mbar;
  int* s_p = reinterpret_cast<int*>(sm);
  double* s_v = reinterpret_cast<double*>(sm + ((chunk * 4 + 127) / 128) * 128);
  const int c0 = blockIdx.x * chunk;
  const int cnt = max(0, min(chunk, n - c0));
  for (int j = threadIdx.x; j < cnt; j += blockDim.x) s_p[j] = perm[c0 + j];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (MODE == 0) {
    for (int j = threadIdx.x; j < cnt; j += blockDim.x) out[c0 + j] = __ldg(v + s_p[j]);
    return;
  }
  if (MODE == 3) {   // split: TMA gather4 for [0, h) issued by warp 0, LDG for [h, cnt)
    const int h = (cnt / 2) & ~3;
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mbar)),
                   "r"((unsigned)(h / 4) * 64u));
    if (threadIdx.x < 32) {
      for (int g = threadIdx.x; g * 4 < h; g += 32) {
        int r[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) r[q] = s_p[g * 4 + q] >> 1;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(su32(s_v + g * 16)),
            "l"(tm), "r"(su32(&mbar)), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3])
            : "memory");
      }
    } else {
      for (int j = h + threadIdx.x - 32; j < cnt; j += blockDim.x - 32) out[c0 + j] = __ldg(v + s_p[j]);
    }
    unsigned ok = 0;
    while (!ok)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
          : "=r"(ok)
          : "r"(su32(&mbar)));
    for (int j = threadIdx.x; j < h; j += blockDim.x)
      out[c0 + j] = s_v[(j >> 2) * 16 + (j & 3) * 2 + (s_p[j] & 1)];
    return;
  }
  const unsigned bytes = MODE == 1 ? ((cnt + 3) / 4) * 64u : cnt * 16u;
  if (threadIdx.x == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mbar)),
                 "r"(bytes));
  __syncthreads();
  if (MODE == 1) {
    for (int g = threadIdx.x; g * 4 < cnt; g += blockDim.x) {
      int r[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) r[q] = (g * 4 + q < cnt ? s_p[g * 4 + q] : 0) >> 1;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(su32(s_v + g * 16)),
          "l"(tm), "r"(su32(&mbar)), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3])
          : "memory");
    }
  } else {
    for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
      const double* src = v + (s_p[j] & ~1);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::
              "r"(su32(s_v + 2 * j)),
          "l"(src), "r"(su32(&mbar))
          : "memory");
    }
  }
  unsigned ok = 0;
  while (!ok)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(su32(&mbar)));
  for (int j = threadIdx.x; j < cnt; j += blockDim.x)
    out[c0 + j] = MODE == 1 ? s_v[(j >> 2) * 16 + (j & 3) * 2 + (s_p[j] & 1)] : s_v[2 * j + (s_p[j] & 1)];
}

int main() {
  const int n = 1000000, NV = 64;
  std::vector<int> perm(n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  std::mt19937 rng(1);
  std::shuffle(perm.begin(), perm.end(), rng);
  int* dp;
  double *dv, *dout;
  cudaMalloc(&dp, 4 * n);
  cudaMalloc(&dv, 8ull * n * NV + 64);
  cudaMalloc(&dout, 8ull * n * NV);
  cudaMemcpy(dp, perm.data(), 4 * n, cudaMemcpyHostToDevice);
  std::vector<double> hv(n);
  for (int i = 0; i < n; ++i) hv[i] = i;
  for (int r = 0; r < NV; ++r) cudaMemcpy(dv + (size_t)r * n, hv.data(), 8 * n, cudaMemcpyHostToDevice);

  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                               const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                               const cuuint32_t*, CUtensorMapInterleave,
                                               CUtensorMapSwizzle, CUtensorMapL2promotion,
                                               CUtensorMapFloatOOBfill)>(fn);
  std::vector<CUtensorMap> hm(NV);
  for (int r = 0; r < NV; ++r) {
    cuuint64_t dims[2] = {2, (cuuint64_t)(n / 2)};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {2, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult e = encode(&hm[r], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dv + (size_t)r * n, dims, strides,
                        box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (e != CUDA_SUCCESS) { printf("encode failed %d\n", (int)e); return 1; }
  }
  CUtensorMap* dm;
  cudaMalloc(&dm, sizeof(CUtensorMap) * NV);
  cudaMemcpy(dm, hm.data(), sizeof(CUtensorMap) * NV, cudaMemcpyHostToDevice);

  const int grid = 148, chunk = (n + grid - 1) / grid;
  const size_t smem = ((chunk * 4 + 127) / 128) * 128 + ((chunk / 2 + 3) / 4) * 128 + 256;
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"LDG gather", "TMA gather4", "bulk 16B", "split TMA+LDG"};
  for (int mode : {0, 3}) {
    auto run = [&](int r) {
      const double* v = dv + (size_t)(r % NV) * n;
      double* o = dout + (size_t)(r % NV) * n;
      if (mode == 0) k<0><<<grid, 256, smem>>>(dm + r % NV, dp, v, o, n, chunk);
      if (mode == 1) k<1><<<grid, 256, smem>>>(dm + r % NV, dp, v, o, n, chunk);
      if (mode == 2) k<2><<<grid, 256, smem>>>(dm + r % NV, dp, v, o, n, chunk);
      if (mode == 3) k<3><<<grid, 256, smem>>>(dm + r % NV, dp, v, o, n, chunk);
    };
    for (int r = 0; r < 10; ++r) run(r);
    if (cudaGetLastError() != cudaSuccess) { printf("launch error\n"); }
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) { printf("%s: %s\n", names[mode], cudaGetErrorString(err)); return 1; }
    std::vector<double> ho(n);
    cudaMemcpy(ho.data(), dout + (size_t)9 * n, 8 * n, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < n; ++i) bad += ho[i] != (double)perm[i];
    cudaEventRecord(e0);
    const int R = 200;
    for (int r = 0; r < R; ++r) run(r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-12s %7.2f us/launch  (mismatches %d)\n", names[mode], ms * 1e3 / R, bad);
  }
  return 0;
}
