// setup.cu -- the stored-sort data structure of the paper (P:191 [§1]; P:338 [§2.1];
// P:531-539 [§2.2.3]) built on the device:
//   a1  scale t_k = sqrt(2 nu) x_k / l_k (P:294 [eq scaled_kernel]), reject NaN/Inf;
//   a2  stable radix sort of (t_1, index) -> perm, and t_k gathered into x1-rank order;
//   a3  d >= 2: level orders of Bentley's divide and conquer over x1-ranks:
//       ord2[l] = for each aligned rank block [b 2^l, (b+1) 2^l), its ranks in (t_2, rank)
//       order -- obtained as ONE stable radix sort of the global t_2 order by the key
//       (rank >> l);  d = 3: ord3[l1][l2] = positions q of ord2[l1] grouped by inner node
//       (q >> l2) and t_3-sorted inside, again by a stable sort of the global t_3 order.
// Ties: every order is a strict total order (value, then index/rank), R3.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cmath>

#include "internal.h"

namespace gpm {

namespace {

__device__ __forceinline__ unsigned long long orderable_key(double v) {
  v = v + 0.0;  // -0.0 -> +0.0
  long long b = __double_as_longlong(v);
  return b < 0 ? ~static_cast<unsigned long long>(b)
               : (static_cast<unsigned long long>(b) | 0x8000000000000000ull);
}

__global__ void k_check_key0(const double* __restrict__ x, int64_t n, int d, double s0,
                             unsigned long long* __restrict__ key, int* __restrict__ val,
                             unsigned long long* __restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    bool ok = true;
    for (int k = 0; k < d; ++k) ok &= isfinite(x[i * d + k]);
    if (!ok) atomicMin(bad, static_cast<unsigned long long>(i));
    // centred on the first point (the kernel depends on differences only; without
    // it a large common offset costs eps * offset / l in every scaled distance)
    key[i] = orderable_key(ok ? s0 * (x[i * d] - x[0]) : 0.0);
    val[i] = static_cast<int>(i);
  }
}

__global__ void k_gather_scaled(const double* __restrict__ x, const int* __restrict__ perm,
                                int64_t n, int d, double s0, double s1, double s2,
                                double* __restrict__ t) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = perm[r];
    const double sc[3] = {s0, s1, s2};
    for (int k = 0; k < d; ++k) t[k * n + r] = sc[k] * (x[i * d + k] - x[k]) + 0.0;   // centred on point 0
  }
}

__global__ void k_key_iota(const double* __restrict__ tk, int64_t n,
                           unsigned long long* __restrict__ key, int* __restrict__ val) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    key[r] = orderable_key(tk[r]);
    val[r] = static_cast<int>(r);
  }
}

__global__ void k_inverse(const int* __restrict__ ord, int64_t n, int* __restrict__ inv) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x)
    inv[ord[q]] = static_cast<int>(q);
}

__global__ void k_compose(const int* __restrict__ a, const int* __restrict__ seq, int64_t n,
                          int* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[seq[i]];
}

inline int grid_for(int64_t n) {
  return static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16));
}

}  // namespace

// allocator hook (gp_set_allocator); process-wide, captured per buffer at allocation
static gp_alloc_fn g_alloc = nullptr;
static gp_free_fn g_free = nullptr;
static void* g_actx = nullptr;

void set_allocator(gp_alloc_fn a, gp_free_fn f, void* ctx) {
  g_alloc = a;
  g_free = f;
  g_actx = ctx;
}

gp_status DevBuf::alloc(size_t b) {
  release();
  if (b == 0) b = 16;
  if (g_alloc) {
    ptr = g_alloc(b, nullptr, g_actx);
    if (!ptr) return fail(GP_ERR_OOM, "allocator hook returned NULL for " + std::to_string(b) + " bytes");
    fr = g_free;
    fctx = g_actx;
    bytes = b;
    return GP_OK;
  }
  cudaError_t e = cudaMalloc(&ptr, b);
  if (e != cudaSuccess) {
    ptr = nullptr;
    (void)cudaGetLastError();
    return fail(GP_ERR_OOM, std::string("cudaMalloc(") + std::to_string(b) + ") failed: " +
                                cudaGetErrorString(e));
  }
  bytes = b;
  return GP_OK;
}

void DevBuf::release() {
  if (ptr) {
    if (fr) {
      cudaDeviceSynchronize();   // the hook's pool may hand the block out at once
      fr(ptr, nullptr, fctx);
    } else {
      cudaFree(ptr);
    }
  }
  ptr = nullptr;
  bytes = 0;
  fr = nullptr;
  fctx = nullptr;
}

void plan_free(Plan& pl) {
  for (DevBuf* b : {&pl.x_raw, &pl.perm, &pl.t, &pl.ord2, &pl.ord3, &pl.u, &pl.acc, &pl.w,
                    &pl.aggs, &pl.bar, &pl.stage_in, &pl.stage_out, &pl.dbg, &pl.d1e, &pl.d1ends, &pl.cg_scratch, &pl.pts, &pl.hpbuf, &pl.hpdesc, &pl.part})
    b->release();
  if (pl.ev_fork) cudaEventDestroy(pl.ev_fork);
  if (pl.ev_join) cudaEventDestroy(pl.ev_join);
  if (pl.ev_join3) cudaEventDestroy(pl.ev_join3);
  if (pl.s2) cudaStreamDestroy(pl.s2);
  if (pl.s3) cudaStreamDestroy(pl.s3);
  pl.s3 = nullptr;
  pl.ev_join3 = nullptr;
  for (cudaEvent_t& e : pl.hev)
    if (e) { cudaEventDestroy(e); e = nullptr; }
  if (pl.hs_in) cudaStreamDestroy(pl.hs_in);
  if (pl.hs_out) cudaStreamDestroy(pl.hs_out);
  pl.hs_in = pl.hs_out = nullptr;
  pl.ev_fork = pl.ev_join = nullptr;
  pl.s2 = nullptr;
}

static gp_status sort_pairs_u64(void* tmp, size_t tmp_bytes, const unsigned long long* kin,
                                unsigned long long* kout, const int* vin, int* vout, int64_t n,
                                cudaStream_t s) {
  size_t tb = tmp_bytes;
  GPM_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, kin, kout, vin, vout, (int)n, 0, 64, s));
  return GP_OK;
}

gp_status plan_build(Plan& pl, const double* x, int64_t n, int d, const gp_kernel& k,
                     cudaStream_t s) {
  pl.n = n;
  pl.d = d;
  pl.kern = k;
  pl.two_nu = k.two_nu;
  pl.P = (k.two_nu - 1) / 2;
  pl.form = (d == 1 || k.two_nu == 1) ? GP_FORM_L1 : k.form;
  pl.os2 = k.outputscale * k.outputscale;
  for (int j = 0; j < 3; ++j) {
    pl.ell[j] = j < d ? k.lengthscale[j] : 1.0;
    pl.scale[j] = j < d ? std::sqrt((double)k.two_nu) / k.lengthscale[j] : 0.0;
  }
  int L = 0;
  while ((int64_t(1) << L) < n) ++L;
  pl.L = L;
  pl.n_src = n;
  pl.tgt_off = 0;

  GPM_TRY(pl.x_raw.alloc(sizeof(double) * n * d));
  GPM_CUDA(cudaMemcpyAsync(pl.x_raw.ptr, x, sizeof(double) * n * d, cudaMemcpyDeviceToDevice, s));
  GPM_TRY(pl.perm.alloc(sizeof(int) * (n + 16)));   // padded: TMA bulk copies round up
  // padding = 0x7f7f7f7f (> any user index): rounded-up bulk copies read no source index
  GPM_CUDA(cudaMemsetAsync(pl.perm.as<int>() + n, 0x7f, sizeof(int) * 16, s));
  GPM_TRY(pl.t.alloc(sizeof(double) * (n * d + 16)));

  // scratch for sorting
  DevBuf keys, keys2, vals, bad, tmp, seq, seq3, inv, qseq;
  auto cleanup = [&]() {
    keys.release(); keys2.release(); vals.release(); bad.release(); tmp.release();
    seq.release(); seq3.release(); inv.release(); qseq.release();
  };
  gp_status st = GP_OK;
  do {
    if ((st = keys.alloc(8 * n)) || (st = keys2.alloc(8 * n)) || (st = vals.alloc(4 * n)) ||
        (st = bad.alloc(8)))
      break;
    size_t tb1 = 0, tb2 = 0;
    cudaError_t e1 = cub::DeviceRadixSort::SortPairs(
        nullptr, tb1, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
        (int*)nullptr, (int*)nullptr, (int)n, 0, 64, s);
    cudaError_t e2 = cub::DeviceRadixSort::SortKeys(nullptr, tb2, (unsigned*)nullptr,
                                                    (unsigned*)nullptr, (int)n, 0, 32, s);
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
      st = fail(GP_ERR_CUDA, "cub temp-size query failed");
      break;
    }
    const size_t tb = std::max(tb1, tb2);
    if ((st = tmp.alloc(tb))) break;

    // a1 + key of dim 0
    unsigned long long init = ~0ull;
    if (cudaMemcpyAsync(bad.ptr, &init, 8, cudaMemcpyHostToDevice, s) != cudaSuccess) {
      st = fail(GP_ERR_CUDA, "memcpy failed");
      break;
    }
    k_check_key0<<<grid_for(n), 256, 0, s>>>(x, n, d, pl.scale[0], keys.as<unsigned long long>(),
                                             vals.as<int>(), bad.as<unsigned long long>());
    unsigned long long badrow = 0;
    if (cudaMemcpyAsync(&badrow, bad.ptr, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
      st = fail(GP_ERR_CUDA, std::string("setup validation failed: ") +
                                 cudaGetErrorString(cudaGetLastError()));
      break;
    }
    if (badrow != ~0ull) {
      st = fail(GP_ERR_NONFINITE, "non-finite coordinate in row " + std::to_string(badrow));
      break;
    }
    // a2: stable sort by t1 (CUB radix sort is stable; values start in index order)
    if ((st = sort_pairs_u64(tmp.ptr, tb, keys.as<unsigned long long>(),
                             keys2.as<unsigned long long>(), vals.as<int>(), pl.perm.as<int>(), n,
                             s)))
      break;
    k_gather_scaled<<<grid_for(n), 256, 0, s>>>(x, pl.perm.as<int>(), n, d, pl.scale[0],
                                                pl.scale[1], pl.scale[2], pl.t.as<double>());
    if (d >= 2 && L >= 1) {
      // a3: global (t2, rank) order of the ranks
      if ((st = seq.alloc(4 * n))) break;
      k_key_iota<<<grid_for(n), 256, 0, s>>>(pl.t.as<double>() + n, n,
                                             keys.as<unsigned long long>(), vals.as<int>());
      if ((st = sort_pairs_u64(tmp.ptr, tb, keys.as<unsigned long long>(),
                               keys2.as<unsigned long long>(), vals.as<int>(), seq.as<int>(), n,
                               s)))
        break;
      if ((st = pl.ord2.alloc(sizeof(int) * n * L))) break;
      for (int l = 1; l <= L; ++l) {
        unsigned* dst = pl.ord2.as<unsigned>() + (size_t)(l - 1) * n;
        if (l == L) {
          GPM_CUDA(cudaMemcpyAsync(dst, seq.ptr, 4 * n, cudaMemcpyDeviceToDevice, s));
        } else {
          size_t tbb = tb;
          GPM_CUDA(cub::DeviceRadixSort::SortKeys(tmp.ptr, tbb, seq.as<unsigned>(), dst, (int)n,
                                                  l, L, s));
        }
      }
      if (d == 3) {
        if ((st = seq3.alloc(4 * n)) || (st = inv.alloc(4 * n)) || (st = qseq.alloc(4 * n)))
          break;
        k_key_iota<<<grid_for(n), 256, 0, s>>>(pl.t.as<double>() + 2 * n, n,
                                               keys.as<unsigned long long>(), vals.as<int>());
        if ((st = sort_pairs_u64(tmp.ptr, tb, keys.as<unsigned long long>(),
                                 keys2.as<unsigned long long>(), vals.as<int>(), seq3.as<int>(),
                                 n, s)))
          break;
        const size_t npairs = (size_t)L * (L + 1) / 2;
        if ((st = pl.ord3.alloc(sizeof(int) * n * npairs))) break;
        for (int l1 = 1; l1 <= L && st == GP_OK; ++l1) {
          k_inverse<<<grid_for(n), 256, 0, s>>>(pl.ord2.as<int>() + (size_t)(l1 - 1) * n, n,
                                                inv.as<int>());
          k_compose<<<grid_for(n), 256, 0, s>>>(inv.as<int>(), seq3.as<int>(), n, qseq.as<int>());
          for (int l2 = 1; l2 <= l1; ++l2) {
            unsigned* dst =
                pl.ord3.as<unsigned>() + ((size_t)(l1 - 1) * l1 / 2 + (l2 - 1)) * n;
            if (l2 == L) {
              GPM_CUDA(cudaMemcpyAsync(dst, qseq.ptr, 4 * n, cudaMemcpyDeviceToDevice, s));
            } else {
              size_t tbb = tb;
              GPM_CUDA(cub::DeviceRadixSort::SortKeys(tmp.ptr, tbb, qseq.as<unsigned>(), dst,
                                                      (int)n, l2, L, s));
            }
          }
        }
        if (st) break;
      }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      st = fail(GP_ERR_CUDA, std::string("setup kernels: ") + cudaGetErrorString(e));
      break;
    }
  } while (0);
  cudaStreamSynchronize(s);
  cleanup();
  if (st != GP_OK) return st;
  pl.struct_bytes = (int64_t)(pl.perm.bytes + pl.t.bytes + pl.ord2.bytes + pl.ord3.bytes);
  return apply_prepare(pl);
}

}  // namespace gpm
