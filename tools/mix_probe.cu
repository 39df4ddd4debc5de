// SpMV-like gather + stream probe (tools/, not part of libpdcs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/mp tools/mix_probe.cu
// Each thread streams (int32 col, fp64 val) pairs and gathers x[col] with x
// spread over F MB -- the inner loop of a column panel pass.  Variants:
//   plain   : default cache policy everywhere
//   hint    : streams L2::evict_first, gathers L2::evict_last (createpolicy)
//   noalloc : streams ld.global.nc.L1::no_allocate + L2 evict_first
//   persist : plain loads, x inside a persisting access-policy window
// Reports ms, effective G gathers/s and DRAM-equivalent GB/s of the stream.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int ld_i_hint(const int* p, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_d_hint(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int ld_i_na(const int* p, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_d_na(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(256) spmv_like(const int* __restrict__ ci, const double* __restrict__ va,
                                                 const double* __restrict__ x, uint64_t rows,
                                                 double* __restrict__ y) {
  const uint64_t pf = pol_first(), pl = pol_last();
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const uint64_t j = 5 * r + k;
      int c;
      double a, xv;
      if (MODE == 0 || MODE == 3) {
        c = __ldg(ci + j); a = __ldg(va + j); xv = __ldg(x + c);
      } else if (MODE == 1) {
        c = ld_i_hint(ci + j, pf); a = ld_d_hint(va + j, pf); xv = ld_d_hint(x + c, pl);
      } else {
        c = ld_i_na(ci + j, pf); a = ld_d_na(va + j, pf); xv = ld_d_hint(x + c, pl);
      }
      s += a * xv;
    }
    y[r] = s;
  }
}

// coalesced form: a CTA loads a tile's (col, val) with consecutive lanes on
// consecutive entries, parks the products in shared memory, then one thread
// per row adds its row's products in order.
__global__ void __launch_bounds__(256) spmv_tile(const int* __restrict__ ci, const double* __restrict__ va,
                                                 const double* __restrict__ x, uint64_t rows,
                                                 double* __restrict__ y) {
  __shared__ double prod[256 * 5];
  const uint64_t ntiles = rows / 256;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t base = t * 256 * 5;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const int e = threadIdx.x + 256 * k;
      prod[e] = __ldg(va + base + e) * __ldg(x + __ldg(ci + base + e));
    }
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 5; ++k) s += prod[threadIdx.x * 5 + k];
    y[t * 256 + threadIdx.x] = s;
    __syncthreads();
  }
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t rows = 10ull << 20, nnz = 5 * rows;  // C5-like: 52M entries, 10M rows
  const uint64_t maxv = (160ull << 20) / 8;
  int* ci;
  double *va, *x, *y;
  cudaMalloc(&ci, nnz * 4);
  cudaMalloc(&va, nnz * 8);
  cudaMalloc(&x, maxv * 8);
  cudaMalloc(&y, rows * 8);
  cudaMemset(va, 0, nnz * 8);
  cudaMemset(x, 0, maxv * 8);
  std::vector<int> h(nnz);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int maxwin = 0, maxpersist = 0;
  cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, 0);
  cudaDeviceGetAttribute(&maxpersist, cudaDevAttrMaxPersistingL2CacheSize, 0);
  printf("max window %.1f MB, max persisting %.1f MB\n", maxwin / 1048576.0, maxpersist / 1048576.0);
  const int grid = nsm * 8;
  auto timeit = [&](auto launch) {
    launch();
    cudaEventRecord(e0, st);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5.0;
  };
  const double stream_gb = (nnz * 12.0 + rows * 8.0) / 1e9;
  printf("stream bytes per launch %.3f GB\n", stream_gb);
  const int mbs[] = {1, 10, 20, 30, 40, 50, 60, 80, 120, 160};
  const char* names[] = {"plain", "hint", "noalloc", "persist"};
  printf("%5s %9s %9s %9s %9s %9s %9s  (ms per launch)\n", "MB", names[0], names[1], names[2],
         names[3], "tile", "tile4/SM");
  uint64_t s = 88172645463325252ull;
  for (int mb : mbs) {
    const uint64_t span = (uint64_t)mb << 17;
    for (uint64_t i = 0; i < nnz; ++i) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      h[i] = (int)(s % span);
    }
    cudaMemcpy(ci, h.data(), nnz * 4, cudaMemcpyHostToDevice);
    double t[6];
    t[4] = timeit([&] { spmv_tile<<<grid, 256, 0, st>>>(ci, va, x, rows, y); });
    t[5] = timeit([&] { spmv_tile<<<nsm * 4, 256, 0, st>>>(ci, va, x, rows, y); });
    t[0] = timeit([&] { spmv_like<0><<<grid, 256, 0, st>>>(ci, va, x, rows, y); });
    t[1] = timeit([&] { spmv_like<1><<<grid, 256, 0, st>>>(ci, va, x, rows, y); });
    t[2] = timeit([&] { spmv_like<2><<<grid, 256, 0, st>>>(ci, va, x, rows, y); });
    {
      const size_t win = std::min<size_t>(span * 8, (size_t)maxwin);
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min<size_t>(win, (size_t)maxpersist));
      cudaStreamAttrValue a = {};
      a.accessPolicyWindow.base_ptr = x;
      a.accessPolicyWindow.num_bytes = win;
      a.accessPolicyWindow.hitRatio = 1.0f;
      a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a);
      t[3] = timeit([&] { spmv_like<3><<<grid, 256, 0, st>>>(ci, va, x, rows, y); });
      a.accessPolicyWindow.num_bytes = 0;
      cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a);
      cudaCtxResetPersistingL2Cache();
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
    }
    printf("%5d %9.3f %9.3f %9.3f %9.3f %9.3f %9.3f\n", mb, t[0], t[1], t[2], t[3], t[4], t[5]);
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
