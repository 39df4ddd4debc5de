// Gather-rate probe with precomputed indices (tools/, not part of libpdcs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gather_probe tools/gather_probe.cu
// Streams a 64M-entry int32 index array (coalesced) and gathers v[idx] (FP64)
// over a footprint of F MB, the access pattern of a random-column SpMV.  Unlike
// tools/l2_probe.cu no index arithmetic sits in the loop, so the rate is the
// memory system's.  Also reports the index stream alone (no gather) and a
// 5-entries-per-thread form matching the thread-per-row step kernel.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__global__ void stream_only(const int* __restrict__ idx, uint64_t n, double* out) {
  double acc = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    acc += (double)__ldg(idx + i);
  if (acc == 12345.678) out[0] = acc;
}

__global__ void gather_flat(const int* __restrict__ idx, const double* __restrict__ v, uint64_t n,
                            double* out) {
  double acc = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    acc += __ldg(v + __ldg(idx + i));
  if (acc == 12345.678) out[0] = acc;
}

// thread per "row" of 5 consecutive indices
__global__ void gather_rows5(const int* __restrict__ idx, const double* __restrict__ v, uint64_t rows,
                             double* out) {
  double acc = 0.0;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows; r += (uint64_t)gridDim.x * blockDim.x) {
    const int* p = idx + 5 * r;
    const int c0 = __ldg(p), c1 = __ldg(p + 1), c2 = __ldg(p + 2), c3 = __ldg(p + 3), c4 = __ldg(p + 4);
    acc += __ldg(v + c0) + __ldg(v + c1) + __ldg(v + c2) + __ldg(v + c3) + __ldg(v + c4);
  }
  if (acc == 12345.678) out[0] = acc;
}

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// indices drawn over [0, span/2); an SM-dependent function picks the half.
// If one function matches the die split and each die's L2 caches its own
// half, the rate at 2x the single-die capacity jumps.
__global__ void gather_split(const int* __restrict__ idx, const double* __restrict__ v, uint64_t n,
                             uint64_t half, int fn, int nsm, double* out) {
  const unsigned s = smid();
  unsigned side;
  switch (fn) {
    case 0: side = s < (unsigned)nsm / 2; break;
    default: side = (s >> (fn - 1)) & 1; break;
  }
  const double* base = v + (side ? half : 0);
  double acc = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    acc += __ldg(base + __ldg(idx + i));
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t nidx = 50ull << 20;  // 52M gathers (C5: 50M)
  const uint64_t maxv = (256ull << 20) / 8;
  int* idx;
  double *v, *out;
  cudaMalloc(&idx, nidx * 4);
  cudaMalloc(&v, maxv * 8);
  cudaMalloc(&out, 8);
  cudaMemset(v, 0, maxv * 8);
  std::vector<int> h(nidx);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto launch) {
    launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5.0;
  };
  const int threads = 256;
  const int occ[] = {4, 8};
  printf("gathers per launch %llu; times in ms; rate in G gathers/s\n", (unsigned long long)nidx);
  for (int o : occ) {
    const int blocks = nsm * o;
    const double t_stream = timeit([&] { stream_only<<<blocks, threads>>>(idx, nidx, out); });
    printf("grid %d: index stream alone %.3f ms (%.0f GB/s)\n", blocks, t_stream, nidx * 4 / t_stream / 1e6);
  }
  const int mbs[] = {8, 16, 32, 48, 64, 80, 96, 112, 128, 160, 192, 256};
  printf("%6s %10s %10s %10s %10s\n", "MB", "flat ms", "G/s", "rows5 ms", "G/s");
  uint64_t s = 88172645463325252ull;
  for (int mb : mbs) {
    const uint64_t span = (uint64_t)mb << 17;
    for (uint64_t i = 0; i < nidx; ++i) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      h[i] = (int)(s % span);
    }
    cudaMemcpy(idx, h.data(), nidx * 4, cudaMemcpyHostToDevice);
    const int blocks = nsm * 8;
    const double tf = timeit([&] { gather_flat<<<blocks, threads>>>(idx, v, nidx, out); });
    const double tr = timeit([&] { gather_rows5<<<blocks, threads>>>(idx, v, nidx / 5, out); });
    printf("%6d %10.3f %10.1f %10.3f %10.1f\n", mb, tf, nidx / tf / 1e6, tr, (nidx / 5 * 5) / tr / 1e6);
  }
  // die-split test: total footprint F, each SM gathers over one half of it
  printf("split: G/s by SM->half function (0: smid<nsm/2, k>0: bit k-1 of smid)\n%6s", "MB");
  for (int fn = 0; fn <= 7; ++fn) printf(" %8d", fn);
  printf("\n");
  const int smbs[] = {64, 96, 128, 160};
  for (int mb : smbs) {
    const uint64_t half = ((uint64_t)mb << 17) / 2;
    for (uint64_t i = 0; i < nidx; ++i) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      h[i] = (int)(s % half);
    }
    cudaMemcpy(idx, h.data(), nidx * 4, cudaMemcpyHostToDevice);
    printf("%6d", mb);
    for (int fn = 0; fn <= 7; ++fn) {
      const double t = timeit([&] { gather_split<<<nsm * 8, threads>>>(idx, v, nidx, half, fn, nsm, out); });
      printf(" %8.1f", nidx / t / 1e6);
    }
    printf("\n");
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
