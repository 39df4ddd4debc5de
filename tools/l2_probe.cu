// L2 probe for random FP64 gathers on B200 (tools/, not part of libpdcs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_probe tools/l2_probe.cu && ./l2_probe
// For footprints F (MB) it times 64M random 8-byte gathers spread over F:
//  (a) every SM gathers over all of F;
//  (b) SMs with even %smid gather over the first half, odd over the second
//      (if L2 halves cache per die, a die-consistent split would double the
//      effective capacity; an even/odd split shows whether SM parity tracks dies);
//  (c) SMs with %smid < nsm/2 take the first half.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}

__global__ void gather(const double* __restrict__ v, uint64_t n, uint64_t iters, int mode, int nsm,
                       double* out) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const unsigned sm = smid();
  uint64_t lo = 0, span = n;
  if (mode == 1) { span = n / 2; lo = (sm & 1) ? span : 0; }
  if (mode == 2) { span = n / 2; lo = (sm < (unsigned)nsm / 2) ? 0 : span; }
  double acc = 0.0;
  uint64_t s = tid * 0x9E3779B97F4A7C15ULL + 12345;
  for (uint64_t i = 0; i < iters; i += 4) {
    const uint64_t a = mix(s + i), b = mix(s + i + 1), c = mix(s + i + 2), d = mix(s + i + 3);
    acc += __ldg(v + lo + a % span) + __ldg(v + lo + b % span) + __ldg(v + lo + c % span) +
           __ldg(v + lo + d % span);
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  printf("SMs %d  L2 %.1f MB\n", nsm, l2 / 1048576.0);
  const uint64_t maxn = (256ull << 20) / 8;
  double* v;
  double* out;
  cudaMalloc(&v, maxn * 8);
  cudaMalloc(&out, 8);
  cudaMemset(v, 0, maxn * 8);
  const int threads = 256, blocks = nsm * 8;
  const uint64_t total = 64ull << 20;
  const uint64_t iters = total / ((uint64_t)threads * blocks);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int mbs[] = {8, 16, 24, 32, 40, 48, 56, 64, 80, 96, 112, 128, 160, 256};
  printf("%8s %14s %14s %14s   (Ggathers/s; modes: all / smid parity halves / smid range halves)\n",
         "MB", "all", "parity", "range");
  for (int mb : mbs) {
    const uint64_t n = (uint64_t)mb << 17;
    double rate[3];
    for (int mode = 0; mode < 3; ++mode) {
      gather<<<blocks, threads>>>(v, n, iters, mode, nsm, out);  // warm
      cudaEventRecord(e0);
      for (int r = 0; r < 3; ++r) gather<<<blocks, threads>>>(v, n, iters, mode, nsm, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      rate[mode] = 3.0 * iters * threads * blocks / (ms * 1e-3) / 1e9;
    }
    printf("%8d %14.2f %14.2f %14.2f\n", mb, rate[0], rate[1], rate[2]);
  }
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
