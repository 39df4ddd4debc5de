// Random FP64 gather throughput on B200: LSU gathers (ld.global.nc) vs TMA
// tile::gather4 (cp.async.bulk.tensor.2d ... tile::gather4: four 16-byte rows of
// a 2-D view [N/2][2] of the vector per instruction, into shared memory).
// The C5 step SpMV passes are L1/TEX-wavefront bound on their random gathers
// (profiles/r02_C5_ncu_full.txt); TMA gathers bypass the LSU/L1 pipe.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_gather_probe tools/tma_gather_probe.cu -lcuda
//   ./tma_gather_probe [footprint_MB] [box_rows]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

__global__ void k_init(double* x, size_t n, int* idx, size_t m, uint32_t range) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    x[i] = 1.0 + (i & 1023) * 1e-3;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t h = i * 0x9E3779B97F4A7C15ull;
    h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
    idx[i] = (int)(h % range);
  }
}

// LSU: thread per gather, 4 independent gathers per thread per round
__global__ void k_ldg(const double* __restrict__ x, const int* __restrict__ idx, size_t m, double* out) {
  double s = 0;
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
  for (size_t i = t; i < m; i += nt) s += __ldg(x + __ldg(idx + i));
  if (s == 12345.0) out[0] = s;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// TMA: each warp owns a ring of stages; lane 0 issues G gather4 ops per stage
// (4*G elements), all lanes then sum the elements they pick from shared memory.
constexpr int G = 8;        // gather4 ops per stage (32 elements)
constexpr int STAGES = 4;   // stages in flight per warp
constexpr int WPB = 8;      // warps per block

__global__ void __launch_bounds__(WPB * 32) k_tma(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx,
                                                  size_t m, double* out, int rowbytes, int shift) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  __shared__ __align__(8) uint64_t bar[WPB][STAGES];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // each gather4 destination is 128-byte aligned (TMA requirement): op stride
  const int ops = 4 * rowbytes < 128 ? 128 : 4 * rowbytes;
  unsigned char* buf = smem + (size_t)w * STAGES * G * ops;
  if (lane == 0)
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar[w][s])));
  __syncwarp();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t per = 4 * G;  // elements per stage
  const size_t wid = blockIdx.x * (size_t)WPB + w, nw = (size_t)gridDim.x * WPB;
  const size_t nchunks = m / per;
  double s = 0;
  uint32_t phase[STAGES] = {0};
  auto issue = [&](int st, size_t chunk) {
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // order prior generic reads of the stage
      const int* ix = idx + chunk * per;
      const uint32_t b = smem_u32(&bar[w][st]);
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(G * 4 * rowbytes));
      for (int g = 0; g < G; ++g) {
        const int r0 = ix[4 * g] >> shift, r1 = ix[4 * g + 1] >> shift, r2 = ix[4 * g + 2] >> shift,
                  r3 = ix[4 * g + 3] >> shift;
        const uint32_t dst = smem_u32(buf + ((size_t)st * G + g) * ops);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
            "l"(&tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b)
            : "memory");
      }
    }
  };
  size_t c = wid;
  int st = 0;
  // prologue
  for (int k = 0; k < STAGES && c + k * nw < nchunks; ++k) issue(k, c + k * nw);
  for (size_t chunk = c; chunk < nchunks; chunk += nw) {
    const uint32_t b = smem_u32(&bar[w][st]);
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done) : "r"(b), "r"(phase[st]) : "memory");
    }
    phase[st] ^= 1;
    // lane l reads element l of the stage: row l (gather op l/4, row l%4), column idx&1
    const int e = idx[chunk * per + lane];
    const double* row =
        reinterpret_cast<const double*>(buf + ((size_t)st * G + (lane >> 2)) * ops + (lane & 3) * rowbytes);
    s += row[e & ((1 << shift) - 1)];
    __syncwarp();
    const size_t nxt = chunk + (size_t)STAGES * nw;
    if (nxt < nchunks) issue(st, nxt);
    st = (st + 1) % STAGES;
  }
  if (s == 12345.0) out[0] = s;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const double mb = argc > 1 ? atof(argv[1]) : 48.0;
  const size_t n = (size_t)(mb * 1048576.0 / 8) & ~(size_t)1;
  const size_t m = 64ull << 20;
  double *x, *out;
  int* idx;
  CK(cudaMalloc(&x, n * 8));
  CK(cudaMalloc(&idx, m * 4));
  CK(cudaMalloc(&out, 64));
  k_init<<<4096, 256>>>(x, n, idx, m, (uint32_t)n);
  CK(cudaDeviceSynchronize());
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  // LSU
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k_ldg<<<nsm * 8, 256>>>(x, idx, m, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
  }
  printf("footprint %.0f MB: LSU gathers %.1f G/s (%.3f ms for %zu)\n", mb, m / ms / 1e6, ms, m);
  // TMA
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  for (int rowdoubles : {2, 4}) {
    CUtensorMap tm;
    const int rowbytes = 8 * rowdoubles;
    cuuint64_t dims[2] = {(cuuint64_t)rowdoubles, (cuuint64_t)(n / rowdoubles)};
    cuuint64_t strides[1] = {(cuuint64_t)rowbytes};
    cuuint32_t box[2] = {(cuuint32_t)rowdoubles, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("encode (row %d B) failed: %d\n", rowbytes, (int)r);
      continue;
    }
    const size_t smem = (size_t)WPB * STAGES * G * (4 * rowbytes < 128 ? 128 : 4 * rowbytes) + 128;
    CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int blocks_per_sm : {4, 8, 16}) {
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k_tma<<<nsm * blocks_per_sm, WPB * 32, smem>>>(tm, idx, m, out, rowbytes, rowdoubles == 2 ? 1 : 2);
        cudaEventRecord(e1);
        cudaError_t err = cudaEventSynchronize(e1);
        if (err != cudaSuccess) {
          printf("tma kernel failed: %s\n", cudaGetErrorString(err));
          return 1;
        }
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("footprint %.0f MB: TMA gather4 rows of %d B, %d CTAs/SM: %.1f G/s (%.3f ms)\n", mb, rowbytes,
             blocks_per_sm, m / best / 1e6, best);
    }
  }
  return 0;
}
