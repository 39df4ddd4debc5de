// C5 y-step SpMV lab: w = G x~ over a C5-shaped matrix (m = 10M rows of 5
// uniformly random columns, n = 20M) fused with a 13-vector y-space epilogue,
// in column panels, with variants of the pass schedule.  Standalone (no
// libpdcs); each variant is timed with CUDA events after a producer kernel
// that streams the x-space like k_step_x and writes x~ (so L2 holds what it
// holds in the real loop).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o c5_lab tools/c5_lab.cu
//   ./c5_lab [reps]
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
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

constexpr int BS = 256;
constexpr int M = 10'000'000, N = 20'000'000, K = 5;

__device__ __forceinline__ uint32_t hash32(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return (uint32_t)x;
}

__global__ void k_gen(int* col, double* val) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < M; r += gridDim.x * blockDim.x) {
    int c[K];
    for (int k = 0; k < K; ++k) c[k] = hash32((uint64_t)r * K + k + 12345) % N;
    for (int i = 1; i < K; ++i)
      for (int j = i; j > 0 && c[j - 1] > c[j]; --j) { int t = c[j]; c[j] = c[j - 1]; c[j - 1] = t; }
    for (int k = 0; k < K; ++k) {
      col[(size_t)r * K + k] = c[k];
      val[(size_t)r * K + k] = 1.0 + (hash32((uint64_t)r * 77 + k) & 1023) * 1e-3;
    }
  }
}

__global__ void k_fill(double* p, size_t n, double v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = v + (i & 7) * 0.01;
}

// panel id of a column for cut points cuts[0..P]
__device__ __forceinline__ int panel_of(const int* cuts, int P, int c) {
  int p = 0;
  while (p + 1 < P && c >= cuts[p + 1]) ++p;
  return p;
}

__global__ void k_count(const int* col, const int* cuts, int P, int* cnt /*[P][M]*/) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < M; r += gridDim.x * blockDim.x) {
    int c[8] = {0};
    for (int k = 0; k < K; ++k) c[panel_of(cuts, P, col[(size_t)r * K + k])]++;
    for (int p = 0; p < P; ++p) cnt[(size_t)p * M + r] = c[p];
  }
}

__global__ void k_scatter(const int* col, const double* val, const int* cuts, int P, const int* po,
                          int* pci, double* pva) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < M; r += gridDim.x * blockDim.x) {
    int o[8];
    for (int p = 0; p < P; ++p) o[p] = po[(size_t)p * M + r];
    for (int k = 0; k < K; ++k) {
      const int c = col[(size_t)r * K + k];
      const int p = panel_of(cuts, P, c);
      pci[o[p]] = c;
      pva[o[p]] = val[(size_t)r * K + k];
      ++o[p];
    }
  }
}

// stream loads: MODE 0 plain __ldg, 1 L2::evict_first policy, 2 L1::no_allocate
template <int MODE, class T>
__device__ __forceinline__ T lds(const T* a) {
  if (MODE == 0) return __ldg(a);
  if (MODE == 1) {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    if (sizeof(T) == 8) {
      double v;
      asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
      return *reinterpret_cast<T*>(&v);
    } else {
      int v;
      asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
      return *reinterpret_cast<T*>(&v);
    }
  }
  if (sizeof(T) == 8) {
    double v;
    asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(a));
    return *reinterpret_cast<T*>(&v);
  } else {
    int v;
    asm("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(a));
    return *reinterpret_cast<T*>(&v);
  }
}

template <int MODE>
__device__ __forceinline__ void sts(double* a, double v) {
  if (MODE == 1) {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
  } else {
    *a = v;
  }
}

struct Y {  // y-space vectors of the epilogue
  double *y, *yh, *ya, *yb, *gx, *gxh, *gxa, *h;
  double *w;
};

// producer: like k_step_x (13 n-vector streams), writes x~
__global__ void __launch_bounds__(BS, 8) k_xstep(const double* a0, const double* a1, const double* a2,
                                                 const double* a3, const double* a4, const double* a5,
                                                 const double* a6, double* b0, double* b1, double* b2,
                                                 double* b3, double* xt, double* part, int j0 = 0, int j1 = N) {
  double acc = 0;
  for (int j = j0 + blockIdx.x * blockDim.x + threadIdx.x; j < j1; j += gridDim.x * blockDim.x) {
    const double x = a0[j], xh = a1[j], xa = a2[j], g = a4[j], gh = a5[j], ga = a6[j];
    const double xn = 0.9 * xh + 0.05 * x + 0.05 * xa, gn = 0.9 * gh + 0.05 * g + 0.05 * ga;
    b0[j] = xn;
    b1[j] = gn;
    b2[j] = 0.5 * (a3[j] + xn);
    const double p = fmin(fmax(xn - 0.01 * gn, -2.0), 2.0);
    b3[j] = p;
    xt[j] = 2.0 * p - xn;
    acc += p * p;
  }
  if (acc == 12345.0) part[0] = acc;
}

template <bool FIRST, int MODE = 0, int GMODE = 0>
__global__ void __launch_bounds__(BS) k_pass(const int* po, const int* ci, const double* va,
                                             const double* x, const double* win, double* wout) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < M; r += gridDim.x * blockDim.x) {
    const int b = lds<MODE>(po + r), e = lds<MODE>(po + r + 1);
    double s = FIRST ? 0.0 : lds<MODE>(win + r);
    for (int j = b; j < e; j += 4) {
      const int q = e - j;
      const int c0 = lds<MODE>(ci + j);
      const int c1 = q > 1 ? lds<MODE>(ci + j + 1) : 0, c2 = q > 2 ? lds<MODE>(ci + j + 2) : 0,
                c3 = q > 3 ? lds<MODE>(ci + j + 3) : 0;
      const double v0 = lds<MODE>(va + j);
      const double v1 = q > 1 ? lds<MODE>(va + j + 1) : 0.0, v2 = q > 2 ? lds<MODE>(va + j + 2) : 0.0,
                   v3 = q > 3 ? lds<MODE>(va + j + 3) : 0.0;
      const int g0 = GMODE ? r : c0, g1 = GMODE ? r : c1, g2 = GMODE ? r : c2, g3 = GMODE ? r : c3;
      const double x0 = __ldg(x + g0);
      const double x1 = q > 1 ? __ldg(x + g1) : 0.0, x2 = q > 2 ? __ldg(x + g2) : 0.0,
                   x3 = q > 3 ? __ldg(x + g3) : 0.0;
      s += v0 * x0;
      if (q > 1) s += v1 * x1;
      if (q > 2) s += v2 * x2;
      if (q > 3) s += v3 * x3;
    }
    sts<MODE>(wout + r, s);
  }
}

// ---- TMA-staged pass: each CTA streams a tile of TR rows' offsets, column
// indices and values into shared memory with cp.async.bulk (no LSU / L1 tag
// work for the streams), double-buffered; the threads read them with LDS and
// gather x with LDG (thread per row, index-order sums, as k_pass).
constexpr int TR = 256;
constexpr int TE = TR * K + 16;
struct __align__(16) Stage {
  int po[TR + 8];
  int ci[TE];
  double va[TE];
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}

template <bool FIRST>
__global__ void __launch_bounds__(TR, 4) k_pass_tma(const int* po, const int* ci, const double* va,
                                                    const double* x, const double* win, double* wout) {
  extern __shared__ __align__(128) unsigned char smraw[];
  Stage* st = reinterpret_cast<Stage*>((reinterpret_cast<uintptr_t>(smraw) + 127) & ~uintptr_t(127));
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ int meta[2][3];  // po base row, ci base entry, va base entry
  const int tid = threadIdx.x;
  const int ntiles = (M + TR - 1) / TR;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bar[0])));
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int s, int t) {
    const int r0 = t * TR, r1 = min(M, r0 + TR);
    const int e0 = po[r0], e1 = po[r1];
    const int a0 = r0 & ~3, npo = ((r1 + 1 - a0) + 3) & ~3;
    const int c0 = e0 & ~3, nci = ((e1 - c0) + 3) & ~3;
    const int v0 = e0 & ~1, nva = ((e1 - v0) + 1) & ~1;
    meta[s][0] = a0; meta[s][1] = c0; meta[s][2] = v0;
    const uint32_t bytes = npo * 4 + nci * 4 + nva * 8;
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(bytes));
    bulk(st[s].po, po + a0, npo * 4, &bar[s]);
    if (nci) bulk(st[s].ci, ci + c0, nci * 4, &bar[s]);
    if (nva) bulk(st[s].va, va + v0, nva * 8, &bar[s]);
  };
  int t = blockIdx.x;
  if (tid == 0) {
    if (t < ntiles) issue(0, t);
    if (t + (int)gridDim.x < ntiles) issue(1, t + gridDim.x);
  }
  uint32_t phase[2] = {0, 0};
  for (int k = 0; t < ntiles; t += gridDim.x, ++k) {
    const int s = k & 1;
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(su32(&bar[s])), "r"(phase[s]) : "memory");
    phase[s] ^= 1;
    const int r0 = t * TR, r = r0 + tid;
    const int a0 = meta[s][0], c0 = meta[s][1], v0 = meta[s][2];
    if (r < M) {
      const int b = st[s].po[r - a0], e = st[s].po[r + 1 - a0];
      double acc = FIRST ? 0.0 : win[r];
      for (int j = b; j < e; j += 4) {
        const int q = e - j;
        const int cc0 = st[s].ci[j - c0];
        const int cc1 = q > 1 ? st[s].ci[j + 1 - c0] : 0, cc2 = q > 2 ? st[s].ci[j + 2 - c0] : 0,
                  cc3 = q > 3 ? st[s].ci[j + 3 - c0] : 0;
        const double w0 = st[s].va[j - v0];
        const double w1 = q > 1 ? st[s].va[j + 1 - v0] : 0.0, w2 = q > 2 ? st[s].va[j + 2 - v0] : 0.0,
                     w3 = q > 3 ? st[s].va[j + 3 - v0] : 0.0;
        const double x0 = __ldg(x + cc0);
        const double x1 = q > 1 ? __ldg(x + cc1) : 0.0, x2 = q > 2 ? __ldg(x + cc2) : 0.0,
                     x3 = q > 3 ? __ldg(x + cc3) : 0.0;
        acc += w0 * x0;
        if (q > 1) acc += w1 * x1;
        if (q > 2) acc += w2 * x2;
        if (q > 3) acc += w3 * x3;
      }
      wout[r] = acc;
    }
    __syncthreads();  // every thread is done with stage s
    if (tid == 0 && t + 2 * (int)gridDim.x < ntiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(s, t + 2 * gridDim.x);
    }
  }
}

__device__ __forceinline__ void yepi(const Y& Yv, int r, double dot, double* acc) {
  const double yo = Yv.y[r];
  const double yn = 0.9 * Yv.yh[r] + 0.05 * yo + 0.05 * Yv.ya[r];
  const double go = Yv.gx[r];
  const double gn = 0.9 * Yv.gxh[r] + 0.05 * go + 0.05 * Yv.gxa[r];
  Yv.yb[r] = 0.5 * (Yv.yb[r] + yn);
  Yv.y[r] = yn;
  Yv.gx[r] = gn;
  const double hi = Yv.h[r];
  const double v = yn + 0.01 * (hi - dot);
  Yv.gxh[r] = 0.5 * (dot + gn);
  const double p = fmax(v, 0.0);
  Yv.yh[r] = p;
  acc[0] += (p - yn) * (p - yn);
  acc[1] += p * hi;
}

// last panel + epilogue
template <int MODE = 0>
__global__ void __launch_bounds__(BS, 6) k_final(const int* po, const int* ci, const double* va,
                                                 const double* x, const double* win, Y Yv, double* part) {
  double acc[2] = {0, 0};
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < M; r += gridDim.x * blockDim.x) {
    const int b = lds<MODE>(po + r), e = lds<MODE>(po + r + 1);
    double s = win ? lds<MODE>(win + r) : 0.0;
    for (int j = b; j < e; j += 4) {
      const int q = e - j;
      const int c0 = lds<MODE>(ci + j);
      const int c1 = q > 1 ? lds<MODE>(ci + j + 1) : 0, c2 = q > 2 ? lds<MODE>(ci + j + 2) : 0,
                c3 = q > 3 ? lds<MODE>(ci + j + 3) : 0;
      const double v0 = lds<MODE>(va + j);
      const double v1 = q > 1 ? lds<MODE>(va + j + 1) : 0.0, v2 = q > 2 ? lds<MODE>(va + j + 2) : 0.0,
                   v3 = q > 3 ? lds<MODE>(va + j + 3) : 0.0;
      const double x0 = __ldg(x + c0);
      const double x1 = q > 1 ? __ldg(x + c1) : 0.0, x2 = q > 2 ? __ldg(x + c2) : 0.0,
                   x3 = q > 3 ? __ldg(x + c3) : 0.0;
      s += v0 * x0;
      if (q > 1) s += v1 * x1;
      if (q > 2) s += v2 * x2;
      if (q > 3) s += v3 * x3;
    }
    yepi(Yv, r, s, acc);
  }
  if (acc[0] == 12345.0) part[0] = acc[0] + acc[1];
}

// epilogue only (w from the passes)
__global__ void __launch_bounds__(BS, 8) k_epi(const double* win, Y Yv, double* part) {
  double acc[2] = {0, 0};
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < M; r += gridDim.x * blockDim.x)
    yepi(Yv, r, win[r], acc);
  if (acc[0] == 12345.0) part[0] = acc[0] + acc[1];
}

struct Panels {
  int P;
  std::vector<int> cuts;
  int* d_po;  // [P][M+1] (each panel's own offsets into pci/pva)
  int* d_pci;
  double* d_pva;
};

Panels build(const int* d_col, const double* d_val, std::vector<int> cuts) {
  Panels Q;
  Q.P = (int)cuts.size() - 1;
  Q.cuts = cuts;
  int* d_cuts;
  CK(cudaMalloc(&d_cuts, sizeof(int) * cuts.size()));
  CK(cudaMemcpy(d_cuts, cuts.data(), sizeof(int) * cuts.size(), cudaMemcpyHostToDevice));
  int* cnt;
  CK(cudaMalloc(&cnt, sizeof(int) * ((size_t)Q.P * M + 1)));
  k_count<<<4096, BS>>>(d_col, d_cuts, Q.P, cnt);
  CK(cudaMalloc(&Q.d_po, sizeof(int) * ((size_t)Q.P * M + 1 + 64)));
  void* tmp = nullptr;
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, Q.d_po, (int)((size_t)Q.P * M + 1));
  CK(cudaMalloc(&tmp, tb));
  CK(cudaMemset(cnt + (size_t)Q.P * M, 0, sizeof(int)));
  cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, Q.d_po, (int)((size_t)Q.P * M + 1));
  CK(cudaDeviceSynchronize());
  CK(cudaMalloc(&Q.d_pci, sizeof(int) * ((size_t)M * K + 64)));
  CK(cudaMalloc(&Q.d_pva, sizeof(double) * ((size_t)M * K + 64)));
  k_scatter<<<4096, BS>>>(d_col, d_val, d_cuts, Q.P, Q.d_po, Q.d_pci, Q.d_pva);
  CK(cudaDeviceSynchronize());
  cudaFree(tmp);
  cudaFree(cnt);
  cudaFree(d_cuts);
  return Q;
}

void free_panels(Panels& Q) {
  cudaFree(Q.d_po);
  cudaFree(Q.d_pci);
  cudaFree(Q.d_pva);
}

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 10;
  int nsm = 148;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  int *d_col;
  double* d_val;
  CK(cudaMalloc(&d_col, sizeof(int) * (size_t)M * K));
  CK(cudaMalloc(&d_val, sizeof(double) * (size_t)M * K));
  k_gen<<<4096, BS>>>(d_col, d_val);
  CK(cudaDeviceSynchronize());
  // x-space
  std::vector<double*> xs(12);
  for (auto& p : xs) { CK(cudaMalloc(&p, sizeof(double) * N)); k_fill<<<4096, BS>>>(p, N, 0.1); }
  double* xt;
  CK(cudaMalloc(&xt, sizeof(double) * N));
  // y-space
  Y Yv;
  double** yp[] = {&Yv.y, &Yv.yh, &Yv.ya, &Yv.yb, &Yv.gx, &Yv.gxh, &Yv.gxa, &Yv.h, &Yv.w};
  for (auto pp : yp) { CK(cudaMalloc(pp, sizeof(double) * M)); k_fill<<<4096, BS>>>(*pp, M, 0.2); }
  double *wA, *wB, *part;
  CK(cudaMalloc(&wA, sizeof(double) * M));
  CK(cudaMalloc(&wB, sizeof(double) * M));
  CK(cudaMalloc(&part, 64));
  CK(cudaDeviceSynchronize());

  int occ_pass = 0, occ_fin = 0, occ_x = 0, occ_epi = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_pass, k_pass<false>, BS, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_fin, k_final<0>, BS, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_x, k_xstep, BS, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_epi, k_epi, BS, 0);
  const int gp = occ_pass * nsm, gf = occ_fin * nsm, gx = occ_x * nsm, ge = occ_epi * nsm;
  const size_t tma_smem = 2 * sizeof(Stage) + 128;
  CK(cudaFuncSetAttribute(k_pass_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tma_smem));
  CK(cudaFuncSetAttribute(k_pass_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tma_smem));
  int occ_tma = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_tma, k_pass_tma<false>, TR, tma_smem);
  const int gtma = occ_tma * nsm;
  printf("tma pass: %zu B smem per CTA, %d CTAs/SM\n", tma_smem, occ_tma);
  printf("grids pass %d final %d xstep %d epi %d\n", gp, gf, gx, ge);

  cudaEvent_t e0, e1, e2, e3;
  cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2); cudaEventCreate(&e3);
  auto xstep = [&]() {
    k_xstep<<<gx, BS>>>(xs[0], xs[1], xs[2], xs[3], xs[4], xs[5], xs[6], xs[7], xs[8], xs[9], xs[10], xt, part);
  };

  if (argc > 2 && atoi(argv[2]) == 1) {
    // pipelined x-step / y passes: x-step over column slice p+1 runs while the
    // pass over panel p gathers (two streams; grids split the SM slots)
    cudaStream_t s1, s2;
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    std::vector<cudaEvent_t> ev(8);
    for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    std::vector<int> cuts = {0, N / 3, (int)(2LL * N / 3), N};
    Panels Q = build(d_col, d_val, cuts);
    const int P = Q.P;
    const double fxs[] = {1.0, 0.5, 0.5, 0.25, 0.75, 0.35};
    const double fps[] = {1.0, 0.5, 1.0, 0.75, 0.5, 1.0};
    for (int pipe = 0; pipe < 2; ++pipe)
      for (int vi = 0; vi < 6; ++vi) {
        if (!pipe && vi) break;
        const int gxs = std::max(1, (int)(gx * fxs[vi])), gps = std::max(1, (int)(gp * fps[vi]));
        float best = 1e9;
        for (int it = 0; it < reps + 2; ++it) {
          CK(cudaEventRecord(e0, s1));
          double* win = nullptr;
          double* bufs[2] = {wA, wB};
          for (int p = 0; p < P; ++p) {
            cudaStream_t sx = pipe ? s1 : s2;
            if (!pipe && p == 0) CK(cudaStreamWaitEvent(s2, e0));
            k_xstep<<<pipe ? (p == 0 ? gx : gxs) : gx, BS, 0, sx>>>(xs[0], xs[1], xs[2], xs[3], xs[4], xs[5], xs[6],
                                                                  xs[7], xs[8], xs[9], xs[10], xt, part,
                                                                  cuts[p], cuts[p + 1]);
            CK(cudaEventRecord(ev[p], sx));
          }
          for (int p = 0; p < P; ++p) {
            CK(cudaStreamWaitEvent(s2, ev[p]));
            const int* po = Q.d_po + (size_t)p * M;
            double* wo = bufs[p & 1];
            if (p == 0) k_pass<true><<<pipe ? gps : gp, BS, 0, s2>>>(po, Q.d_pci, Q.d_pva, xt, nullptr, wo);
            else k_pass<false><<<pipe ? gps : gp, BS, 0, s2>>>(po, Q.d_pci, Q.d_pva, xt, win, wo);
            win = wo;
          }
          k_epi<<<ge, BS, 0, s2>>>(win, Yv, part);
          CK(cudaEventRecord(e2, s2));
          CK(cudaEventSynchronize(e2));
          float ms = 0;
          cudaEventElapsedTime(&ms, e0, e2);
          if (it >= 2) best = std::min(best, ms);
        }
        CK(cudaGetLastError());
        printf("%s fx %.2f fp %.2f: x-step + 3 passes + epilogue %.4f ms\n", pipe ? "pipelined " : "sequential",
               fxs[vi], fps[vi], best);
        fflush(stdout);
      }
    free_panels(Q);
    return 0;
  }

  struct Variant { const char* name; std::vector<double> fr; int order; int split; int mode = 0; int gmode = 0; int tma = 0; };
  // fr: panel width fractions; order 0 = panels 0..P-1, 1 = reversed; split: epilogue in its own kernel
  std::vector<Variant> V = {
      {"P3 equal fwd (current)", {1, 1, 1}, 0, 0},
      {"P3 split-epi evict_first", {1, 1, 1}, 0, 1, 1},
      {"P3 split-epi TMA-staged passes", {1, 1, 1}, 0, 1, 0, 0, 1},
      {"P3 split-epi plain passes", {1, 1, 1}, 0, 1, 0, 0, 0},
      {"P4 split-epi TMA-staged passes", {1, 1, 1, 1}, 0, 1, 0, 0, 1},
      {"P2 split-epi TMA-staged passes", {1, 1}, 0, 1, 0, 0, 1},
  };
  for (const Variant& v : V) {
    double tot = 0;
    for (double f : v.fr) tot += f;
    std::vector<int> cuts(1, 0);
    double acc = 0;
    for (size_t i = 0; i + 1 < v.fr.size(); ++i) { acc += v.fr[i]; cuts.push_back((int)(N * acc / tot)); }
    cuts.push_back(N);
    Panels Q = build(d_col, d_val, cuts);
    const int P = Q.P;
    std::vector<int> ord(P);
    for (int i = 0; i < P; ++i) ord[i] = v.order ? P - 1 - i : i;
    float best = 1e9, sum = 0, xbest = 1e9, ebest = 1e9;
    for (int it = 0; it < reps + 2; ++it) {
      CK(cudaEventRecord(e0));
      xstep();
      CK(cudaEventRecord(e1));
      double* win = nullptr;
      double* bufs[2] = {wA, wB};
      const int npass = v.split ? P : P - 1;
      for (int i = 0; i < npass; ++i) {
        const int p = ord[i];
        const int* po = Q.d_po + (size_t)p * M;
        double* wo = bufs[i & 1];
        if (v.tma) {
          const size_t smem = 2 * sizeof(Stage) + 128;
          if (i == 0) k_pass_tma<true><<<gtma, TR, smem>>>(po, Q.d_pci, Q.d_pva, xt, nullptr, wo);
          else k_pass_tma<false><<<gtma, TR, smem>>>(po, Q.d_pci, Q.d_pva, xt, win, wo);
        } else if (v.gmode == 1) {
          if (i == 0) k_pass<true, 0, 1><<<gp, BS>>>(po, Q.d_pci, Q.d_pva, xt, nullptr, wo);
          else k_pass<false, 0, 1><<<gp, BS>>>(po, Q.d_pci, Q.d_pva, xt, win, wo);
        } else if (v.mode == 1) {
          if (i == 0) k_pass<true, 1><<<gp, BS>>>(po, Q.d_pci, Q.d_pva, xt, nullptr, wo);
          else k_pass<false, 1><<<gp, BS>>>(po, Q.d_pci, Q.d_pva, xt, win, wo);
        } else if (v.mode == 2) {
          if (i == 0) k_pass<true, 2><<<gp, BS>>>(po, Q.d_pci, Q.d_pva, xt, nullptr, wo);
          else k_pass<false, 2><<<gp, BS>>>(po, Q.d_pci, Q.d_pva, xt, win, wo);
        } else {
          if (i == 0) k_pass<true><<<gp, BS>>>(po, Q.d_pci, Q.d_pva, xt, nullptr, wo);
          else k_pass<false><<<gp, BS>>>(po, Q.d_pci, Q.d_pva, xt, win, wo);
        }
        win = wo;
      }
      if (v.split) {
        CK(cudaEventRecord(e3));
        k_epi<<<ge, BS>>>(win, Yv, part);
      } else {
        const int p = ord[P - 1];
        if (v.mode == 1) k_final<1><<<gf, BS>>>(Q.d_po + (size_t)p * M, Q.d_pci, Q.d_pva, xt, win, Yv, part);
        else if (v.mode == 2) k_final<2><<<gf, BS>>>(Q.d_po + (size_t)p * M, Q.d_pci, Q.d_pva, xt, win, Yv, part);
        else k_final<0><<<gf, BS>>>(Q.d_po + (size_t)p * M, Q.d_pci, Q.d_pva, xt, win, Yv, part);
      }
      CK(cudaEventRecord(e2));
      CK(cudaEventSynchronize(e2));
      float ms = 0, xms = 0, ems = 0;
      cudaEventElapsedTime(&xms, e0, e1);
      cudaEventElapsedTime(&ms, e1, e2);
      if (v.split) cudaEventElapsedTime(&ems, e3, e2);
      if (it >= 2) { best = std::min(best, ms); sum += ms; xbest = std::min(xbest, xms); ebest = std::min(ebest, ems); }
    }
    CK(cudaGetLastError());
    double cs = 0.0;
    if (v.split) {  // checksum of the product w the passes produced (bit-identical schedules agree)
      std::vector<double> hw(M);
      const int npass = P;
      CK(cudaMemcpy(hw.data(), (npass - 1) & 1 ? wB : wA, sizeof(double) * M, cudaMemcpyDeviceToHost));
      for (double vv : hw) cs += vv;
    }
    printf("%-34s ystep best %.4f ms avg %.4f ms   (xstep %.4f ms, epilogue %.4f ms) w-sum %.17g\n", v.name,
           best, sum / reps, xbest, v.split ? ebest : 0.0f, cs);
    fflush(stdout);
    free_panels(Q);
  }
  return 0;
}
