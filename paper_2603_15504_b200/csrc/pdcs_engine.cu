// libpdcs: host orchestration and the C ABI (include/pdcs.h).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "pdcs_kernels.cuh"

using namespace pdcs;

namespace {

// PDCS_TIMING=1: host-side phase times of engine setup on stderr (each phase
// ends with a stream synchronize, so only use it to find setup hot spots).
struct PhaseTimer {
  bool on = false;
  cudaStream_t s = nullptr;
  std::chrono::steady_clock::time_point t0;
  const char* what = "";
  PhaseTimer(const char* w, cudaStream_t st) : s(st), what(w) {
    const char* e = getenv("PDCS_TIMING");
    on = e && e[0] == '1';
    t0 = std::chrono::steady_clock::now();
  }
  void lap(const char* phase) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto t1 = std::chrono::steady_clock::now();
    fprintf(stderr, "[pdcs timing] %s %-22s %8.2f ms\n", what, phase,
            std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  }
};


thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      g_err = std::string(#call) + ": " + cudaGetErrorString(e_) + " (" + __FILE__ + ":" + \
              std::to_string(__LINE__) + ")";                                            \
      return 1;                                                                          \
    }                                                                                    \
  } while (0)

#define CKL()                                                                              \
  do {                                                                                     \
    g_launches.fetch_add(1, std::memory_order_relaxed);                                    \
    cudaError_t e_ = cudaGetLastError();                                                   \
    if (e_ != cudaSuccess) {                                                               \
      g_err = std::string("kernel launch: ") + cudaGetErrorString(e_) + " (" + __FILE__ + \
              ":" + std::to_string(__LINE__) + ")";                                        \
      return 1;                                                                            \
    }                                                                                      \
  } while (0)

// ---- NCCL, bound at run time to the libnccl the process already loaded -------
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*reduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
} g_nccl;

bool nccl_load() {
  if (g_nccl.tried) return g_nccl.ok;
  g_nccl.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    g_err = std::string("libnccl.so.2 not found: ") + dlerror();
    return false;
  }
  g_nccl.getUniqueId = (decltype(g_nccl.getUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.commInitRank = (decltype(g_nccl.commInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.allReduce = (decltype(g_nccl.allReduce))dlsym(h, "ncclAllReduce");
  g_nccl.allGather = (decltype(g_nccl.allGather))dlsym(h, "ncclAllGather");
  g_nccl.reduceScatter = (decltype(g_nccl.reduceScatter))dlsym(h, "ncclReduceScatter");
  g_nccl.broadcast = (decltype(g_nccl.broadcast))dlsym(h, "ncclBroadcast");
  g_nccl.reduce = (decltype(g_nccl.reduce))dlsym(h, "ncclReduce");
  g_nccl.groupStart = (decltype(g_nccl.groupStart))dlsym(h, "ncclGroupStart");
  g_nccl.groupEnd = (decltype(g_nccl.groupEnd))dlsym(h, "ncclGroupEnd");
  g_nccl.commDestroy = (decltype(g_nccl.commDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.errorString = (decltype(g_nccl.errorString))dlsym(h, "ncclGetErrorString");
  g_nccl.ok = g_nccl.getUniqueId && g_nccl.commInitRank && g_nccl.allReduce && g_nccl.allGather &&
              g_nccl.reduceScatter && g_nccl.broadcast && g_nccl.reduce && g_nccl.groupStart &&
              g_nccl.groupEnd && g_nccl.commDestroy && g_nccl.errorString;
  if (!g_nccl.ok) g_err = "libnccl.so.2 lacks the expected symbols";
  return g_nccl.ok;
}

#define CKN(call)                                                                     \
  do {                                                                                \
    ncclResult_t r_ = (call);                                                         \
    if (r_ != ncclSuccess) {                                                          \
      g_err = std::string(#call) + ": " + g_nccl.errorString(r_);                     \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

int nccl_allreduce(const double* send, double* recv, size_t count, void* comm, cudaStream_t s,
                   ncclRedOp_t op = ncclSum) {
  if (count == 0) return 0;
  CKN(g_nccl.allReduce(send, recv, count, ncclDouble, op, (ncclComm_t)comm, s));
  return 0;
}

// x-space exchanges of the sharded engine: rank r owns x-slice [xcut[r],
// xcut[r+1]).  Equal slices (cut r = r * xcnt, clipped to n) use the NCCL
// all-gather / reduce-scatter on buffers padded to nranks * xcnt; slices cut
// at primal cone-block boundaries use grouped per-root broadcasts / reduces.
int nccl_x_allgather(const Engine* E, double* v, cudaStream_t s) {
  // no early exit at one rank: the (in-place, no-op) all-gather then runs in the
  // world-1 sharded tests, so the captured NCCL call itself is exercised on the GPU
  ncclComm_t comm = (ncclComm_t)E->comm;
  if (E->xcnt > 0) {
    CKN(g_nccl.allGather(v + (size_t)E->rank * E->xcnt, v, E->xcnt, ncclDouble, comm, s));
    return 0;
  }
  CKN(g_nccl.groupStart());
  for (int r = 0; r < E->nranks; ++r) {
    const int a = E->xcut[r], len = E->xcut[r + 1] - a;
    if (len > 0) CKN(g_nccl.broadcast(v + a, v + a, len, ncclDouble, r, comm, s));
  }
  CKN(g_nccl.groupEnd());
  return 0;
}

// sum over the ranks of `part` (x-space, padded), each rank receiving its slice in `out`
int nccl_x_reduce_scatter(const Engine* E, const double* part, double* out, cudaStream_t s) {
  ncclComm_t comm = (ncclComm_t)E->comm;
  if (E->xcnt > 0) {
    CKN(g_nccl.reduceScatter(part, out + (size_t)E->rank * E->xcnt, E->xcnt, ncclDouble, ncclSum, comm,
                             s));
    return 0;
  }
  CKN(g_nccl.groupStart());
  for (int r = 0; r < E->nranks; ++r) {
    const int a = E->xcut[r], len = E->xcut[r + 1] - a;
    if (len > 0) CKN(g_nccl.reduce(part + a, out + a, len, ncclDouble, ncclSum, r, comm, s));
  }
  CKN(g_nccl.groupEnd());
  return 0;
}

inline int grid_for(int64_t n, int per = BS, int cap = MAX_GRID) {
  int64_t g = (n + per - 1) / per;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

int choose_vw(int64_t nnz, int64_t nrows) {
  if (nrows <= 0) return 1;
  const double mean = (double)nnz / (double)nrows;
  if (mean <= 6.0) return 1;
  int vw = 1;
  while (vw < 32 && vw < mean / 2.0) vw <<= 1;
  return vw;
}

KArgs make_args(const Engine* E) {
  const PdcsEngineDesc& d = E->d;
  KArgs A;
  A.n = E->n; A.m = E->m; A.nbox = E->nbox; A.m_zero = E->m_zero; A.m_elem = E->m_elem;
  A.x0 = E->xs0; A.x1 = E->xs1;
  A.c = d.d_c; A.h = d.d_h; A.l = d.d_l; A.u = d.d_u;
  A.c0 = d.d_c0; A.h0 = d.d_h0; A.l0 = d.d_l0; A.u0 = d.d_u0;
  A.d1 = d.d_d1; A.d2 = d.d_d2;
  A.x = d.d_x; A.y = d.d_y; A.xh = d.d_xh; A.yh = d.d_yh; A.xb = d.d_xb; A.yb = d.d_yb;
  A.xa = d.d_xa; A.ya = d.d_ya;
  A.gx = d.d_gx; A.gty = d.d_gty; A.gxa = d.d_gxa; A.gtya = d.d_gtya; A.w = d.d_w;
  A.gxh = d.d_gxh; A.gth = d.d_gth; A.gtr = d.d_gtr; A.xt = d.d_xt;
  A.tx0 = d.d_tx0; A.tx1 = d.d_tx1; A.tx2 = d.d_tx2;
  A.ty0 = d.d_ty0; A.ty1 = d.d_ty1; A.ty2 = d.d_ty2;
  A.ctrl = E->d_ctrl;
  A.err = E->d_err;
  A.keep_xt = E->keep_xt;
  A.keep_yh = E->keep_yh;
  A.exp_rho = E->d_exp_rho;
  A.ub = E->ubox ? (E->precond_mode == 2 ? 2 : 1) : 0;
  A.lu = E->ubox_l;
  A.uu = E->ubox_u;
  return A;
}

// ---- SpMV plan -------------------------------------------------------------
int build_plan(SpmvPlan& P, int nrows, int ncols, int nnz, const int* d_rp, const int* d_ci,
               const double* d_val, cudaStream_t s) {
  P.nrows = nrows; P.ncols = ncols; P.nnz = nnz;
  P.rowptr = d_rp; P.colidx = d_ci; P.val = d_val;
  P.vw = choose_vw(nnz, nrows);
  P.long_t = TILE_NNZ;
  // on the device: the spread of the short rows' lengths (chooses lane-mapped
  // vs tiled step kernels) and the long rows with their extents -- no copy of
  // the row pointers to the host (setup was 117 ms on C5 with a host pass)
  std::vector<int> lrows;
  std::vector<int2> lext;
  if (nrows > 0) {
    unsigned long long* st = nullptr;
    CK(cudaMallocAsync(&st, sizeof(unsigned long long) * 4, s));
    CK(cudaMemsetAsync(st, 0, sizeof(unsigned long long) * 4, s));
    k_row_stats<<<grid_for(nrows), BS, 0, s>>>(d_rp, nrows, P.long_t, st);
    CKL();
    unsigned long long h[4];
    CK(cudaMemcpyAsync(h, st, sizeof(h), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const double cnt = (double)h[2];
    const double mean = cnt > 0 ? (double)h[0] / cnt : 0.0;
    const double var = cnt > 0 ? std::max(0.0, (double)h[1] / cnt - mean * mean) : 0.0;
    P.len_cv = mean > 0.0 ? std::sqrt(var) / mean : 0.0;
    const int nl = (int)h[3];
    if (nl > 0) {
      int *rows = nullptr, *num = nullptr;
      int2* ext = nullptr;
      CK(cudaMallocAsync(&rows, sizeof(int) * nl, s));
      CK(cudaMallocAsync(&num, sizeof(int), s));
      CK(cudaMallocAsync(&ext, sizeof(int2) * nl, s));
      size_t tb = 0;
      thrust::counting_iterator<int> it(0);
      CK(cub::DeviceSelect::If(nullptr, tb, it, rows, num, nrows, IsLongRow{d_rp, P.long_t}, s));
      void* tmp = nullptr;
      CK(cudaMallocAsync(&tmp, tb, s));
      CK(cub::DeviceSelect::If(tmp, tb, it, rows, num, nrows, IsLongRow{d_rp, P.long_t}, s));
      k_row_extents<<<grid_for(nl), BS, 0, s>>>(d_rp, rows, nl, ext);
      CKL();
      lrows.resize(nl);
      lext.resize(nl);
      CK(cudaMemcpyAsync(lrows.data(), rows, sizeof(int) * nl, cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(lext.data(), ext, sizeof(int2) * nl, cudaMemcpyDeviceToHost, s));
      CK(cudaFreeAsync(tmp, s));
      CK(cudaFreeAsync(rows, s));
      CK(cudaFreeAsync(num, s));
      CK(cudaFreeAsync(ext, s));
      CK(cudaStreamSynchronize(s));
    }
    CK(cudaFreeAsync(st, s));
  }
  // entries per long-row chunk (one CTA reduction each): the long rows' entries
  // spread over one wave of k_long_partial (8 CTAs per SM; a partial second
  // wave cost C4 ~8%), each row cut into equal chunks; PDCS_TUNE=chunk=N fixes N
  long long total = 0;
  for (const int2& x : lext) total += x.y - x.x;
  int dev = 0, nsm_ = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm_, cudaDevAttrMultiProcessorCount, dev);
  const long long resident = 8LL * nsm_;
  const long long slots = std::max<long long>(resident - (long long)lrows.size(), resident / 2);
  long long chunk = std::max<long long>(2048, (total + slots - 1) / slots);
  if (const char* env = getenv("PDCS_TUNE")) {
    const char* p = strstr(env, "chunk=");
    if (p && (p == env || p[-1] == ',')) chunk = std::max(256, atoi(p + 6));
  }
  std::vector<int> lfirst;
  std::vector<int4> chunks;
  for (size_t i = 0; i < lrows.size(); ++i) {
    const int r = lrows[i], b = lext[i].x, e = lext[i].y;
    const long long len = e - b, nc = (len + chunk - 1) / chunk, cl = (len + nc - 1) / nc;
    lfirst.push_back((int)chunks.size());
    for (long long j = b; j < e; j += cl)
      chunks.push_back(make_int4(r, (int)j, (int)std::min<long long>(e, j + cl), (int)i));
  }
  lfirst.push_back((int)chunks.size());
  P.n_long = (int)lrows.size();
  P.n_chunks = (int)chunks.size();
  if (P.n_long > 0) {
    CK(cudaMalloc(&P.d_long_rows, sizeof(int) * P.n_long));
    CK(cudaMalloc(&P.d_long_first, sizeof(int) * (P.n_long + 1)));
    CK(cudaMalloc(&P.d_chunks, sizeof(int4) * P.n_chunks));
    CK(cudaMalloc(&P.d_chunk_out, sizeof(double) * P.n_chunks));
    CK(cudaMalloc(&P.d_long_cnt, sizeof(unsigned) * P.n_long));
    CK(cudaMemsetAsync(P.d_long_cnt, 0, sizeof(unsigned) * P.n_long, s));
    CK(cudaMemcpyAsync(P.d_long_rows, lrows.data(), sizeof(int) * P.n_long, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(P.d_long_first, lfirst.data(), sizeof(int) * (P.n_long + 1), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(P.d_chunks, chunks.data(), sizeof(int4) * P.n_chunks, cudaMemcpyHostToDevice, s));
    k_chunk_dense<<<std::min(P.n_chunks, MAX_GRID), BS, 0, s>>>(P.d_chunks, P.n_chunks, d_ci);
    CKL();
    CK(cudaStreamSynchronize(s));
  }
  P.grid = grid_for(nrows, BS / P.vw);
  return 0;
}

// CSR-stream tiles over the short rows (<= TILE_ROWS rows, <= TILE_NNZ
// entries): only built when the tiled step kernels are chosen.
// head[r] (optional): first row of the cone block holding row r, -1 outside
// blocks; tiles are then never cut inside a block.  Returns 4 when a block
// does not fit in one tile (the caller falls back to the unfused y-step).
int build_tiles(SpmvPlan& P, cudaStream_t s, const std::vector<int>* head = nullptr) {
  const int nrows = P.nrows;
  std::vector<int> rp(nrows + 1, 0);
  if (nrows > 0) {
    CK(cudaMemcpyAsync(rp.data(), P.rowptr, sizeof(int) * (nrows + 1), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  std::vector<int> tiles(1, 0);
  for (int r = 0; r < nrows;) {
    const int t0 = r;
    int nz = 0, cnt = 0;
    while (r < nrows && cnt < TILE_ROWS) {
      int len = rp[r + 1] - rp[r];
      if (len > P.long_t) len = 0;
      if (cnt > 0 && nz + len > TILE_NNZ) break;
      nz += len;
      ++cnt;
      ++r;
    }
    if (head && r < nrows && (*head)[r] >= 0 && (*head)[r] < r) {  // cut inside a block: back up
      if ((*head)[r] <= t0) return 4;
      r = (*head)[r];
    }
    tiles.push_back(r);
  }
  P.ntiles = (int)tiles.size() - 1;
  CK(cudaMalloc(&P.d_tiles, sizeof(int) * tiles.size()));
  CK(cudaMemcpyAsync(P.d_tiles, tiles.data(), sizeof(int) * tiles.size(), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  return 0;
}

// PDCS_TUNE="key=value,..." launch-configuration override (dflt when absent)
double tune_env(const char* key, double dflt) {
  const char* env = getenv("PDCS_TUNE");
  if (!env) return dflt;
  std::string s(env), k = std::string(key) + "=";
  size_t p = s.find(k);
  if (p == std::string::npos || (p > 0 && s[p - 1] != ',')) return dflt;
  return atof(s.c_str() + p + k.size());
}

// Row classes for the class-split step SpMV (mixed row lengths, no chunked
// long rows): the rows of more than CLS_SHORT entries, listed ascending (the
// epilogue sums the short ones), and the lanes per long row.
struct IsLongClassRow {
  const int* rp;
  __host__ __device__ bool operator()(int r) const { return rp[r + 1] - rp[r] > CLS_SHORT; }
};

int build_classes(SpmvPlan& P, cudaStream_t s, int nsm) {
  const int nrows = P.nrows;
  unsigned long long* st = nullptr;
  CK(cudaMallocAsync(&st, sizeof(unsigned long long) * 4, s));
  CK(cudaMemsetAsync(st, 0, sizeof(unsigned long long) * 4, s));
  k_row_stats<<<grid_for(nrows), BS, 0, s>>>(P.rowptr, nrows, CLS_SHORT, st);
  CKL();
  unsigned long long h[4];
  CK(cudaMemcpyAsync(h, st, sizeof(h), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaFreeAsync(st, s));
  P.n_cls_short = (int)h[2];
  P.n_cls_long = (int)h[3];
  P.nnz_cls_long = (long long)P.nnz - (long long)h[0];
  const double mean_long = P.n_cls_long ? (double)(P.nnz - (long long)h[0]) / P.n_cls_long : 0.0;
  // lanes per long row: about 4-8 entries per lane (PDCS_TUNE cls_vw=8|16|32)
  const int vw = (int)tune_env("cls_vw", mean_long <= 64.0 ? 8.0 : (mean_long <= 160.0 ? 16.0 : 32.0));
  P.cls_vw = vw == 32 ? 32 : (vw == 16 ? 16 : (vw == 4 ? 4 : 8));
  CK(cudaMalloc(&P.d_cls_long, sizeof(int) * std::max(P.n_cls_long, 1)));
  int* num = nullptr;
  CK(cudaMallocAsync(&num, sizeof(int), s));
  thrust::counting_iterator<int> it(0);
  size_t tb = 0;
  CK(cub::DeviceSelect::If(nullptr, tb, it, P.d_cls_long, num, nrows, IsLongClassRow{P.rowptr}, s));
  void* tmp = nullptr;
  CK(cudaMallocAsync(&tmp, std::max<size_t>(tb, 1), s));
  CK(cub::DeviceSelect::If(tmp, tb, it, P.d_cls_long, num, nrows, IsLongClassRow{P.rowptr}, s));
  CK(cudaFreeAsync(tmp, s));
  CK(cudaFreeAsync(num, s));
  CK(cudaStreamSynchronize(s));
  int occ = 1;
  const void* fn = P.cls_vw == 32   ? (const void*)k_rows_pass<32>
                   : P.cls_vw == 16 ? (const void*)k_rows_pass<16>
                   : P.cls_vw == 4  ? (const void*)k_rows_pass<4>
                                    : (const void*)k_rows_pass<8>;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, BS, 0) != cudaSuccess || occ < 1) occ = 1;
  P.cls_grid_l = std::max(1, std::min(grid_for(P.n_cls_long, BS / P.cls_vw, 1 << 30), occ * nsm));
  return 0;
}

void free_plan(SpmvPlan& P) {
  cudaFree(P.d_cls_long);
  cudaFree(P.d_long_rows);
  cudaFree(P.d_long_first);
  cudaFree(P.d_chunks);
  cudaFree(P.d_chunk_out);
  cudaFree(P.d_long_cnt);
  cudaFree(P.d_tiles);
  P = SpmvPlan();
}

// Long rows: chunk partials then per-row finalize into y.
int launch_long(const SpmvPlan& P, const double* x, double* y, const PdcsCtrl* ctrl, int gate,
                cudaStream_t s) {
  if (P.n_long == 0) return 0;
  k_long_partial<<<grid_for(P.n_chunks, 1), BS, 0, s>>>(P.d_chunks, P.n_chunks, P.colidx, P.val, x,
                                                        P.d_chunk_out, ctrl, gate, P.d_long_first,
                                                        P.d_long_cnt, y);
  CKL();
  return 0;
}

template <int VW>
int launch_spmv_vw(const SpmvPlan& P, const double* x, double* y, cudaStream_t s,
                   const PdcsCtrl* ctrl, int gate) {
  k_spmv<VW><<<P.grid, BS, 0, s>>>(P.nrows, P.rowptr, P.colidx, P.val, x, y, P.long_t, ctrl, gate);
  CKL();
  return 0;
}

// y = A x over the CSR (long rows chunked); with ctrl, gated like the step kernels.
int launch_spmv(const SpmvPlan& P, const double* x, double* y, cudaStream_t s,
                const PdcsCtrl* ctrl = nullptr, int gate = 0) {
  if (P.nrows == 0) return 0;
  if (launch_long(P, x, y, ctrl, gate, s)) return 1;
  switch (P.vw) {
    case 1: return launch_spmv_vw<1>(P, x, y, s, ctrl, gate);
    case 2: return launch_spmv_vw<2>(P, x, y, s, ctrl, gate);
    case 4: return launch_spmv_vw<4>(P, x, y, s, ctrl, gate);
    case 8: return launch_spmv_vw<8>(P, x, y, s, ctrl, gate);
    case 16: return launch_spmv_vw<16>(P, x, y, s, ctrl, gate);
    default: return launch_spmv_vw<32>(P, x, y, s, ctrl, gate);
  }
}

template <int OP>
int launch_rowred(const SpmvPlan& P, const double* val, double* out, cudaStream_t s) {
  if (P.nrows == 0) return 0;
  k_rowred_short<OP><<<grid_for(P.nrows), BS, 0, s>>>(P.nrows, P.rowptr, val, out, P.long_t);
  CKL();
  if (P.n_long) {
    k_rowred_long_partial<OP><<<grid_for(P.n_chunks, 1), BS, 0, s>>>(P.d_chunks, P.n_chunks, val,
                                                                    P.d_chunk_out);
    CKL();
    k_rowred_long_final<OP><<<grid_for(P.n_long, 128), 128, 0, s>>>(
        P.d_long_rows, P.d_long_first, P.n_long, P.d_chunk_out, out);
    CKL();
  }
  return 0;
}

// ---- cone block tables -------------------------------------------------------
int build_table(BlockTable& T, std::vector<PdcsBlock> blocks, cudaStream_t s, bool giant_ok = false,
                int thread_max = THREAD_CLASS_MAX) {
  std::vector<PdcsBlock> ex, th, hf, wa, ct, gi;
  for (auto& b : blocks) {
    if ((b.kind == PDCS_EXP || b.kind == PDCS_DUAL_EXP) && b.dim == 3) ex.push_back(b);
    else if (b.dim <= thread_max) th.push_back(b);
    else if (b.dim <= HALF_CLASS_MAX) hf.push_back(b);
    else if (b.dim <= WARP_CLASS_MAX) wa.push_back(b);
    else if (giant_ok && b.kind == PDCS_SOC && b.dim > GIANT_MIN) gi.push_back(b);
    else ct.push_back(b);
  }
  T.n_exp = (int)ex.size();
  T.n_thread = (int)th.size();
  T.n_half = (int)hf.size();
  T.n_warp = (int)wa.size();
  T.n_cta = (int)ct.size();
  T.n_giant = (int)gi.size();
  std::vector<PdcsBlock> all;
  all.insert(all.end(), ex.begin(), ex.end());
  all.insert(all.end(), th.begin(), th.end());
  all.insert(all.end(), hf.begin(), hf.end());
  all.insert(all.end(), wa.begin(), wa.end());
  all.insert(all.end(), ct.begin(), ct.end());
  all.insert(all.end(), gi.begin(), gi.end());
  T.g_exp = T.n_exp ? grid_for(T.n_exp) : 0;
  T.g_thread = T.n_thread ? grid_for(T.n_thread) : 0;
  T.g_half = T.n_half ? grid_for(T.n_half, BS / 16) : 0;
  T.g_warp = T.n_warp ? grid_for(T.n_warp, BS / 32) : 0;
  T.g_cta = T.n_cta ? std::min(T.n_cta, MAX_GRID) : 0;
  T.g_giant = T.n_giant ? GIANT_GRID : 0;
  if (!all.empty()) {
    CK(cudaMalloc(&T.d_all, sizeof(PdcsBlock) * all.size()));
    CK(cudaMemcpyAsync(T.d_all, all.data(), sizeof(PdcsBlock) * all.size(), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
  }
  if (T.n_giant) {
    CK(cudaMalloc(&T.d_gpart, sizeof(double) * 2 * T.g_giant * T.n_giant));
    CK(cudaMalloc(&T.d_gcoef, sizeof(double) * 8 * T.n_giant));
  }
  return 0;
}

void free_table(BlockTable& T) {
  cudaFree(T.d_queue);
  cudaFree(T.d_qcount);
  cudaFree(T.d_all);
  cudaFree(T.d_gpart);
  cudaFree(T.d_gcoef);
  T = BlockTable();
}

template <int OP>
int launch_blocks(const BlockTable& T, const KArgs& A, const BlkParams& P, double* part, int cap,
                  int slot0, int gate, cudaStream_t s) {
  int slot = slot0;
  const PdcsBlock* base = T.d_all;
  if (T.n_exp && OP == OP_STEP_Y && T.exp_split) {
    auto fast = T.exp_minb == 2 ? k_exp_y_fast<2> : (T.exp_minb == 3 ? k_exp_y_fast<3> : k_exp_y_fast<4>);
    fast<<<T.g_exp, BS, 0, s>>>(base, T.n_exp, T.exp_per, A, T.d_queue, T.d_qcount, part, cap, slot, gate);
    CKL();
    k_exp_y_slow<<<T.g_exp, BS, 0, s>>>(base, T.exp_per, A, T.d_queue, T.d_qcount, part, cap,
                                        slot + T.g_exp, gate);
    CKL();
    slot += T.g_exp;
  } else if (T.n_exp) {
    // PDCS_TUNE expminb=2|3: more registers per thread for the (FP64-bound) y-step exp blocks
    if (OP == OP_STEP_Y && T.exp_minb == 2)
      k_blk_exp<OP, 2><<<T.g_exp, BS, 0, s>>>(base, T.n_exp, A, P, part, cap, slot, gate);
    else if (OP == OP_STEP_Y && T.exp_minb == 3)
      k_blk_exp<OP, 3><<<T.g_exp, BS, 0, s>>>(base, T.n_exp, A, P, part, cap, slot, gate);
    else
      k_blk_exp<OP><<<T.g_exp, BS, 0, s>>>(base, T.n_exp, A, P, part, cap, slot, gate);
    CKL();
  }
  slot += T.g_exp;
  base += T.n_exp;
  if (T.n_thread) {
    k_blk_thread<OP><<<T.g_thread, BS, 0, s>>>(base, T.n_thread, A, P, part, cap, slot, gate);
    CKL();
  }
  slot += T.g_thread;
  base += T.n_thread;
  if (T.n_half) {
    // register budget of the step half-warp blocks: 3 CTAs per SM (80 registers)
    // measured best on C2 (PDCS_TUNE halfminb=1|3|4; profiles/r02_sweeps.txt)
    // lanes per block: 4 (default; fewer CTAs than the class's slots), 8, 2 or 16
    if (OP != OP_PROJECT && T.half_w == 4)
      k_blk_half<OP, 3, 4><<<std::min(T.g_half, grid_for(T.n_half, BS / 4)), BS, 0, s>>>(base, T.n_half, A, P,
                                                                                         part, cap, slot, gate);
    else if (OP != OP_PROJECT && T.half_w == 8)
      k_blk_half<OP, 3, 8><<<std::min(T.g_half, grid_for(T.n_half, BS / 8)), BS, 0, s>>>(base, T.n_half, A, P,
                                                                                         part, cap, slot, gate);
    else if (OP != OP_PROJECT && T.half_w == 2)
      k_blk_half<OP, 3, 2><<<std::min(T.g_half, grid_for(T.n_half, BS / 2)), BS, 0, s>>>(base, T.n_half, A, P,
                                                                                         part, cap, slot, gate);
    else if (OP != OP_PROJECT && T.half_minb == 4)
      k_blk_half<OP, 4><<<T.g_half, BS, 0, s>>>(base, T.n_half, A, P, part, cap, slot, gate);
    else if (OP != OP_PROJECT && T.half_minb == 3)
      k_blk_half<OP, 3><<<T.g_half, BS, 0, s>>>(base, T.n_half, A, P, part, cap, slot, gate);
    else
      k_blk_half<OP><<<T.g_half, BS, 0, s>>>(base, T.n_half, A, P, part, cap, slot, gate);
    CKL();
  }
  slot += T.g_half;
  base += T.n_half;
  if (T.n_warp) {
    k_blk_warp<OP><<<T.g_warp, BS, 0, s>>>(base, T.n_warp, A, P, part, cap, slot, gate);
    CKL();
  }
  slot += T.g_warp;
  base += T.n_warp;
  if (T.n_cta) {
    k_blk_cta<OP><<<T.g_cta, CTA_BLOCK_THREADS, 0, s>>>(base, T.n_cta, A, P, part, cap, slot, gate);
    CKL();
  }
  slot += T.g_cta;
  base += T.n_cta;
  if (T.n_giant) {
    const PdcsBlock* gt = base;
    if (OP == OP_STEP_Y) {
      k_giant_soc_a<<<T.g_giant, BS, 0, s>>>(gt, T.n_giant, A, T.d_gpart, T.g_giant);
      CKL();
      k_giant_soc_b<<<1, BS, 0, s>>>(gt, T.n_giant, A, T.d_gpart, T.g_giant, T.g_giant, T.d_gcoef);
      CKL();
      k_giant_soc_c<<<T.g_giant, BS, 0, s>>>(gt, T.n_giant, A, T.d_gcoef, part, cap, slot);
      CKL();
    } else if (OP == OP_PROJECT) {
      k_giant_proj_a<<<T.g_giant, BS, 0, s>>>(gt, T.n_giant, P.in, T.d_gpart, T.g_giant);
      CKL();
      k_giant_proj_b<<<1, BS, 0, s>>>(gt, T.n_giant, P.in, T.d_gpart, T.g_giant, T.g_giant, T.d_gcoef);
      CKL();
      k_giant_proj_c<<<T.g_giant, BS, 0, s>>>(gt, T.n_giant, P.in, P.out, T.d_gcoef);
      CKL();
    } else {
      // other uses: one CTA per giant block; reduction slots are the giant
      // class's, the surplus ones stay zero
      k_blk_cta<OP><<<std::min(T.n_giant, T.g_giant), CTA_BLOCK_THREADS, 0, s>>>(gt, T.n_giant, A, P, part,
                                                                                 cap, slot, gate);
      CKL();
    }
  }
  return 0;
}

// Launch of a step kernel of the trial; with pdl (E->pdl) as a programmatic
// dependent launch: the kernel's CTAs are scheduled while the previous
// kernel's last CTAs (and its folded controller) finish, and wait in
// pdl_enter() for its completion.
template <typename... KP, typename... Args>
cudaError_t launch_step(bool pdl, void (*k)(KP...), int grid, cudaStream_t s, Args... args) {
  if (!pdl) {
    k<<<grid, BS, 0, s>>>(args...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(BS);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, args...);
}
bool use_pdl(const Engine* E) { return E->pdl && !E->comm; }

// ---- one line-search trial (graph slot) ----------------------------------
// Final-pass source of a fused step SpMV: the last panel (after np-1 partial
// passes into wpart) or the whole CSR.
// Tile source of pass p of a panelled step SpMV (p = np-1: the fused last pass).
TileSrc tile_source(const SpmvPlan& P, const PanelPlan& Q, int p, const double* wpart) {
  TileSrc S;
  S.tiles = P.d_tiles;
  S.ntiles = P.ntiles;
  S.po = Q.d_po + (size_t)p * P.nrows;
  S.ci = Q.d_pci;
  S.va = Q.d_pva;
  S.wpart = p > 0 ? wpart : nullptr;
  S.orig_rp = (p == Q.np - 1 && P.n_long) ? P.rowptr : nullptr;
  S.long_t = P.long_t;
  return S;
}

int launch_panel_passes(Engine* E, const SpmvPlan& P, const PanelPlan& Q, const double* x,
                        double* wpart, int grid, int gate) {
  for (int p = 0; p + 1 < Q.np; ++p) {
    k_tile_pass<<<grid, BS, 0, E->stream>>>(tile_source(P, Q, p, wpart), x, wpart, E->d_ctrl, gate);
    CKL();
  }
  return 0;
}

template <int VW, int GP>
int lane_passes(Engine* E, const SpmvPlan& P, const PanelPlan& Q, const double* x, double* wpart,
                int gate, float keep) {
  for (int p = 0; p + 1 < Q.np; ++p) {
    CK(launch_step(use_pdl(E), k_lane_pass<VW, GP>, P.pass_grid, E->stream, tile_source(P, Q, p, wpart),
                   P.nrows, x, wpart, (const PdcsCtrl*)E->d_ctrl, gate, keep));
    CKL();
  }
  return 0;
}

// Controllers folded into the step kernels when no cone-block kernel (and no
// collective) follows them in the slot.
CtrlFuse fuse_ls(const Engine* E) {
  CtrlFuse F{};
  if (E->comm || (E->has_yblocks && !E->soc_tile) || !E->fuse_ctrl) return F;
  F.mode = 1; F.ticket = E->d_ticket; F.C = E->d_ctrl;
  F.partA = E->d_partX; F.capA = E->capX; F.partB = E->d_partY; F.capB = E->capY;
  F.red = E->d_red; F.err = E->d_err;
  return F;
}
CtrlFuse fuse_beta(const Engine* E) {
  CtrlFuse F{};
  if (E->comm || E->has_xblocks || !E->fuse_ctrl) return F;
  F.mode = 2; F.ticket = E->d_ticket + 1; F.C = E->d_ctrl;
  F.partB = E->d_partT; F.capB = E->capT; F.red = E->d_red; F.err = E->d_err;
  return F;
}

// Split step (E->split): every panel a gather-only pass, the last writing the
// full product into `out`; then the pure-streaming epilogue kernel.
template <int VW, int GP, bool HS>
int split_passes(Engine* E, const SpmvPlan& P, const PanelPlan& Q, const double* x, double* wpart,
                 double* out, int gate, float keep) {
  for (int p = 0; p < Q.np; ++p) {
    double* dst = p + 1 == Q.np ? out : wpart;
    CK(launch_step(use_pdl(E), k_lane_pass<VW, GP, HS>, P.pass_grid, E->stream, tile_source(P, Q, p, wpart),
                   P.nrows, x, dst, (const PdcsCtrl*)E->d_ctrl, gate, keep));
    CKL();
  }
  return 0;
}

template <bool HS>
int split_y(Engine* E, const KArgs& A) {
  if (split_passes<1, 0, HS>(E, E->G, E->PG, E->d.d_xt, E->d_wpart_y, E->d.d_w, 1, E->keep_xt)) return 1;
  if (E->vec && E->m_elem == E->m)
    CK(launch_step(use_pdl(E), k_y_epi2, E->G.grid, E->stream, A, E->d_partY, E->capY, fuse_ls(E)));
  else
    CK(launch_step(use_pdl(E), k_y_epi<false>, E->G.grid, E->stream, A, E->d_partY, E->capY, fuse_ls(E), ShortRows{}));
  CKL();
  return 0;
}

template <bool HS>
int split_t(Engine* E, const KArgs& A) {
  if (split_passes<1, 0, HS>(E, E->GT, E->PGT, E->d.d_yh, E->d_wpart_x, E->d.d_gth, 2, E->keep_yh)) return 1;
  if (E->vec && E->ubox && E->nbox == E->n)
    CK(launch_step(use_pdl(E), k_t_epi2, E->GT.grid, E->stream, A, E->d_partT, E->capT, fuse_beta(E), ShortRows{}));
  else
    CK(launch_step(use_pdl(E), k_t_epi<false>, E->GT.grid, E->stream, A, E->d_partT, E->capT, fuse_beta(E), ShortRows{}));
  CKL();
  return 0;
}

template <int VW, int GP>
int lane_y(Engine* E, const KArgs& A) {
  if (lane_passes<VW, GP>(E, E->G, E->PG, E->d.d_xt, E->d_wpart_y, 1, E->keep_xt)) return 1;
  CK(launch_step(use_pdl(E), k_step_y_lane<VW, GP>, E->G.grid, E->stream, A, E->exp_fused ? E->m_elem : E->G.nrows,
                 tile_source(E->G, E->PG, E->PG.np - 1, E->d_wpart_y), E->d_partY, E->capY, fuse_ls(E)));
  CKL();
  return 0;
}

template <int VW, int GP>
int lane_t(Engine* E, const KArgs& A) {
  if (lane_passes<VW, GP>(E, E->GT, E->PGT, E->d.d_yh, E->d_wpart_x, 2, E->keep_yh)) return 1;
  CK(launch_step(use_pdl(E), k_step_t_lane<VW, GP>, E->GT.grid, E->stream, A, (E->texp_fused && !E->comm) ? E->nbox : E->GT.nrows,
                 tile_source(E->GT, E->PGT, E->PGT.np - 1, E->d_wpart_x), E->d_partT, E->capT,
                 fuse_beta(E)));
  CKL();
  return 0;
}

// Sharded engine: the rank's G_p^T y_hat_p partial sums over all of x-space
// (reduce-scattered afterwards) through the same column-panelled lane passes
// as the single-GPU G^T step, the last pass writing the raw partial product.
// Matrices with chunked long rows or tiled steps keep the generic SpMV.
template <int VW, int GP>
int lane_t_partial(Engine* E) {
  const SpmvPlan& P = E->GT;
  const PanelPlan& Q = E->PGT;
  if (lane_passes<VW, GP>(E, P, Q, E->d.d_yh, E->d_wpart_x, 2, E->keep_yh)) return 1;
  CK(launch_step(use_pdl(E), k_lane_pass<VW, GP>, P.pass_grid, E->stream,
                 tile_source(P, Q, Q.np - 1, E->d_wpart_x), P.nrows, (const double*)E->d.d_yh, E->d_gtp,
                 (const PdcsCtrl*)E->d_ctrl, 2, E->keep_yh));
  CKL();
  return 0;
}

int launch_gt_partial(Engine* E) {
  if (E->GT.n_long || E->tile_t || E->GT.nrows == 0)
    return launch_spmv(E->GT, E->d.d_yh, E->d_gtp, E->stream, E->d_ctrl, 2);
  switch (E->GT.step_vw * 2 + E->gp) {
    case 2: return lane_t_partial<1, 0>(E);
    case 3: return lane_t_partial<1, 1>(E);
    case 16: return lane_t_partial<8, 0>(E);
    case 17: return lane_t_partial<8, 1>(E);
    case 65: return lane_t_partial<32, 1>(E);
    default: return lane_t_partial<32, 0>(E);
  }
}

// class-split step: short rows thread per row, long rows cls_vw lanes per row,
// the product into `out`, then the streaming epilogue
int class_pass(Engine* E, const SpmvPlan& P, const double* x, double* out, int gate) {
  if (!P.n_cls_long) return 0;
  const PdcsCtrl* c = E->d_ctrl;
  auto fn = P.cls_vw == 32 ? k_rows_pass<32>
            : P.cls_vw == 16 ? k_rows_pass<16>
            : P.cls_vw == 4  ? k_rows_pass<4>
                             : k_rows_pass<8>;
  CK(launch_step(use_pdl(E), fn, P.cls_grid_l, E->stream, (const int*)P.d_cls_long, P.n_cls_long,
                 P.rowptr, P.colidx, (const double*)P.val, x, out, c, gate));
  CKL();
  return 0;
}

int class_y(Engine* E, const KArgs& A) {
  if (class_pass(E, E->G, E->d.d_xt, E->d.d_w, 1)) return 1;
  const ShortRows R{E->G.rowptr, E->G.colidx, E->G.val, E->d.d_xt};
  if (E->yblk_fused) {
    const BlockTable& T = E->tabY;
    const PdcsBlock* half = T.d_all + T.n_exp + T.n_thread;
    CK(launch_step(use_pdl(E), k_y_epi_blk<3>, E->G.grid, E->stream, A, E->d_partY, E->capY, R, half, T.n_half,
                   E->yblk_ga));
    CKL();
    return 0;
  }
  CK(launch_step(use_pdl(E), k_y_epi<false>, E->G.grid, E->stream, A, E->d_partY, E->capY, fuse_ls(E), R));
  CKL();
  return 0;
}

int class_t(Engine* E, const KArgs& A) {
  if (class_pass(E, E->GT, E->d.d_yh, E->d.d_gth, 2)) return 1;
  const ShortRows R{E->GT.rowptr, E->GT.colidx, E->GT.val, E->d.d_yh};
  if (E->vec && E->ubox && E->nbox == E->n)
    CK(launch_step(use_pdl(E), k_t_epi2, E->GT.grid, E->stream, A, E->d_partT, E->capT, fuse_beta(E), R));
  else
    CK(launch_step(use_pdl(E), k_t_epi<false>, E->GT.grid, E->stream, A, E->d_partT, E->capT, fuse_beta(E), R));
  CKL();
  return 0;
}

int launch_step_y(Engine* E, const KArgs& A) {
  if (E->cls_y) return class_y(E, A);
  if (E->split) return E->hs ? split_y<true>(E, A) : split_y<false>(E, A);
  if (E->tile_y) {
    if (launch_panel_passes(E, E->G, E->PG, E->d.d_xt, E->d_wpart_y, E->G.grid, 1)) return 1;
    const TileSrc src = tile_source(E->G, E->PG, E->PG.np - 1, E->d_wpart_y);
    if (E->soc_tile)
      k_step_y<true><<<E->G.grid, BS, 0, E->stream>>>(A, src, E->d_partY, E->capY, fuse_ls(E), E->d_rowhead);
    else
      k_step_y<false><<<E->G.grid, BS, 0, E->stream>>>(A, src, E->d_partY, E->capY, fuse_ls(E), nullptr);
    CKL();
    return 0;
  }
  switch (E->G.step_vw * 2 + E->gp) {
    case 2: return lane_y<1, 0>(E, A);
    case 3: return lane_y<1, 1>(E, A);
    case 16: return lane_y<8, 0>(E, A);
    case 17: return lane_y<8, 1>(E, A);
    case 65: return lane_y<32, 1>(E, A);
    default: return lane_y<32, 0>(E, A);
  }
}

int launch_step_t(Engine* E, const KArgs& A) {
  if (E->cls_t) return class_t(E, A);
  if (E->split) return E->hs ? split_t<true>(E, A) : split_t<false>(E, A);
  if (E->tile_t) {
    if (launch_panel_passes(E, E->GT, E->PGT, E->d.d_yh, E->d_wpart_x, E->GT.grid, 2)) return 1;
    k_step_t<<<E->GT.grid, BS, 0, E->stream>>>(A, tile_source(E->GT, E->PGT, E->PGT.np - 1, E->d_wpart_x),
                                               E->d_partT, E->capT, fuse_beta(E));
    CKL();
    return 0;
  }
  switch (E->GT.step_vw * 2 + E->gp) {
    case 2: return lane_t<1, 0>(E, A);
    case 3: return lane_t<1, 1>(E, A);
    case 16: return lane_t<8, 0>(E, A);
    case 17: return lane_t<8, 1>(E, A);
    case 65: return lane_t<32, 1>(E, A);
    default: return lane_t<32, 0>(E, A);
  }
}

// step-kernel lanes per row: 1 (short rows, index-order sums), 8 or 32
int step_lanes(int64_t nnz, int64_t nrows) {
  if (nrows <= 0) return 1;
  const double mean = (double)nnz / (double)nrows;
  return mean <= 6.0 ? 1 : (mean <= 64.0 ? 8 : 32);
}

// the lane-step kernel instance for (lanes per row, GP mode)
template <auto... K>
const void* lane_fn(int vw, int gp) {
  const void* fns[] = {(const void*)K...};
  const int row = vw == 1 ? 0 : (vw == 8 ? 1 : 2);
  return fns[row * 2 + (gp & 1)];
}

const void* pass_fn(int vw, int gp) {
  return lane_fn<k_lane_pass<1, 0>, k_lane_pass<1, 1>, k_lane_pass<8, 0>, k_lane_pass<8, 1>,
                 k_lane_pass<32, 0>, k_lane_pass<32, 1>>(vw, gp);
}

const void* step_y_fn(const Engine* E) {
  if (E->tile_y) return E->soc_tile ? (const void*)k_step_y<true> : (const void*)k_step_y<false>;
  return lane_fn<k_step_y_lane<1, 0>, k_step_y_lane<1, 1>, k_step_y_lane<8, 0>, k_step_y_lane<8, 1>,
                 k_step_y_lane<32, 0>, k_step_y_lane<32, 1>>(E->G.step_vw, E->gp);
}

const void* step_t_fn(const Engine* E) {
  if (E->tile_t) return (const void*)k_step_t;
  return lane_fn<k_step_t_lane<1, 0>, k_step_t_lane<1, 1>, k_step_t_lane<8, 0>, k_step_t_lane<8, 1>,
                 k_step_t_lane<32, 0>, k_step_t_lane<32, 1>>(E->GT.step_vw, E->gp);
}

// Panelled copy of a CSR pattern (values filled by refresh_panel_values).
int build_panels(PanelPlan& Q, const SpmvPlan& P, int np, cudaStream_t s) {
  Q = PanelPlan();
  Q.np = std::max(1, np);
  if (P.nrows == 0) {
    Q.np = 1;
    return 0;
  }
  if (P.ncols < Q.np) Q.np = std::max(1, P.ncols);
  Q.width = (P.ncols + Q.np - 1) / Q.np;
  const size_t nflat = (size_t)Q.np * P.nrows;
  int* cnt = nullptr;
  CK(cudaMallocAsync(&cnt, sizeof(int) * (nflat + 1), s));
  CK(cudaMemsetAsync(cnt, 0, sizeof(int) * (nflat + 1), s));
  CK(cudaMallocAsync(&Q.d_po, sizeof(int) * (nflat + 1), s));
  k_panel_count<<<grid_for(P.nrows), BS, 0, s>>>(P.nrows, P.rowptr, P.colidx, P.long_t, Q.np, Q.width, cnt);
  CKL();
  size_t tmp_bytes = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, Q.d_po, (int)(nflat + 1), s));
  void* tmp = nullptr;
  CK(cudaMallocAsync(&tmp, tmp_bytes, s));
  CK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, Q.d_po, (int)(nflat + 1), s));
  int total = 0;
  CK(cudaMemcpyAsync(&total, Q.d_po + nflat, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaFreeAsync(tmp, s));
  CK(cudaFreeAsync(cnt, s));
  CK(cudaStreamSynchronize(s));
  Q.nnz_short = total;
  // stream-ordered (pooled) allocations: a later engine's setup reuses them
  CK(cudaMallocAsync(&Q.d_pci, sizeof(int) * std::max(total, 1), s));
  CK(cudaMallocAsync(&Q.d_pperm, sizeof(int) * std::max(total, 1), s));
  CK(cudaMallocAsync(&Q.d_pva, sizeof(double) * std::max(total, 1), s));
  k_panel_scatter<<<grid_for(P.nrows), BS, 0, s>>>(P.nrows, P.rowptr, P.colidx, P.long_t, Q.np, Q.width,
                                                   Q.d_po, Q.d_pci, Q.d_pperm);
  CKL();
  CK(cudaStreamSynchronize(s));
  return 0;
}

int refresh_panel_values(const PanelPlan& Q, const double* val, cudaStream_t s) {
  if (Q.d_pva == nullptr || Q.nnz_short == 0) return 0;
  k_gather<<<grid_for(Q.nnz_short), BS, 0, s>>>(Q.d_pva, val, Q.d_pperm, Q.nnz_short);
  CKL();
  return 0;
}

void free_panels(PanelPlan& Q, cudaStream_t s) {
  if (Q.d_po) cudaFreeAsync(Q.d_po, s);
  if (Q.d_pci) cudaFreeAsync(Q.d_pci, s);
  if (Q.d_pva) cudaFreeAsync(Q.d_pva, s);
  if (Q.d_pperm) cudaFreeAsync(Q.d_pperm, s);
  Q = PanelPlan();
}

// Optional per-stage event markers for pdcs_profile_slot (never active while
// a graph is being captured).
struct StageProf {
  bool on = false;
  std::vector<cudaEvent_t> ev;
  std::vector<const char*> names;
} g_prof;

void mark(cudaStream_t s, const char* name) {
  if (!g_prof.on) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, s);
  g_prof.ev.push_back(e);
  g_prof.names.push_back(name);
}

int launch_slot(Engine* E) {
  const KArgs A = make_args(E);
  cudaStream_t s = E->stream;
  BlkParams none{nullptr, nullptr, nullptr, 0, -1};
  // primal candidate (pairs of coordinates per 16-byte access when the whole
  // x-space is one uniform box on one GPU)
  if (E->vec && E->ubox && E->nbox == E->n && !E->comm && !E->xsplit) {
    CK(launch_step(use_pdl(E), k_step_x2, E->gridStepX2, s, A, E->d_partX, E->capX));
  } else if (E->xexp_fused) {  // the cone coordinates are stepped by k_exp_xstep
    KArgs Ab = A;
    Ab.x1 = std::min(A.x1, E->nbox);
    CK(launch_step(use_pdl(E), k_step_x<false>, E->gridStepX, s, Ab, E->d_partX, E->capX));
  } else {
    CK(launch_step(use_pdl(E), k_step_x<false>, E->gridStepX, s, A, E->d_partX, E->capX));
  }
  CKL();
  mark(s, "step_x");
  // x-space cone blocks this engine steps (its slice's blocks when sharded)
  const BlockTable& TX = E->xsplit ? E->tabXs : E->tabX;
  const bool xblk = TX.total() > 0;
  if (E->comm && E->nranks > 1 && !E->xsplit) {
    g_err = "sharded engine: pdcs_engine_set_xsplit is required with more than one rank";
    return 2;
  }
  if (E->xexp_fused) {
    k_exp_xstep<4><<<TX.g_exp, BS, 0, s>>>(TX.d_all, TX.n_exp, A, E->d_partX, E->capX, E->gridStepX);
    CKL();
  } else if (xblk && launch_blocks<OP_STEP_X>(TX, A, none, E->d_partX, E->capX, E->gridStepX, 1, s)) {
    return 1;
  }
  if (xblk) mark(s, "blocks_x");
  if (E->comm) {
    // sharded: every rank stepped its x-slice; G_p x~ needs all of x~
    if (nccl_x_allgather(E, E->d.d_xt, s)) return 1;
    mark(s, "allgather_xt");
  }
  // dual candidate with w = G^ x~
  if (E->G.n_long && launch_long(E->G, E->d.d_xt, E->d.d_w, E->d_ctrl, 1, s)) return 1;
  if (E->G.n_long) mark(s, "long_rows_g");
  int rc = 0;
  rc = launch_step_y(E, A);
  if (rc) return 1;
  mark(s, "step_y_spmv");
  // else projected inside the tiled y-step (soc_tile) or the class-split epilogue (yblk_fused)
  const bool yblk = E->has_yblocks && !E->soc_tile && !E->yblk_fused;
  if (E->exp_fused) {  // the exp rows' y-step inside the block kernel (k_exp_ystep)
    const ShortRows R{E->G.rowptr, E->G.colidx, E->G.val, E->d.d_xt};
    auto fn = E->tabY.exp_minb == 3 ? k_exp_ystep<3> : (E->tabY.exp_minb == 2 ? k_exp_ystep<2> : k_exp_ystep<4>);
    fn<<<E->tabY.g_exp, BS, 0, s>>>(E->tabY.d_all, E->tabY.n_exp, A, R, E->d_partY, E->capY, E->G.grid);
    CKL();
  } else if (yblk && launch_blocks<OP_STEP_Y>(E->tabY, A, none, E->d_partY, E->capY, E->G.grid, 1, s)) {
    return 1;
  }
  if (yblk) mark(s, "blocks_y");
  if (E->comm) {
    // sharded: the five y-space and three x-space line-search sums over all
    // ranks (each rank holds a row slice and an x-slice)
    k_finalize<<<1, BS, 0, s>>>(E->d_partY, E->capY, E->capY, GY_N, 0u, E->d_yred);
    CKL();
    k_finalize<<<1, BS, 0, s>>>(E->d_partX, E->capX, E->capX, GX_N, 0u, E->d_yred + GY_N);
    CKL();
    if (nccl_allreduce(E->d_yred, E->d_yred, GY_N + GX_N, E->comm, s)) return 1;
    mark(s, "allreduce_xy");
  }
  if (!fuse_ls(E).mode) {
    k_ctrl_ls<<<1, 1024, 0, s>>>(E->d_ctrl, E->d_partX, E->capX, E->d_partY, E->capY, E->d_red,
                               E->comm ? E->d_yred : nullptr);
    CKL();
    mark(s, "ctrl_linesearch");
  }
  // accepted: G^T y_hat, beta, Halpern coefficients
  if (E->comm) {
    // sharded: local G_p^T y_hat_p partial sums over all of x-space,
    // reduce-scattered so each rank gets its x-slice of G^T y_hat, then the
    // x-space epilogue on that slice
    if (launch_gt_partial(E)) return 1;
    mark(s, "step_t_partial");
    if (nccl_x_reduce_scatter(E, E->d_gtp, E->d.d_gth, s)) return 1;
    mark(s, "reduce_scatter_gty");
    k_t_epilogue<<<E->GT.grid, BS, 0, s>>>(A, E->d_partT, E->capT);
    CKL();
    mark(s, "step_t_epilogue");
  } else {
    if (E->GT.n_long && launch_long(E->GT, E->d.d_yh, E->d.d_gtr, E->d_ctrl, 2, s)) return 1;
    if (E->GT.n_long) mark(s, "long_rows_gt");
    rc = launch_step_t(E, A);
    if (rc) return 1;
    mark(s, "step_t_spmv");
  }
  if (E->texp_fused && !E->comm) {  // sharded: G^T y_hat comes from the reduce-scatter
    const ShortRows R{E->GT.rowptr, E->GT.colidx, E->GT.val, E->d.d_yh};
    k_exp_tstep<4><<<TX.g_exp, BS, 0, s>>>(TX.d_all, TX.n_exp, A, R, E->d_partT, E->capT, E->GT.grid);
    CKL();
  } else if (xblk && launch_blocks<OP_TLAM>(TX, A, none, E->d_partT, E->capT, E->GT.grid, 2, s)) {
    return 1;
  }
  if (xblk) mark(s, "blocks_t");
  const double* tred = nullptr;
  if (E->comm) {
    // sharded: the three x-space beta sums over all ranks, plus the ranks'
    // projection error codes, so every rank takes the same stop decision
    k_finalize<<<1, BS, 0, s>>>(E->d_partT, E->capT, E->capT, GT_N, 0u, E->d_yred + 8);
    CKL();
    k_err_to_double<<<1, 1, 0, s>>>(E->d_err, E->d_yred + 8 + GT_N);
    CKL();
    if (nccl_allreduce(E->d_yred + 8, E->d_yred + 8, GT_N + 1, E->comm, s)) return 1;
    mark(s, "allreduce_t");
    tred = E->d_yred + 8;
  }
  if (!fuse_beta(E).mode) {
    k_ctrl_beta<<<1, 1024, 0, s>>>(E->d_ctrl, E->d_partT, E->capT, E->d_red, E->d_err, tred);
    CKL();
    mark(s, "ctrl_beta");
  }
  return 0;
}

int finalize_to_host(Engine* E, const double* part, int cap, int nslots, int nq, unsigned mask,
                     double* h_out) {
  k_finalize<<<1, BS, 0, E->stream>>>(part, cap, nslots, nq, mask, E->d_out);
  CKL();
  CK(cudaMemcpyAsync(E->h_pinned, E->d_out, sizeof(double) * nq, cudaMemcpyDeviceToHost, E->stream));
  CK(cudaStreamSynchronize(E->stream));
  std::memcpy(h_out, E->h_pinned, sizeof(double) * nq);
  return 0;
}

}  // namespace

struct PdcsEngine : public Engine {};

// =============================================================================
// C ABI
// =============================================================================
extern "C" {

const char* pdcs_last_error(void) { return g_err.c_str(); }
int pdcs_abi_version(void) { return PDCS_ABI_VERSION; }
int64_t pdcs_launch_count(void) { return g_launches.load(); }

int pdcs_spmv_csr(int32_t nrows, const int32_t* d_rowptr, const int32_t* d_colidx,
                  const double* d_val, const double* d_x, double* d_y, void* stream) {
  if (nrows < 0) { g_err = "pdcs_spmv_csr: negative nrows"; return 2; }
  if (nrows == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  SpmvPlan P;
  int nnz = 0;
  CK(cudaMemcpyAsync(&nnz, d_rowptr + nrows, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (build_plan(P, nrows, 0, nnz, d_rowptr, d_colidx, d_val, s)) return 1;
  int rc = launch_spmv(P, d_x, d_y, s);
  CK(cudaStreamSynchronize(s));
  free_plan(P);
  return rc;
}

int pdcs_transpose_csr(int32_t nrows, int32_t ncols, int32_t nnz, const int32_t* d_rowptr,
                       const int32_t* d_colidx, const double* d_val, int32_t* d_t_rowptr,
                       int32_t* d_t_colidx, double* d_t_val, int32_t* d_perm, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (nrows < 0 || ncols < 0 || nnz < 0) { g_err = "pdcs_transpose_csr: bad sizes"; return 2; }
  int* cnt = nullptr;
  CK(cudaMallocAsync(&cnt, sizeof(int) * (ncols + 1), s));
  CK(cudaMemsetAsync(cnt, 0, sizeof(int) * (ncols + 1), s));
  if (nnz > 0) {
    int *rowid = nullptr, *keys_out = nullptr, *idx = nullptr;
    CK(cudaMallocAsync(&rowid, sizeof(int) * nnz, s));
    CK(cudaMallocAsync(&keys_out, sizeof(int) * nnz, s));
    CK(cudaMallocAsync(&idx, sizeof(int) * nnz, s));
    k_iota_rows<<<grid_for(nrows), BS, 0, s>>>(d_rowptr, nrows, rowid);
    CKL();
    k_iota<<<grid_for(nnz), BS, 0, s>>>(idx, nnz);
    CKL();
    k_count_cols<<<grid_for(nnz), BS, 0, s>>>(d_colidx, nnz, cnt);
    CKL();
    int bits = 1;
    while ((1ll << bits) < (int64_t)ncols + 1 && bits < 31) ++bits;
    size_t tmp_bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, d_colidx, keys_out, idx, d_perm, nnz, 0,
                                       bits, s));
    void* tmp = nullptr;
    CK(cudaMallocAsync(&tmp, tmp_bytes, s));
    CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, d_colidx, keys_out, idx, d_perm, nnz, 0, bits,
                                       s));
    k_transpose_scatter<<<grid_for(nnz), BS, 0, s>>>(d_perm, rowid, d_val, nnz, d_t_colidx, d_t_val);
    CKL();
    CK(cudaFreeAsync(tmp, s));
    CK(cudaFreeAsync(rowid, s));
    CK(cudaFreeAsync(keys_out, s));
    CK(cudaFreeAsync(idx, s));
  }
  size_t scan_bytes = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, cnt, d_t_rowptr, ncols + 1, s));
  void* scan_tmp = nullptr;
  CK(cudaMallocAsync(&scan_tmp, scan_bytes, s));
  CK(cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, cnt, d_t_rowptr, ncols + 1, s));
  CK(cudaFreeAsync(scan_tmp, s));
  CK(cudaFreeAsync(cnt, s));
  CK(cudaStreamSynchronize(s));
  return 0;
}

int pdcs_project_segments(int32_t len, const double* d_in, double* d_out, const PdcsBlock* h_blocks,
                          int32_t nblocks, const double* d_scale, int32_t* h_err, void* stream) {
  return pdcs_project_segments_ex(len, d_in, d_out, h_blocks, nblocks, d_scale, 1e-12, 100, h_err,
                                  stream);
}

int pdcs_project_segments_ex(int32_t len, const double* d_in, double* d_out, const PdcsBlock* h_blocks,
                             int32_t nblocks, const double* d_scale, double root_tol,
                             int32_t max_root_iters, int32_t* h_err, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!(root_tol >= 0.0) || max_root_iters < 1) {
    g_err = "pdcs_project_segments_ex: root_tol must be >= 0 and max_root_iters >= 1";
    return 2;
  }
  if (len < 0 || nblocks < 0) { g_err = "pdcs_project_segments: bad sizes"; return 2; }
  for (int i = 0; i < nblocks; ++i) {
    const PdcsBlock& b = h_blocks[i];
    if (b.start < 0 || b.dim < 1 || b.start + b.dim > len || b.kind < 0 || b.kind > 5) {
      g_err = "pdcs_project_segments: block out of range";
      return 2;
    }
    if (b.smode != PDCS_SCALE_NONE && d_scale == nullptr) {
      g_err = "pdcs_project_segments: scaled block without a scale vector";
      return 2;
    }
  }
  if (len > 0 && d_in != d_out)
    CK(cudaMemcpyAsync(d_out, d_in, sizeof(double) * len, cudaMemcpyDeviceToDevice, s));
  int* d_err = nullptr;
  CK(cudaMalloc(&d_err, sizeof(int)));
  CK(cudaMemsetAsync(d_err, 0, sizeof(int), s));
  BlockTable T;
  if (build_table(T, std::vector<PdcsBlock>(h_blocks, h_blocks + nblocks), s)) return 1;
  KArgs A;
  std::memset(&A, 0, sizeof(A));
  A.err = d_err;
  BlkParams P{d_out, d_out, d_scale, 0, -1};
  P.rc.tol = root_tol;
  P.rc.iters = max_root_iters;
  int rc = launch_blocks<OP_PROJECT>(T, A, P, nullptr, 0, 0, 0, s);
  int herr = 0;
  CK(cudaMemcpyAsync(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (h_err) *h_err = herr;
  cudaFree(d_err);
  cudaFree(T.d_all);
  return rc;
}

int pdcs_engine_create(const PdcsEngineDesc* desc, void* stream, PdcsEngine** out) {
  if (!desc || !out) { g_err = "pdcs_engine_create: null argument"; return 2; }
  const PdcsEngineDesc& d = *desc;
  if (d.n < 0 || d.m < 0 || d.nnz < 0 || d.num_box < 0 || d.num_box > d.n || d.m_zero < 0 ||
      d.m_zero > d.m_elem || d.m_elem > d.m) {
    g_err = "pdcs_engine_create: inconsistent sizes";
    return 2;
  }
  PdcsEngine* E = new PdcsEngine();
  E->d = d;
  E->stream = (cudaStream_t)stream;
  E->n = d.n; E->m = d.m; E->nbox = d.num_box; E->nnz = d.nnz;
  E->xs0 = 0; E->xs1 = d.n;
  E->m_zero = d.m_zero; E->m_elem = d.m_elem;
  E->allow_nonuniform_dual_soc = d.allow_nonuniform_dual_soc;
  cudaStream_t s = E->stream;
  auto fail = [&](int rc) { pdcs_engine_destroy(E); return rc; };
  PhaseTimer T("create", s);
  {
    // setup temporaries are stream-ordered allocations (cudaMallocAsync): keep
    // up to 4 GB of them pooled so a later engine's setup reuses the mapping
    // (cudaMalloc / cudaFree of the same buffers cost tens of ms and a device sync)
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = (uint64_t)(tune_env("pool_gb", 4.0) * (double)(1ull << 30));
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
  }

  // cone tables: primal blocks start after the box; dual blocks beyond m_elem
  std::vector<PdcsBlock> xb, yb, ux, uy;
  int pos = d.num_box;
  for (int i = 0; i < d.n_pcones; ++i) {
    const int k = d.h_pcone_kind[i], dim = d.h_pcone_dim[i];
    if (k < 1 || k > 5 || dim < 1) { g_err = "pdcs_engine_create: bad primal cone"; return fail(2); }
    xb.push_back(PdcsBlock{k, pos, dim, PDCS_SCALE_DIRECT});
    if (k == PDCS_EXP || k == PDCS_DUAL_EXP) ux.push_back(PdcsBlock{k, pos, dim, 0});
    pos += dim;
  }
  if (pos != d.n) { g_err = "pdcs_engine_create: primal cone dims do not sum to n - num_box"; return fail(2); }
  pos = 0;
  for (int i = 0; i < d.n_dcones; ++i) {
    const int k = d.h_dcone_kind[i], dim = d.h_dcone_dim[i];
    if (k < 1 || k > 5 || dim < 1) { g_err = "pdcs_engine_create: bad dual cone"; return fail(2); }
    if (k == PDCS_ZERO || k == PDCS_NONNEG) {
      if (pos >= d.m_elem && dim > 0) { g_err = "pdcs_engine_create: elementwise dual block after cone blocks"; return fail(2); }
    } else {
      if (pos < d.m_elem) { g_err = "pdcs_engine_create: cone block inside the elementwise rows"; return fail(2); }
      yb.push_back(PdcsBlock{k, pos, dim, PDCS_SCALE_DIRECT});
      if (k == PDCS_EXP || k == PDCS_DUAL_EXP || (k == PDCS_SOC && !d.allow_nonuniform_dual_soc))
        uy.push_back(PdcsBlock{k, pos, dim, 0});
    }
    pos += dim;
  }
  if (pos != d.m) { g_err = "pdcs_engine_create: dual cone dims do not sum to m"; return fail(2); }
  // blocks up to thread_max rows (default 4) get one thread each, the next class 4-lane
  // groups (half_w): measured better than a thread per SOC(11) block (C2 10.1k, C2p 3.5k it/s)
  // and than 16-lane groups.  PDCS_TUNE thread_max=N / xthread_max=N override.
  const int ythr = (int)tune_env("thread_max", (double)THREAD_CLASS_MAX);
  const int xthr = (int)tune_env("xthread_max", (double)THREAD_CLASS_MAX);
  if (build_table(E->tabX, xb, s, false, xthr) ||
      build_table(E->tabY, yb, s, !d.allow_nonuniform_dual_soc, ythr))
    return fail(1);
  E->xblocks = xb;
  E->has_xblocks = E->tabX.total() > 0;
  E->tabY.half_minb = (int)tune_env("halfminb", 3.0);
  E->tabX.half_minb = (int)tune_env("xhalfminb", 3.0);
  // 4 lanes per block of 5-16 rows: C2 10.6k it/s vs 10.1k (a thread per block) and 9.7k
  // (16 lanes); C2p 5.9k vs 5.3k (profiles/r02_sweeps.txt)
  E->tabY.half_w = (int)tune_env("halfw", 4.0);
  E->tabX.half_w = (int)tune_env("xhalfw", 4.0);
  if (E->tabY.n_exp) {  // Newton warm starts of the dual exp blocks, NaN = cold
    const size_t cnt = 2 * (size_t)E->tabY.n_exp;
    if (cudaMalloc(&E->d_exp_rho, sizeof(double) * cnt) != cudaSuccess) return fail(1);
    // fast / slow split of the y-step exp blocks (PDCS_TUNE=expsplit=1).  Off by
    // default: measured slower on C3 (blocks_y 0.146-0.172 ms vs 0.135 ms in
    // one kernel, 2.27-2.41k vs 2.75k it/s; profiles/r02_sweeps.txt)
    const char* env = getenv("PDCS_TUNE");
    const bool on = env && (strstr(env, "expsplit=1") != nullptr);
    const char* mb = env ? strstr(env, "expminb=") : nullptr;
    E->tabY.exp_minb = mb ? atoi(mb + 8) : 4;
    if (on) {
      BlockTable& T = E->tabY;
      T.exp_split = true;
      T.exp_per = (T.n_exp + T.g_exp - 1) / T.g_exp;
      if (cudaMalloc(&T.d_queue, sizeof(int) * T.n_exp) != cudaSuccess ||
          cudaMalloc(&T.d_qcount, sizeof(int) * T.g_exp) != cudaSuccess)
        return fail(1);
    }
    std::vector<double> nan_init(cnt, NAN);
    if (cudaMemcpyAsync(E->d_exp_rho, nan_init.data(), sizeof(double) * cnt, cudaMemcpyHostToDevice,
                        s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return fail(1);
  }
  E->has_yblocks = E->tabY.total() > 0;
  auto upload_blocks = [&](const std::vector<PdcsBlock>& v, PdcsBlock** dst) -> int {
    if (v.empty()) return 0;
    CK(cudaMalloc(dst, sizeof(PdcsBlock) * v.size()));
    CK(cudaMemcpyAsync(*dst, v.data(), sizeof(PdcsBlock) * v.size(), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    return 0;
  };
  if (upload_blocks(ux, &E->d_unif_x) || upload_blocks(uy, &E->d_unif_y)) return fail(1);
  E->n_unif_x = (int)ux.size();
  E->n_unif_y = (int)uy.size();

  T.lap("cone tables");
  // transpose of the pattern (values are written by pdcs_precondition)
  if (pdcs_transpose_csr(d.m, d.n, d.nnz, d.d_g_rowptr, d.d_g_colidx, nullptr, d.d_gt_rowptr,
                         d.d_gt_colidx, nullptr, d.d_perm, s))
    return fail(1);
  T.lap("transpose");
  if (build_plan(E->G, d.m, d.n, d.nnz, d.d_g_rowptr, d.d_g_colidx, d.d_g_val, s)) return fail(1);
  if (build_plan(E->GT, d.n, d.m, d.nnz, d.d_gt_rowptr, d.d_gt_colidx, d.d_gt_val, s)) return fail(1);
  T.lap("spmv plans");

  // grids and reduction capacities: the streaming step kernels get exactly one
  // wave of resident CTAs (grid-stride loops), the rest a capped grid
  E->gridX = grid_for(d.n);
  E->gridY = grid_for(d.m);
  {
    int dev = 0, nsm = NSM, l2 = 126 << 20;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    // PDCS_TUNE="py=3,pt=2,panel_mb=48,gx=8,gy=5,gt=6" overrides (panels of the
    // G^ / G^T step SpMVs, gathered-slice budget, CTAs per SM of step kernels)
    auto tune = [](const char* key, double dflt) { return tune_env(key, dflt); };
    // Column panels: cut the gathered vector into slices of at most ~0.42 L2.
    // Random 8-byte gathers stay L2-rate bound only while their footprint is
    // below ~50 MB on B200 (tools/gather_probe.cu: 267 G/s up to 48 MB, 196 at
    // 80 MB, 90 at 160 MB); each extra panel costs a partial-sum round trip.
    // C5 measured best at 3 panels for G^ x~ (160 MB) and 2 for G^T y_hat
    // (80 MB): 692 it/s against 684 with 4 and 2 (profiles/r01_sweeps.txt).
    const double budget = tune("panel_mb", 0.42 * l2 / 1048576.0) * 1048576.0;
    auto panels_for = [&](int ncols, int nrows, int nnz) {
      if (nnz < (1 << 20)) return 1;  // small matrices: the whole vector is L2-resident
      int np = (int)std::ceil(8.0 * ncols / budget);
      return std::max(1, std::min(np, 16));
    };
    const int py = (int)tune("py", panels_for(d.n, d.m, d.nnz));
    const int pt = (int)tune("pt", panels_for(d.m, d.n, d.nnz));
    if (build_panels(E->PG, E->G, py, s) || build_panels(E->PGT, E->GT, pt, s)) return fail(1);
    T.lap("panels");
    // gp=1: gathers of the lane-mapped step SpMVs fetch 64 B into L2 (PTX
    // L2::64B).  Measured slower on C5, as were two rows per thread and
    // loading the epilogue operands ahead of the gathers (profiles/r01_sweeps.txt).
    E->gp = (int)tune("gp", 0.0) & 1;
    E->fuse_ctrl = tune("fuse", 1.0) > 0.0;
    // pdl=0: the step kernels of a trial are ordinary stream-ordered launches
    E->pdl = tune("pdl", 1.0) > 0.0;
    E->G.step_vw = step_lanes(E->PG.nnz_short / std::max(1, E->PG.np), d.m);
    E->GT.step_vw = step_lanes(E->PGT.nnz_short / std::max(1, E->PGT.np), d.n);
    auto lanes_knob = [&](const char* key, int dflt) {  // 1, 8 or 32 lanes per row
      const int v = (int)tune(key, (double)dflt);
      return v == 1 || v == 8 || v == 32 ? v : dflt;
    };
    E->G.step_vw = lanes_knob("vwy", E->G.step_vw);
    E->GT.step_vw = lanes_knob("vwt", E->GT.step_vw);
    // Measured (profiles/r01_sweeps.txt): thread-per-row lanes win for short
    // rows (C3, C5); 8 lanes per row win for uniform rows of ~40 (C4's and
    // C2's G^T: 5.1k -> 5.7k and 8.8k -> 9.2k it/s); the tiled CSR-stream
    // kernel wins for long-ish rows of very mixed length (C2's G: rows of 1-2
    // and of ~48 entries).
    const double big = d.nnz >= (1 << 20) ? 1.0 : 0.0;
    // G^ x~ rows of mixed length: tiles (C2: 0.044 vs 0.047 ms); G^T y_hat: 8 lanes
    // even for mixed rows (C2: 0.032 vs 0.048 ms), tiles only where 32 lanes
    // would be needed
    E->tile_y = tune("tile_y", tune("tile", big * (E->G.step_vw > 1 && E->G.len_cv > 0.5))) > 0.0;
    E->tile_t = tune("tile_t", tune("tile", big * (E->GT.step_vw == 32))) > 0.0;
    // dual SOC blocks projected inside the tiled y-step (C2 class): uniform
    // dual scales, only SOC blocks of at most one tile, no chunked long rows
    // Opt-in (PDCS_TUNE socfuse=1): measured equal on C2 (8704 vs 8701 it/s; the fused
    // k_step_y<1> takes 70 us against 43 + 22 + 12 us unfused), profiles/r02_sweeps.txt
    bool soc_tile = E->tile_y && tune("socfuse", 0.0) > 0.0 && !d.allow_nonuniform_dual_soc &&
                    E->tabY.total() > 0 && E->tabY.n_exp == 0 && E->tabY.n_giant == 0 && E->G.n_long == 0;
    std::vector<int> head;
    if (soc_tile) {
      head.assign(d.m, -1);
      for (const PdcsBlock& b : yb) {
        if (b.kind != PDCS_SOC || b.dim > TILE_ROWS) { soc_tile = false; break; }
        for (int r = b.start; r < b.start + b.dim; ++r) head[r] = b.start;
      }
    }
    if (soc_tile) {
      const int rc = build_tiles(E->G, s, &head);
      if (rc == 4) {
        soc_tile = false;
        cudaFree(E->G.d_tiles);
        E->G.d_tiles = nullptr;
      } else if (rc) {
        return fail(1);
      }
    }
    if (soc_tile) {
      if (cudaMalloc(&E->d_rowhead, sizeof(int) * std::max(d.m, 1)) != cudaSuccess ||
          cudaMemcpyAsync(E->d_rowhead, head.data(), sizeof(int) * d.m, cudaMemcpyHostToDevice, s) !=
              cudaSuccess ||
          cudaStreamSynchronize(s) != cudaSuccess)
        return fail(1);
      E->soc_tile = true;
    }
    if ((E->tile_y && !E->soc_tile && build_tiles(E->G, s)) || (E->tile_t && build_tiles(E->GT, s)))
      return fail(1);
    T.lap("tiles");
    if (E->PG.np > 1 && cudaMallocAsync(&E->d_wpart_y, sizeof(double) * std::max(d.m, 1), s) != cudaSuccess)
      return fail(1);
    if (E->PGT.np > 1 && cudaMallocAsync(&E->d_wpart_x, sizeof(double) * std::max(d.n, 1), s) != cudaSuccess)
      return fail(1);
    auto fit = [&](const void* fn, int needed) {
      int occ = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, BS, 0) != cudaSuccess || occ < 1) occ = 1;
      return std::max(1, std::min(needed, occ * nsm));
    };
    auto grid_per_sm = [&](const char* key, int needed, int dflt) {
      const int per = (int)tune(key, 0.0);
      return per > 0 ? std::max(1, std::min(needed, per * nsm)) : dflt;
    };
    E->gridStepX = grid_per_sm("gx", E->gridX, fit((const void*)k_step_x<false>, E->gridX));
    E->gridStepX2 = std::min(E->gridStepX, fit((const void*)k_step_x2, grid_for(d.n / 2 + 1)));
    const int need_y = E->tile_y ? std::max(1, E->G.ntiles) : grid_for(d.m, BS / E->G.step_vw, 1 << 30);
    const int need_t = E->tile_t ? std::max(1, E->GT.ntiles) : grid_for(d.n, BS / E->GT.step_vw, 1 << 30);
    E->G.grid = grid_per_sm("gy", need_y, fit(step_y_fn(E), need_y));
    E->GT.grid = grid_per_sm("gt", need_t, fit(step_t_fn(E), need_t));
    // split step: thread-per-row gather-only passes + streaming epilogues
    // (single GPU, no chunked long rows, lane-mapped thread-per-row steps);
    // the epilogue kernels take the step kernels' reduction slots
    // Measured on C5 (profiles/r02_sweeps.txt): split + hs 704 it/s vs 682 fused
    // (step_y 0.520 vs 0.555 ms, step_t 0.467 vs 0.506 ms); default on where it applies
    E->split = tune("split", 1.0) > 0.0 && E->G.n_long == 0 && E->GT.n_long == 0 && !E->tile_y &&
               !E->tile_t && E->G.step_vw == 1 && E->GT.step_vw == 1 && E->gp == 0 &&
               E->PG.np > 1 && E->PGT.np > 1;
    E->hs = tune("hs", 1.0) > 0.0;
    E->vec = tune("vec", 1.0) > 0.0;  // double2 streaming epilogues (split step only)
    if (E->split) {
      const void* ye = (E->vec && d.m_elem == d.m) ? (const void*)k_y_epi2 : (const void*)k_y_epi<false>;
      // one wave of the epilogue kernel that will run (k_t_epi2 also needs the uniform box,
      // known after create; without it k_t_epi runs on the same grid)
      const int ny = grid_for(d.m, BS, 1 << 30), nx = grid_for(d.n, BS, 1 << 30);
      E->G.grid = grid_per_sm("gy", ny, fit(ye, ny));
      E->GT.grid = grid_per_sm("gt", nx, E->vec ? fit((const void*)k_t_epi2, nx)
                                                : fit((const void*)k_t_epi<false>, nx));
    }
    // class split (one panel, no chunked long rows; PDCS_TUNE cls=0 off): rows of
    // > 6 entries 8/16/32 lanes per row, then the streaming epilogue, which sums
    // the short rows itself.  Taken when the long class holds at least half of
    // the entries (cls_frac): C2's G and G^T (+7%), C4's G^T of 42-entry rows;
    // mostly-short matrices keep the fused lane kernels (C5's pattern at 1/10:
    // 6.3k vs 6.8k it/s with the class split of its G^T)
    {
      const bool cls_on = tune("cls", 1.0) > 0.0;
      const double cls_nnz = tune("cls_nnz", (double)(1 << 20)), cls_frac = tune("cls_frac", 0.5);
      auto classes = [&](SpmvPlan& P, const PanelPlan& Q, bool& on) {
        if (!cls_on || E->split || P.n_long != 0 || Q.np != 1 || (double)d.nnz < cls_nnz || P.nnz == 0) return 0;
        if (build_classes(P, s, nsm)) return 1;
        if ((double)P.nnz_cls_long >= cls_frac * (double)P.nnz) {
          on = true;
        } else {
          cudaFree(P.d_cls_long);
          P.d_cls_long = nullptr;
          P.n_cls_long = 0;
        }
        return 0;
      };
      if (classes(E->G, E->PG, E->cls_y)) return fail(1);
      if (classes(E->GT, E->PGT, E->cls_t)) return fail(1);
      if (E->cls_y) {
        const int ny = grid_for(d.m, BS, 1 << 30);
        E->G.grid = grid_per_sm("gy", ny, fit((const void*)k_y_epi<false>, ny));
        // dual cone blocks all of the half-warp class (C2's SOC(11)): projected inside the
        // epilogue kernel.  Opt-in (PDCS_TUNE yblkfuse=1): measured equal on C2 (9.5-9.8k vs
        // 9.6k it/s; profiles/r02_sweeps.txt) -- the block work, not the launch, is the cost
        const BlockTable& T = E->tabY;
        if (tune("yblkfuse", 0.0) > 0.0 && T.n_half > 0 && T.n_half == T.total() && T.n_giant == 0) {
          int occ = 1;
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_y_epi_blk<3>, BS, 0);
          const int slots = std::max(2, occ * nsm);
          const int need_a = std::max(1, grid_for(d.m_elem, BS, 1 << 30));
          const int need_b = std::max(1, grid_for((long long)T.n_half * 16, BS, 1 << 30));
          // one wave, the SM slots split in proportion to the two parts' threads
          int ga = (int)std::max(1LL, std::min<long long>(need_a, (long long)slots * need_a / (need_a + need_b)));
          int gb = std::max(1, std::min(need_b, slots - ga));
          E->yblk_fused = true;
          E->yblk_ga = ga;
          E->G.grid = ga + gb;
        }
      }
      if (E->cls_t) {
        const int nx = grid_for(d.n, BS, 1 << 30);
        E->GT.grid = grid_per_sm("gt", nx, E->vec ? fit((const void*)k_t_epi2, nx)
                                                  : fit((const void*)k_t_epi<false>, nx));
      }
    }
    // primal exp coordinates' x-step in the exp block kernel (PDCS_TUNE xexpfuse=0 off):
    // every primal block exponential (single GPU: the sharded x-slice tables differ)
    {
      const BlockTable& T = E->tabX;
      E->xexp_fused = tune("xexpfuse", 1.0) > 0.0 && T.n_exp > 0 && T.n_exp == T.total();
      // ... and their G^T rows + lambda_2 projection (lane-mapped single-panel t-step)
      E->texp_fused = E->xexp_fused && tune("texpfuse", 1.0) > 0.0 && !E->cls_t && !E->split && !E->tile_t &&
                      E->PGT.np == 1 && E->GT.n_long == 0;
    }
    // exp-cone rows' y-step in the exp block kernel (PDCS_TUNE expfuse=0 off): lane-mapped
    // single-panel y-step, dual blocks all exponential, long rows only among the elementwise rows
    {
      const BlockTable& T = E->tabY;
      if (tune("expfuse", 1.0) > 0.0 && !E->cls_y && !E->split && !E->tile_y && E->PG.np == 1 && T.n_exp > 0 &&
          T.n_exp == T.total() && d.m_elem < d.m && !T.exp_split) {
        E->exp_fused = true;
      }
    }
    // the partial-sum passes are latency bound (dependent rowptr -> col ->
    // gather chains): they get every warp slot their registers allow
    const int need_py = grid_for(d.m, BS / E->G.step_vw, 1 << 30);
    const int need_pt = grid_for(d.n, BS / E->GT.step_vw, 1 << 30);
    E->G.pass_grid = grid_per_sm("gpass", need_py, fit(pass_fn(E->G.step_vw, E->gp), need_py));
    E->GT.pass_grid = grid_per_sm("gpass", need_pt, fit(pass_fn(E->GT.step_vw, E->gp), need_pt));
    // optional persisting-L2 set-aside (evict_last lines only persist inside it)
    int max_persist = 0;
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    size_t want = (size_t)(tune("persist_mb", 0.0) * 1048576.0);
    if (want > (size_t)max_persist) want = (size_t)max_persist;
    if (want > 0 && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess)
      E->l2_persist = want;
    E->keep_xt = (float)tune("keep_xt", 1.0);
    E->keep_yh = (float)tune("keep_yh", 1.0);
    cudaGetLastError();
  }
  {
    // persistent trials (k_persist) for small block-free instances on one GPU:
    // C1 class (launch-latency bound); PDCS_TUNE persist=0 keeps the graph path
    const char* env = getenv("PDCS_TUNE");
    const bool off = env && strstr(env, "persist=0");
    const bool vw_ok = [](int v) { return v == 1 || v == 8 || v == 32; }(E->G.step_vw) &&
                       [](int v) { return v == 1 || v == 8 || v == 32; }(E->GT.step_vw);
    int coop = 0, dev = 0, nsm = NSM;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (!off && coop && vw_ok && !E->has_xblocks && !E->has_yblocks && E->G.n_long == 0 &&
        E->GT.n_long == 0 && E->PG.np == 1 && E->PGT.np == 1 && !E->tile_y && !E->tile_t && !E->split &&
        d.nnz <= (1 << 22) && d.n > 0 && d.m > 0) {
      // one CTA per SM: measured best for one C1 solve (55.3k it/s against 51.4k at 74
      // CTAs, 38.7k at 37, 27.9k at 18; profiles/r02_sweeps.txt).  Concurrent small
      // solves belong in batch.solve_many (one graph for all), not in host threads
      // each launching a whole-GPU cooperative kernel.  PDCS_TUNE pgrid=N overrides.
      const char* pg = env ? strstr(env, "pgrid=") : nullptr;
      E->pgrid = pg ? std::max(1, std::min(nsm, atoi(pg + 6))) : nsm;
      if (cudaMalloc(&E->d_pX, sizeof(double) * GX_N * E->pgrid) == cudaSuccess &&
          cudaMalloc(&E->d_pY, sizeof(double) * GY_N * E->pgrid) == cudaSuccess &&
          cudaMalloc(&E->d_pT, sizeof(double) * GT_N * E->pgrid) == cudaSuccess)
        E->persist = true;
      cudaGetLastError();
    }
  }
  E->capX = E->gridStepX + E->tabX.grids();
  E->capY = E->G.grid + E->tabY.grids();
  E->capT = E->GT.grid + E->tabX.grids();
  E->capC = E->gridX + E->gridY + 2;
  if (cudaMalloc(&E->d_ctrl, sizeof(PdcsCtrl)) != cudaSuccess ||
      cudaMalloc(&E->d_red, sizeof(double) * 16) != cudaSuccess ||
      cudaMalloc(&E->d_partX, sizeof(double) * GX_N * E->capX) != cudaSuccess ||
      cudaMalloc(&E->d_partY, sizeof(double) * GY_N * E->capY) != cudaSuccess ||
      cudaMalloc(&E->d_partT, sizeof(double) * GT_N * E->capT) != cudaSuccess ||
      cudaMalloc(&E->d_partC, sizeof(double) * std::max(PDCS_NMET, 4 * GAP_K) * E->capC) != cudaSuccess ||
      cudaMalloc(&E->d_out, sizeof(double) * 64) != cudaSuccess ||
      cudaMalloc(&E->d_err, sizeof(int)) != cudaSuccess ||
      cudaMalloc(&E->d_ticket, sizeof(unsigned) * 4) != cudaSuccess ||
      cudaMallocHost(&E->h_pinned, sizeof(double) * 128) != cudaSuccess ||
      cudaEventCreateWithFlags(&E->ev_ctrl[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&E->ev_ctrl[1], cudaEventDisableTiming) != cudaSuccess) {
    g_err = "pdcs_engine_create: workspace allocation failed";
    return fail(1);
  }
  if (cudaMemsetAsync(E->d_ctrl, 0, sizeof(PdcsCtrl), s) != cudaSuccess ||
      cudaMemsetAsync(E->d_err, 0, sizeof(int), s) != cudaSuccess ||
      cudaMemsetAsync(E->d_ticket, 0, sizeof(unsigned) * 4, s) != cudaSuccess ||
      cudaMemsetAsync(E->d_partX, 0, sizeof(double) * GX_N * E->capX, s) != cudaSuccess ||
      cudaMemsetAsync(E->d_partY, 0, sizeof(double) * GY_N * E->capY, s) != cudaSuccess ||
      cudaMemsetAsync(E->d_partT, 0, sizeof(double) * GT_N * E->capT, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess) {
    g_err = "pdcs_engine_create: workspace init failed";
    return fail(1);
  }
  T.lap("grids + workspace");
  *out = E;
  return 0;
}

void pdcs_engine_destroy(PdcsEngine* E) {
  if (!E) return;
  PhaseTimer T("destroy", E->stream);
  if (E->stream) cudaStreamSynchronize(E->stream);
  T.lap("stream drain");
  if (E->exec) cudaGraphExecDestroy(E->exec);
  if (E->graph) cudaGraphDestroy(E->graph);
  T.lap("graph");
  free_plan(E->G);
  free_plan(E->GT);
  T.lap("plans");
  free_panels(E->PG, E->stream);
  free_panels(E->PGT, E->stream);
  if (E->d_wpart_y) cudaFreeAsync(E->d_wpart_y, E->stream);
  if (E->d_wpart_x) cudaFreeAsync(E->d_wpart_x, E->stream);
  if (E->stream) cudaStreamSynchronize(E->stream);  // the stream may go away with the caller
  T.lap("panels");
  if (E->comm && g_nccl.ok) g_nccl.commDestroy((ncclComm_t)E->comm);
  T.lap("comm");
  cudaFree(E->d_yred);
  cudaFree(E->d_gtp);
  free_table(E->tabX);
  free_table(E->tabXs);
  cudaFree(E->d_exp_rho);
  cudaFree(E->d_rowhead);
  cudaFree(E->d_pX);
  cudaFree(E->d_pY);
  cudaFree(E->d_pT);
  free_table(E->tabY);
  cudaFree(E->d_unif_x);
  cudaFree(E->d_unif_y);
  cudaFree(E->d_ctrl);
  cudaFree(E->d_red);
  cudaFree(E->d_partX);
  cudaFree(E->d_partY);
  cudaFree(E->d_partT);
  cudaFree(E->d_partC);
  cudaFree(E->d_out);
  cudaFree(E->d_err);
  cudaFree(E->d_ticket);
  T.lap("device buffers");
  if (E->h_pinned) cudaFreeHost(E->h_pinned);
  T.lap("pinned");
  for (cudaEvent_t ev : E->ev_ctrl)
    if (ev) cudaEventDestroy(ev);
  T.lap("events");
  delete E;
}

int pdcs_precondition(PdcsEngine* E, int32_t enabled, int32_t ruiz_iters, int32_t use_pc) {
  if (!E) { g_err = "pdcs_precondition: null engine"; return 2; }
  const PdcsEngineDesc& d = E->d;
  cudaStream_t s = E->stream;
  const KArgs A = make_args(E);
  const int n = E->n, m = E->m, nnz = E->nnz;
  PhaseTimer T("precondition", s);
  T.lap("queued work");
  int* rowid = nullptr;
  if (nnz > 0) {
    CK(cudaMallocAsync(&rowid, sizeof(int) * nnz, s));
    k_iota_rows<<<grid_for(m), BS, 0, s>>>(d.d_g_rowptr, m, rowid);
    CKL();
  }
  T.lap("row ids");
  E->precond_mode = enabled;
  // enabled: 0 identity, 1 Ruiz + PC on this matrix, 2 as-is (d1/d2 = cone
  // scales, values untouched), 3 d1/d2 written by the caller (a shard taking
  // the scaling of the full matrix), values scaled by them
  if (enabled == 0 || enabled == 1) {
    k_fill<<<grid_for(m), BS, 0, s>>>(d.d_d1, m, 1.0);
    CKL();
    k_fill<<<grid_for(n), BS, 0, s>>>(d.d_d2, n, 1.0);
    CKL();
  }
  // sharded engine (communicator attached): this rank holds a row slice of
  // G; row statistics are local, column statistics are all-reduced over the
  // ranks (max-abs for Ruiz, sums of |a_ij| for Pock-Chambolle), so every
  // rank ends with its slice of D1 and the global D2 (SURVEY 8(e) "At setup")
  const bool shard = E->comm && E->nranks > 1;
  if (enabled == 1 && (nnz > 0 || shard)) {
    // Ruiz rounds on working copies held in g_val and gt_val (scaling.py:84-90):
    // both are scaled in place each round, G^T's entries with the operands of
    // their G entries ((r_row * v) * c_col, the same operations, so gt_val stays
    // the exact transpose of g_val) -- no random gather of g_val per round
    int* rowid_t = nullptr;
    if (nnz > 0) {
      CK(cudaMemcpyAsync(d.d_g_val, d.d_g_val0, sizeof(double) * nnz, cudaMemcpyDeviceToDevice, s));
      k_gather<<<grid_for(nnz), BS, 0, s>>>(d.d_gt_val, d.d_g_val, d.d_perm, nnz);
      CKL();
      CK(cudaMallocAsync(&rowid_t, sizeof(int) * nnz, s));
      k_iota_rows<<<grid_for(n), BS, 0, s>>>(d.d_gt_rowptr, n, rowid_t);
      CKL();
    }
    for (int it = 0; it < ruiz_iters; ++it) {
      if (launch_rowred<0>(E->G, d.d_g_val, d.d_ty0, s)) return 1;
      if (launch_rowred<0>(E->GT, d.d_gt_val, d.d_tx0, s)) return 1;
      if (shard && nccl_allreduce(d.d_tx0, d.d_tx0, n, E->comm, s, ncclMax)) return 1;
      k_inv_sqrt_mul<<<grid_for(m), BS, 0, s>>>(d.d_ty0, d.d_ty1, d.d_d1, m);
      CKL();
      k_inv_sqrt_mul<<<grid_for(n), BS, 0, s>>>(d.d_tx0, d.d_tx1, d.d_d2, n);
      CKL();
      k_scale_vals<<<grid_for(nnz), BS, 0, s>>>(d.d_g_val, d.d_g_val, rowid, d.d_g_colidx, d.d_ty1,
                                                d.d_tx1, nnz);
      CKL();
      k_scale_vals<<<grid_for(nnz), BS, 0, s>>>(d.d_gt_val, d.d_gt_val, d.d_gt_colidx, rowid_t, d.d_ty1,
                                                d.d_tx1, nnz);
      CKL();
    }
    if (rowid_t) CK(cudaFreeAsync(rowid_t, s));
    T.lap("ruiz rounds");
    if (use_pc) {  // Pock-Chambolle alpha = 1 (scaling.py:92-96); gt_val is g_val's transpose
      if (launch_rowred<1>(E->G, d.d_g_val, d.d_ty0, s)) return 1;
      if (launch_rowred<1>(E->GT, d.d_gt_val, d.d_tx0, s)) return 1;
      if (shard && nccl_allreduce(d.d_tx0, d.d_tx0, n, E->comm, s, ncclSum)) return 1;
      k_inv_sqrt_mul<<<grid_for(m), BS, 0, s>>>(d.d_ty0, d.d_ty1, d.d_d1, m);
      CKL();
      k_inv_sqrt_mul<<<grid_for(n), BS, 0, s>>>(d.d_tx0, d.d_tx1, d.d_d2, n);
      CKL();
    }
    if (E->n_unif_x) {
      k_geo_mean<<<grid_for(E->n_unif_x, BS / 32), BS, 0, s>>>(E->d_unif_x, E->n_unif_x, d.d_d2);
      CKL();
    }
    if (E->n_unif_y) {
      k_geo_mean<<<grid_for(E->n_unif_y, BS / 32), BS, 0, s>>>(E->d_unif_y, E->n_unif_y, d.d_d1);
      CKL();
    }
    k_clip<<<grid_for(m), BS, 0, s>>>(d.d_d1, m, 1e-8, 1e8);
    CKL();
    k_clip<<<grid_for(n), BS, 0, s>>>(d.d_d2, n, 1e-8, 1e8);
    CKL();
  }
  T.lap("pc + clip");
  // G^ = D1 G D2 from the original values, then its transpose by the perm map
  if (nnz > 0) {
    if (enabled == 2) {
      CK(cudaMemcpyAsync(d.d_g_val, d.d_g_val0, sizeof(double) * nnz, cudaMemcpyDeviceToDevice, s));
    } else {
      k_scale_vals<<<grid_for(nnz), BS, 0, s>>>(d.d_g_val, d.d_g_val0, rowid, d.d_g_colidx, d.d_d1,
                                                d.d_d2, nnz);
      CKL();
    }
    k_gather<<<grid_for(nnz), BS, 0, s>>>(d.d_gt_val, d.d_g_val, d.d_perm, nnz);
    CKL();
    if (refresh_panel_values(E->PG, d.d_g_val, s) || refresh_panel_values(E->PGT, d.d_gt_val, s))
      return 1;
  }
  k_scale_x<<<grid_for(n), BS, 0, s>>>(A, enabled == 2);
  CKL();
  k_scale_y<<<grid_for(m), BS, 0, s>>>(A, enabled == 2);
  CKL();
  if (rowid) CK(cudaFreeAsync(rowid, s));
  CK(cudaStreamSynchronize(s));
  T.lap("scale + panels");
  return 0;
}

int pdcs_stats(PdcsEngine* E, double* h_out) {
  const KArgs A = make_args(E);
  cudaStream_t s = E->stream;
  if (E->m > 0 && launch_rowred<1>(E->G, E->d.d_g_val, E->d.d_ty2, s)) return 1;
  const int g = std::max(E->gridX, E->gridY);
  if (g > E->capC) { g_err = "pdcs_stats: partial capacity"; return 1; }
  k_stats<<<g, BS, 0, s>>>(A, E->d.d_g_val, E->nnz, E->d.d_ty2, E->d_partC, E->capC);
  CKL();
  return finalize_to_host(E, E->d_partC, E->capC, g, 6, 0x30u, h_out);
}

int pdcs_engine_info(PdcsEngine* E, double* h_out) {
  const double v[] = {(double)E->G.vw, (double)E->GT.vw, (double)E->gridStepX, (double)E->G.grid,
                      (double)E->GT.grid, (double)E->keep_xt, (double)E->keep_yh,
                      (double)E->l2_persist, (double)E->G.n_long, (double)E->GT.n_long,
                      (double)E->tabX.total(), (double)E->tabY.total(), (double)E->PG.np,
                      (double)E->PGT.np, (double)E->G.step_vw, (double)E->GT.step_vw};
  std::memcpy(h_out, v, sizeof(v));
  return 0;
}

int pdcs_engine_get_ctrl(PdcsEngine* E, PdcsCtrl* h) {
  CK(cudaMemcpyAsync(E->h_pinned, E->d_ctrl, sizeof(PdcsCtrl), cudaMemcpyDeviceToHost, E->stream));
  CK(cudaStreamSynchronize(E->stream));
  std::memcpy(h, E->h_pinned, sizeof(PdcsCtrl));
  int err = 0;
  CK(cudaMemcpyAsync(&err, E->d_err, sizeof(int), cudaMemcpyDeviceToHost, E->stream));
  CK(cudaStreamSynchronize(E->stream));
  if (err && !h->error) h->error = err;
  return 0;
}

int pdcs_engine_set_ctrl(PdcsEngine* E, const PdcsCtrl* h) {
  std::memcpy(E->h_pinned, h, sizeof(PdcsCtrl));
  CK(cudaMemcpyAsync(E->d_ctrl, E->h_pinned, sizeof(PdcsCtrl), cudaMemcpyHostToDevice, E->stream));
  CK(cudaMemsetAsync(E->d_err, 0, sizeof(int), E->stream));
  CK(cudaStreamSynchronize(E->stream));
  return 0;
}

extern "C++" {
template <int VWY, int VWT>
static int persist_launch(Engine* E, long long max_trials) {
  KArgs A = make_args(E);
  TileSrc SY = tile_source(E->G, E->PG, 0, nullptr), ST = tile_source(E->GT, E->PGT, 0, nullptr);
  double *pX = E->d_pX, *pY = E->d_pY, *pT = E->d_pT;
  int cap = E->pgrid;
  void* args[] = {&A, &SY, &ST, &pX, &pY, &pT, &cap, &max_trials};
  CK(cudaLaunchCooperativeKernel((const void*)k_persist<VWY, VWT>, E->pgrid, BS, args, 0, E->stream));
  g_launches.fetch_add(1);
  return 0;
}

// The device loop of a persistent engine: one cooperative launch until the
// control block stops (batch end, check, budget, error).  The trial cap only
// guards against a hang: 61 trials per remaining iteration (60 rejections
// trip the trial cap) plus slack.
static int run_persist(Engine* E) {
  PdcsCtrl c;
  CK(cudaMemcpyAsync(E->h_pinned, E->d_ctrl, sizeof(PdcsCtrl), cudaMemcpyDeviceToHost, E->stream));
  CK(cudaStreamSynchronize(E->stream));
  std::memcpy(&c, E->h_pinned, sizeof(PdcsCtrl));
  const long long left = std::max<long long>(1, std::min<long long>(c.k_bar_stop, c.max_iter) - c.k_bar);
  const long long max_trials = left * 61 + 128;
  int rc = 0;
  switch (E->G.step_vw * 100 + E->GT.step_vw) {
    case 101: rc = persist_launch<1, 1>(E, max_trials); break;
    case 108: rc = persist_launch<1, 8>(E, max_trials); break;
    case 132: rc = persist_launch<1, 32>(E, max_trials); break;
    case 801: rc = persist_launch<8, 1>(E, max_trials); break;
    case 808: rc = persist_launch<8, 8>(E, max_trials); break;
    case 832: rc = persist_launch<8, 32>(E, max_trials); break;
    case 3201: rc = persist_launch<32, 1>(E, max_trials); break;
    case 3208: rc = persist_launch<32, 8>(E, max_trials); break;
    default: rc = persist_launch<32, 32>(E, max_trials); break;
  }
  if (rc) return rc;
  CK(cudaStreamSynchronize(E->stream));
  return 0;
}
}  // extern "C++"

int pdcs_run_inner(PdcsEngine* E, int32_t slots) {
  if (slots < 1) slots = 1;
  if (E->persist && !E->comm) return run_persist(E);
  cudaStream_t s = E->stream;
  if (!E->exec || E->graph_slots != slots) {
    if (E->exec) { cudaGraphExecDestroy(E->exec); E->exec = nullptr; }
    if (E->graph) { cudaGraphDestroy(E->graph); E->graph = nullptr; }
    PhaseTimer T("run_inner", s);
    const int64_t before = g_launches.load();
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < slots; ++i) {
      if (launch_slot(E)) {
        cudaGraph_t tmp;
        cudaStreamEndCapture(s, &tmp);
        if (tmp) cudaGraphDestroy(tmp);
        return 1;
      }
    }
    CK(cudaStreamEndCapture(s, &E->graph));
    CK(cudaGraphInstantiate(&E->exec, E->graph, 0));
    T.lap("graph capture");
    E->graph_nodes = g_launches.load() - before;
    g_launches.fetch_sub(E->graph_nodes);  // captured, not launched
    E->graph_slots = slots;
  }
  // Two graph replays stay in flight: while replay i runs, the host waits for
  // the control block copied after replay i-1, so the GPU never idles on the
  // host round trip.  Once the device loop has stopped every kernel is gated
  // off, so the one extra replay costs only its empty launches.
  // Watchdog: k_bar must advance (every trial advances it); replays that leave
  // it unchanged 8 times in a row mean the device loop is stuck.
  PdcsCtrl* hc[2] = {reinterpret_cast<PdcsCtrl*>(E->h_pinned),
                     reinterpret_cast<PdcsCtrl*>(E->h_pinned + 64)};
  static_assert(sizeof(PdcsCtrl) <= 64 * sizeof(double), "ctrl copy slot");
  auto replay = [&](int b) -> int {
    CK(cudaGraphLaunch(E->exec, s));
    g_launches.fetch_add(E->graph_nodes);
    CK(cudaMemcpyAsync(hc[b], E->d_ctrl, sizeof(PdcsCtrl), cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(E->ev_ctrl[b], s));
    return 0;
  };
  int64_t last_kbar = -1;
  int stuck = 0, b = 0;
  if (replay(0)) return 1;
  for (;;) {
    if (replay(b ^ 1)) return 1;
    CK(cudaEventSynchronize(E->ev_ctrl[b]));
    if (hc[b]->stop) break;
    if (hc[b]->k_bar == last_kbar) {
      if (++stuck >= 8) {
        CK(cudaStreamSynchronize(s));
        g_err = "pdcs_run_inner: device loop made no progress";
        return 3;
      }
    } else {
      stuck = 0;
      last_kbar = hc[b]->k_bar;
    }
    b ^= 1;
  }
  CK(cudaStreamSynchronize(s));
  return 0;
}

// ---- batched engines: one CUDA graph advances many independent solves ------
// The graph forks from the batch stream into every member engine's stream
// (each branch = `slots` line-search trials of that engine, the same launch
// sequence pdcs_run_inner captures), joins back, and gathers the members'
// control blocks.  Members whose device loop has stopped are gated off (every
// step kernel returns on ctrl->stop), so one replay advances exactly the
// members the host has released; results are bit-identical to running each
// engine alone.
struct PdcsBatch {
  std::vector<Engine*> E;
  cudaStream_t stream = nullptr;
  PdcsCtrl** d_src = nullptr;   // [n] member control blocks
  PdcsCtrl* d_ctrls = nullptr;  // [n] gathered copies
  PdcsCtrl* h_ctrls = nullptr;  // pinned [2][n]
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaEvent_t fork = nullptr;
  std::vector<cudaEvent_t> join;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int slots = 0;
  int64_t nodes = 0;
};

int pdcs_batch_create(PdcsEngine** engines, int32_t n, void* stream, PdcsBatch** out) {
  if (!engines || n < 1 || !out) { g_err = "pdcs_batch_create: bad arguments"; return 2; }
  PdcsBatch* B = new PdcsBatch();
  B->stream = (cudaStream_t)stream;
  std::vector<PdcsCtrl*> src;
  for (int i = 0; i < n; ++i) {
    if (!engines[i] || engines[i]->comm) {
      delete B;
      g_err = "pdcs_batch_create: null or sharded engine";
      return 2;
    }
    B->E.push_back(engines[i]);
    src.push_back(engines[i]->d_ctrl);
  }
  B->join.assign(n, nullptr);
  if (cudaMalloc(&B->d_src, sizeof(PdcsCtrl*) * n) != cudaSuccess ||
      cudaMalloc(&B->d_ctrls, sizeof(PdcsCtrl) * n) != cudaSuccess ||
      cudaMallocHost(&B->h_ctrls, sizeof(PdcsCtrl) * 2 * n) != cudaSuccess ||
      cudaEventCreateWithFlags(&B->ev[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&B->ev[1], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&B->fork, cudaEventDisableTiming) != cudaSuccess) {
    pdcs_batch_destroy(B);
    g_err = "pdcs_batch_create: allocation failed";
    return 1;
  }
  for (int i = 0; i < n; ++i) {
    if (cudaEventCreateWithFlags(&B->join[i], cudaEventDisableTiming) != cudaSuccess) {
      pdcs_batch_destroy(B);
      g_err = "pdcs_batch_create: event creation failed";
      return 1;
    }
  }
  if (cudaMemcpyAsync(B->d_src, src.data(), sizeof(PdcsCtrl*) * n, cudaMemcpyHostToDevice, B->stream) !=
          cudaSuccess ||
      cudaStreamSynchronize(B->stream) != cudaSuccess) {
    pdcs_batch_destroy(B);
    g_err = "pdcs_batch_create: upload failed";
    return 1;
  }
  *out = B;
  return 0;
}

void pdcs_batch_destroy(PdcsBatch* B) {
  if (!B) return;
  if (B->stream) cudaStreamSynchronize(B->stream);
  if (B->exec) cudaGraphExecDestroy(B->exec);
  if (B->graph) cudaGraphDestroy(B->graph);
  cudaFree(B->d_src);
  cudaFree(B->d_ctrls);
  if (B->h_ctrls) cudaFreeHost(B->h_ctrls);
  for (auto e : B->ev) if (e) cudaEventDestroy(e);
  if (B->fork) cudaEventDestroy(B->fork);
  for (auto e : B->join) if (e) cudaEventDestroy(e);
  delete B;
}

static int batch_capture(PdcsBatch* B, int slots) {
  if (B->exec) { cudaGraphExecDestroy(B->exec); B->exec = nullptr; }
  if (B->graph) { cudaGraphDestroy(B->graph); B->graph = nullptr; }
  const int n = (int)B->E.size();
  cudaStream_t s = B->stream;
  const int64_t before = g_launches.load();
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  auto abort = [&]() {
    cudaGraph_t tmp = nullptr;
    cudaStreamEndCapture(s, &tmp);
    if (tmp) cudaGraphDestroy(tmp);
    return 1;
  };
  if (cudaEventRecord(B->fork, s) != cudaSuccess) return abort();
  for (int i = 0; i < n; ++i) {
    Engine* E = B->E[i];
    if (cudaStreamWaitEvent(E->stream, B->fork, 0) != cudaSuccess) return abort();
    for (int k = 0; k < slots; ++k)
      if (launch_slot(E)) return abort();
    if (cudaEventRecord(B->join[i], E->stream) != cudaSuccess ||
        cudaStreamWaitEvent(s, B->join[i], 0) != cudaSuccess)
      return abort();
  }
  k_gather_ctrl<<<grid_for((int64_t)n * (sizeof(PdcsCtrl) / 8)), BS, 0, s>>>(B->d_src, B->d_ctrls, n);
  if (cudaGetLastError() != cudaSuccess) return abort();
  CK(cudaStreamEndCapture(s, &B->graph));
  CK(cudaGraphInstantiate(&B->exec, B->graph, 0));
  B->nodes = g_launches.load() - before;
  g_launches.fetch_sub(B->nodes);
  B->slots = slots;
  return 0;
}

int pdcs_batch_run(PdcsBatch* B, int32_t slots) {
  if (!B) { g_err = "pdcs_batch_run: null batch"; return 2; }
  if (slots < 1) slots = 1;
  if (!B->exec || B->slots != slots) {
    if (batch_capture(B, slots)) return 1;
  }
  const int n = (int)B->E.size();
  cudaStream_t s = B->stream;
  PdcsCtrl* hc[2] = {B->h_ctrls, B->h_ctrls + n};
  auto replay = [&](int b) -> int {
    CK(cudaGraphLaunch(B->exec, s));
    g_launches.fetch_add(B->nodes);
    CK(cudaMemcpyAsync(hc[b], B->d_ctrls, sizeof(PdcsCtrl) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(B->ev[b], s));
    return 0;
  };
  // two replays in flight, as in pdcs_run_inner; done when every member's
  // device loop has stopped; watchdog on the members still running
  std::vector<int64_t> last(n, -1);
  int stuck = 0, b = 0;
  if (replay(0)) return 1;
  for (;;) {
    if (replay(b ^ 1)) return 1;
    CK(cudaEventSynchronize(B->ev[b]));
    bool all = true, moved = false;
    for (int i = 0; i < n; ++i) {
      if (hc[b][i].stop) continue;
      all = false;
      if (hc[b][i].k_bar != last[i]) moved = true;
      last[i] = hc[b][i].k_bar;
    }
    if (all) break;
    if (!moved) {
      if (++stuck >= 8) {
        CK(cudaStreamSynchronize(s));
        g_err = "pdcs_batch_run: device loop made no progress";
        return 3;
      }
    } else {
      stuck = 0;
    }
    b ^= 1;
  }
  CK(cudaStreamSynchronize(s));
  return 0;
}

int pdcs_profile_slot(PdcsEngine* E, int32_t reps, double* h_ms, const char** h_names, int32_t cap) {
  cudaStream_t s = E->stream;
  int count = 0;
  std::vector<double> acc;
  for (int r = 0; r < reps; ++r) {
    g_prof.ev.clear();
    g_prof.names.clear();
    g_prof.on = true;
    mark(s, "start");
    int rc = launch_slot(E);
    g_prof.on = false;
    if (rc) return rc;
    CK(cudaStreamSynchronize(s));
    const int k = (int)g_prof.ev.size() - 1;
    if (r == 0) {
      count = k;
      acc.assign(k, 0.0);
    }
    for (int i = 0; i < k && i < count; ++i) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, g_prof.ev[i], g_prof.ev[i + 1]));
      acc[i] += ms;
    }
    for (auto e : g_prof.ev) cudaEventDestroy(e);
  }
  for (int i = 0; i < count && i < cap; ++i) {
    h_ms[i] = acc[i] / reps;
    h_names[i] = g_prof.names[i + 1];
  }
  return count;
}

int pdcs_flush(PdcsEngine* E) {
  const KArgs A = make_args(E);
  k_flush_x<<<E->gridX, BS, 0, E->stream>>>(A);
  CKL();
  k_flush_y<<<E->gridY, BS, 0, E->stream>>>(A);
  CKL();
  k_clear_pending<<<1, 1, 0, E->stream>>>(E->d_ctrl);
  CKL();
  CK(cudaStreamSynchronize(E->stream));
  return 0;
}

int pdcs_engine_spmv(PdcsEngine* E, int32_t transpose, const double* in, double* out) {
  int rc = launch_spmv(transpose ? E->GT : E->G, in, out, E->stream);
  if (rc) return rc;
  CK(cudaStreamSynchronize(E->stream));
  return 0;
}

static int project_blocks(Engine* E, const BlockTable& T, const double* buf, int dualize, int smode,
                          const double* scale, RootCfg rcfg = RootCfg()) {
  if (T.total() == 0) return 0;
  const KArgs A = make_args(E);
  BlkParams P{buf, const_cast<double*>(buf), scale, dualize, smode};
  P.rc = rcfg;
  return launch_blocks<OP_PROJECT>(T, A, P, nullptr, 0, 0, 0, E->stream);
}

static int check_err(Engine* E) {
  int err = 0;
  CK(cudaMemcpyAsync(&err, E->d_err, sizeof(int), cudaMemcpyDeviceToHost, E->stream));
  CK(cudaStreamSynchronize(E->stream));
  if (err) {
    CK(cudaMemsetAsync(E->d_err, 0, sizeof(int), E->stream));
    g_err = "numerical failure in a cone projection (code " + std::to_string(err) + ")";
    return 3;
  }
  return 0;
}

int pdcs_metrics(PdcsEngine* E, int32_t mode, const double* x, const double* y, const double* gx,
                 const double* gty, double* h_out) {
  const KArgs A = make_args(E);
  cudaStream_t s = E->stream;
  const int orig = mode == 1;
  if (E->has_xblocks || E->has_yblocks) {
    k_met_fill<<<std::max(E->gridX, E->gridY), BS, 0, s>>>(A, mode, gx, gty);
    CKL();
    if (project_blocks(E, E->tabX, E->d.d_tx1, 1, orig ? PDCS_SCALE_NONE : PDCS_SCALE_INVERT, E->d.d_d2))
      return 1;
    if (project_blocks(E, E->tabY, E->d.d_ty1, 0, orig ? PDCS_SCALE_NONE : PDCS_SCALE_INVERT, E->d.d_d1))
      return 1;
  }
  k_met_y<<<E->gridY, BS, 0, s>>>(A, mode, y, gx, E->d_partC, E->capC, 0);
  CKL();
  k_met_x<<<E->gridX, BS, 0, s>>>(A, mode, x, gty, E->d_partC, E->capC, E->gridY);
  CKL();
  if (finalize_to_host(E, E->d_partC, E->capC, E->gridX + E->gridY, PDCS_NMET, MET_MAXMASK, h_out))
    return 1;
  return check_err(E);
}

int pdcs_rays(PdcsEngine* E, const double* x, const double* y, const double* gx, const double* gty,
              double xnorm, double ynorm, double* h_out) {
  const KArgs A = make_args(E);
  cudaStream_t s = E->stream;
  if (E->has_xblocks || E->has_yblocks) {
    k_ray_fill<<<std::max(E->gridX, E->gridY), BS, 0, s>>>(A, x, gx, gty, xnorm, ynorm);
    CKL();
    if (project_blocks(E, E->tabX, E->d.d_tx1, 1, PDCS_SCALE_NONE, nullptr)) return 1;
    if (project_blocks(E, E->tabX, E->d.d_tx2, 0, PDCS_SCALE_NONE, nullptr)) return 1;
    if (project_blocks(E, E->tabY, E->d.d_ty1, 0, PDCS_SCALE_NONE, nullptr)) return 1;
  }
  k_ray_y<<<E->gridY, BS, 0, s>>>(A, y, gx, xnorm, E->d_partC, E->capC, 0);
  CKL();
  k_ray_x<<<E->gridX, BS, 0, s>>>(A, x, gty, xnorm, ynorm, E->d_partC, E->capC, E->gridY);
  CKL();
  if (finalize_to_host(E, E->d_partC, E->capC, E->gridX + E->gridY, PDCS_NRAY, RAY_MAXMASK, h_out))
    return 1;
  return check_err(E);
}

int pdcs_gap_probe(PdcsEngine* E, const double* x, const double* y, const double* gx,
                   const double* gty, double t, double tau, double sigma, double* h_out) {
  const KArgs A = make_args(E);
  cudaStream_t s = E->stream;
  k_gap_x<<<E->gridX, BS, 0, s>>>(A, x, gty, t * tau);
  CKL();
  k_gap_y<<<E->gridY, BS, 0, s>>>(A, y, gx, t * sigma);
  CKL();
  if (project_blocks(E, E->tabX, E->d.d_tx0, 0, PDCS_SCALE_DIRECT, E->d.d_d2)) return 1;
  if (project_blocks(E, E->tabY, E->d.d_ty0, 1, PDCS_SCALE_DIRECT, E->d.d_d1)) return 1;
  const int g = std::max(E->gridX, E->gridY);
  k_gap_red<<<g, BS, 0, s>>>(A, x, y, gx, gty, E->d_partC, E->capC);
  CKL();
  if (finalize_to_host(E, E->d_partC, E->capC, g, 4, 0u, h_out)) return 1;
  return check_err(E);
}

int pdcs_gap_probes(PdcsEngine* E, const double* x, const double* y, const double* gx,
                    const double* gty, const double* ts, int32_t k, double tau, double sigma,
                    double* h_out) {
  if (k < 1 || k > GAP_K) { g_err = "pdcs_gap_probes: k must be in [1, 16]"; return 2; }
  const KArgs A = make_args(E);
  cudaStream_t s = E->stream;
  const int g = std::max(E->gridX, E->gridY);
  const bool blocks = E->has_xblocks || E->has_yblocks;
  if (!blocks) {
    GapTs T;
    T.k = k;
    for (int i = 0; i < GAP_K; ++i) {
      const double t = ts[std::min(i, k - 1)];
      T.tt[i] = t * tau;
      T.ts[i] = t * sigma;
    }
    k_gap_multi<<<g, BS, 0, s>>>(A, x, y, gx, gty, T, E->d_partC, E->capC);
    CKL();
  } else {
    // cone blocks: one probe pass per t (the block projections run on the
    // materialised z(t)), all partials kept for a single read-back
    for (int i = 0; i < k; ++i) {
      k_gap_x<<<E->gridX, BS, 0, s>>>(A, x, gty, ts[i] * tau);
      CKL();
      k_gap_y<<<E->gridY, BS, 0, s>>>(A, y, gx, ts[i] * sigma);
      CKL();
      if (project_blocks(E, E->tabX, E->d.d_tx0, 0, PDCS_SCALE_DIRECT, E->d.d_d2)) return 1;
      if (project_blocks(E, E->tabY, E->d.d_ty0, 1, PDCS_SCALE_DIRECT, E->d.d_d1)) return 1;
      k_gap_red<<<g, BS, 0, s>>>(A, x, y, gx, gty, E->d_partC + (size_t)4 * i * E->capC, E->capC);
      CKL();
    }
  }
  const int nq = blocks ? 4 * k : 4 * GAP_K;
  k_finalize_rows<<<nq, BS, 0, s>>>(E->d_partC, E->capC, g, E->d_out);
  CKL();
  CK(cudaMemcpyAsync(E->h_pinned, E->d_out, sizeof(double) * nq, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const double* o = E->h_pinned;
  for (int i = 0; i < k; ++i) {
    if (blocks) {
      for (int q = 0; q < 4; ++q) h_out[4 * i + q] = o[4 * i + q];
    } else {  // rows: x pass [2i] dx2, [2i+1] b1dx; y pass [2K+2i] dy2, [2K+2i+1] b2dy
      h_out[4 * i + 0] = o[2 * i];
      h_out[4 * i + 1] = o[2 * GAP_K + 2 * i];
      h_out[4 * i + 2] = o[2 * i + 1];
      h_out[4 * i + 3] = o[2 * GAP_K + 2 * i + 1];
    }
  }
  return check_err(E);
}

int pdcs_dist2(PdcsEngine* E, int32_t space, const double* a, const double* b, double* h_out) {
  const int n = space == 0 ? E->n : E->m;
  const int g = space == 0 ? E->gridX : E->gridY;
  k_dist2<<<g, BS, 0, E->stream>>>(a, b, n, E->d_partC, E->capC);
  CKL();
  return finalize_to_host(E, E->d_partC, E->capC, g, 1, 0u, h_out);
}

int pdcs_dot_diff(PdcsEngine* E, int32_t space, const double* a, const double* b, const double* c,
                  const double* d, double* h_out) {
  const int n = space == 0 ? E->n : E->m;
  const int g = space == 0 ? E->gridX : E->gridY;
  k_dot_diff<<<g, BS, 0, E->stream>>>(a, b, c, d, n, E->d_partC, E->capC);
  CKL();
  return finalize_to_host(E, E->d_partC, E->capC, g, 1, 0u, h_out);
}

int pdcs_project_set(PdcsEngine* E, int32_t which, const double* in, double* out) {
  return pdcs_project_set_ex(E, which, in, out, 1e-12, 100);
}

int pdcs_project_set_ex(PdcsEngine* E, int32_t which, const double* in, double* out, double root_tol,
                        int32_t max_root_iters) {
  const KArgs A = make_args(E);
  cudaStream_t s = E->stream;
  if (which < 0 || which > 4) { g_err = "pdcs_project_set: bad set"; return 2; }
  if (!(root_tol >= 0.0) || max_root_iters < 1) {
    g_err = "pdcs_project_set_ex: root_tol must be >= 0 and max_root_iters >= 1";
    return 2;
  }
  RootCfg rcfg;
  rcfg.tol = root_tol;
  rcfg.iters = max_root_iters;
  const bool xs = which == 0 || which == 3 || which == 4;
  k_proj_elem<<<xs ? E->gridX : E->gridY, BS, 0, s>>>(A, which, in, out);
  CKL();
  int rc = 0;
  switch (which) {
    case 0: rc = project_blocks(E, E->tabX, out, 0, PDCS_SCALE_DIRECT, E->d.d_d2, rcfg); break;
    case 1: rc = project_blocks(E, E->tabY, out, 1, PDCS_SCALE_DIRECT, E->d.d_d1, rcfg); break;
    case 2: rc = project_blocks(E, E->tabY, out, 0, PDCS_SCALE_INVERT, E->d.d_d1, rcfg); break;
    case 3: rc = project_blocks(E, E->tabX, out, 1, PDCS_SCALE_INVERT, E->d.d_d2, rcfg); break;
    case 4: rc = project_blocks(E, E->tabX, out, 0, PDCS_SCALE_DIRECT, E->d.d_d2, rcfg); break;
  }
  if (rc) return rc;
  return check_err(E);
}

int pdcs_step_input(PdcsEngine* E, int32_t space, const double* v, const double* g, double step,
                    double* out) {
  const KArgs A = make_args(E);
  k_step_input<<<space == 0 ? E->gridX : E->gridY, BS, 0, E->stream>>>(A, space, v, g, step, out);
  CKL();
  CK(cudaStreamSynchronize(E->stream));
  return 0;
}

int pdcs_axpby(PdcsEngine* E, int32_t space, double a, const double* p, double b, const double* q,
               double* out) {
  const int n = space == 0 ? E->n : E->m;
  k_axpby<<<space == 0 ? E->gridX : E->gridY, BS, 0, E->stream>>>(n, a, p, b, q, 1.0, out);
  CKL();
  CK(cudaStreamSynchronize(E->stream));
  return 0;
}

int pdcs_project_box(int32_t len, const double* in, const double* l, const double* u, double* out,
                     void* stream) {
  if (len < 0) { g_err = "pdcs_project_box: negative length"; return 2; }
  if (len == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  k_box<<<grid_for(len), BS, 0, s>>>(len, in, l, u, out);
  CKL();
  CK(cudaStreamSynchronize(s));
  return 0;
}

int pdcs_vec_axpby(int32_t len, double a, const double* p, double b, const double* q, double d,
                   double* out, void* stream) {
  if (len < 0) { g_err = "pdcs_vec_axpby: negative length"; return 2; }
  if (len == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  k_axpby<<<grid_for(len), BS, 0, s>>>(len, a, p, b, q, d, out);
  CKL();
  CK(cudaStreamSynchronize(s));
  return 0;
}

int pdcs_unscale(PdcsEngine* E, const double* x, const double* y, const double* gx,
                 const double* gty, double* xo, double* yo, double* slack, double* lam) {
  const KArgs A = make_args(E);
  k_unscale<<<std::max(E->gridX, E->gridY), BS, 0, E->stream>>>(A, x, y, gx, gty, xo, yo, slack, lam);
  CKL();
  CK(cudaStreamSynchronize(E->stream));
  return 0;
}

int pdcs_comm_unique_id(unsigned char* h_id) {
  if (!nccl_load()) return 1;
  ncclUniqueId id;
  CKN(g_nccl.getUniqueId(&id));
  std::memcpy(h_id, id.internal, NCCL_UNIQUE_ID_BYTES);
  return 0;
}

int pdcs_engine_set_persist(PdcsEngine* E, int32_t on) {
  if (!E) { g_err = "pdcs_engine_set_persist: null engine"; return 2; }
  E->persist = on && E->d_pX != nullptr;  // only engines set up for it at create
  return 0;
}

int pdcs_engine_set_uniform_box(PdcsEngine* E, double lo, double hi) {
  if (!E) { g_err = "pdcs_engine_set_uniform_box: null engine"; return 2; }
  const char* env = getenv("PDCS_TUNE");
  if (env && strstr(env, "ubox=0")) return 0;  // measurement switch: read l^, u^ as before
  E->ubox = true;
  E->ubox_l = lo;
  E->ubox_u = hi;
  if (E->exec) { cudaGraphExecDestroy(E->exec); E->exec = nullptr; }  // KArgs are baked into the graph
  if (E->graph) { cudaGraphDestroy(E->graph); E->graph = nullptr; }
  E->graph_slots = 0;
  return 0;
}

int pdcs_engine_set_comm(PdcsEngine* E, const unsigned char* h_id, int32_t rank, int32_t nranks) {
  if (!E || !h_id || nranks < 1 || rank < 0 || rank >= nranks) {
    g_err = "pdcs_engine_set_comm: bad arguments";
    return 2;
  }
  if (!nccl_load()) return 1;
  ncclUniqueId id;
  std::memcpy(id.internal, h_id, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t comm = nullptr;
  CKN(g_nccl.commInitRank(&comm, nranks, id, rank));
  if (E->comm) g_nccl.commDestroy((ncclComm_t)E->comm);
  E->comm = comm;
  E->rank = rank;
  E->nranks = nranks;
  if (!E->d_yred) CK(cudaMalloc(&E->d_yred, sizeof(double) * 16));
  // G^T y partials, padded for the equal-slice reduce-scatter (nranks * ceil(n / nranks))
  const size_t gtp_len = (size_t)nranks * ((E->n + nranks - 1) / nranks) + 1;
  if (E->d_gtp) cudaFree(E->d_gtp);
  CK(cudaMalloc(&E->d_gtp, sizeof(double) * gtp_len));
  CK(cudaMemsetAsync(E->d_gtp, 0, sizeof(double) * gtp_len, E->stream));
  // until pdcs_engine_set_xsplit: every rank steps all of x-space
  E->xs0 = 0;
  E->xs1 = E->n;
  E->xcnt = 0;
  E->xcut.assign(nranks + 1, E->n);
  E->xcut[0] = 0;
  CK(cudaStreamSynchronize(E->stream));
  // the captured graph (if any) predates the communicator
  if (E->exec) { cudaGraphExecDestroy(E->exec); E->exec = nullptr; }
  if (E->graph) { cudaGraphDestroy(E->graph); E->graph = nullptr; }
  E->graph_slots = 0;
  return 0;
}

int pdcs_engine_set_xsplit(PdcsEngine* E, const int32_t* h_cuts, int32_t nranks) {
  if (!E || !h_cuts || !E->comm || nranks != E->nranks) {
    g_err = "pdcs_engine_set_xsplit: needs the engine's communicator and its rank count";
    return 2;
  }
  std::vector<int> cut(h_cuts, h_cuts + nranks + 1);
  if (cut[0] != 0 || cut[nranks] != E->n) { g_err = "pdcs_engine_set_xsplit: cuts must span [0, n]"; return 2; }
  for (int r = 0; r < nranks; ++r)
    if (cut[r + 1] < cut[r]) { g_err = "pdcs_engine_set_xsplit: cuts must be nondecreasing"; return 2; }
  for (const PdcsBlock& b : E->xblocks)
    for (int r = 1; r < nranks; ++r)
      if (cut[r] > b.start && cut[r] < b.start + b.dim) {
        g_err = "pdcs_engine_set_xsplit: a cut splits a primal cone block";
        return 2;
      }
  const int cnt = (E->n + nranks - 1) / nranks;
  bool equal = true;
  for (int r = 0; r <= nranks; ++r) equal = equal && cut[r] == std::min(r * cnt, E->n);
  E->xcut = cut;
  E->xcnt = equal ? cnt : 0;
  E->xs0 = cut[E->rank];
  E->xs1 = cut[E->rank + 1];
  std::vector<PdcsBlock> mine;
  for (const PdcsBlock& b : E->xblocks)
    if (b.start >= E->xs0 && b.start < E->xs1) mine.push_back(b);
  free_table(E->tabXs);
  if (build_table(E->tabXs, mine, E->stream)) return 1;
  E->xsplit = true;
  // fewer reduction slots may be written now: the rest must read as zero
  CK(cudaMemsetAsync(E->d_partX, 0, sizeof(double) * GX_N * E->capX, E->stream));
  CK(cudaMemsetAsync(E->d_partT, 0, sizeof(double) * GT_N * E->capT, E->stream));
  CK(cudaStreamSynchronize(E->stream));
  if (E->exec) { cudaGraphExecDestroy(E->exec); E->exec = nullptr; }
  if (E->graph) { cudaGraphDestroy(E->graph); E->graph = nullptr; }
  E->graph_slots = 0;
  return 0;
}

int pdcs_allgather_x(PdcsEngine* E, double* const* d_vecs, int32_t count) {
  if (!E || count < 0 || (count > 0 && !d_vecs)) { g_err = "pdcs_allgather_x: bad arguments"; return 2; }
  if (!E->comm || !E->xsplit || E->nranks <= 1) return 0;
  for (int i = 0; i < count; ++i)
    if (nccl_x_allgather(E, d_vecs[i], E->stream)) return 1;
  CK(cudaStreamSynchronize(E->stream));
  return 0;
}

int pdcs_debug_inject_nan(PdcsEngine* E, int64_t after_calls) {
  PdcsCtrl c;
  if (pdcs_engine_get_ctrl(E, &c)) return 1;
  c.nan_after = after_calls;
  return pdcs_engine_set_ctrl(E, &c);
}

}  // extern "C"
