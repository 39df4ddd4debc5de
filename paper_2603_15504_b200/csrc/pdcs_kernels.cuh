// Kernels of libpdcs.  Included by pdcs_engine.cu only.
#pragma once
#include <cooperative_groups.h>

#include "pdcs_internal.cuh"

namespace pdcs {

// All engine pointers, passed by value to kernels.
struct KArgs {
  int n, m, nbox, m_zero, m_elem;
  int x0, x1;  // x-space range this engine steps: [0, n), or the rank's slice when sharded
  const double *c, *h, *l, *u, *c0, *h0, *l0, *u0, *d1, *d2;
  double *x, *y, *xh, *yh, *xb, *yb, *xa, *ya;
  double *gx, *gty, *gxa, *gtya, *w, *gxh, *gth, *gtr, *xt;
  double *tx0, *tx1, *tx2, *ty0, *ty1, *ty2;
  PdcsCtrl* ctrl;
  int* err;
  float keep_xt, keep_yh;  // evict_last fractions of the gathered x~ / y_hat lines
  double* exp_rho;         // per dual exp block: Newton warm starts of its 2 projections (or null)
  // uniform box (every box coordinate has the same unscaled bounds lu, uu):
  // ub 1 = the scaled bounds are lu / d2_j, uu / d2_j (exactly k_scale_x's
  // division), read from d2 -- one stream instead of l^ and u^; ub 2 = as-is
  // scaling, the bounds are the constants themselves; ub 0 = read l^, u^
  int ub;
  double lu, uu;
};

// Scaled box bounds of coordinate j < nbox (k_scale_x: l^ = l0 / d2).
template <bool H>
__device__ __forceinline__ void box_bounds(const KArgs& A, int j, uint64_t ps, double& lj, double& uj) {
  if (A.ub == 1) {
    const double dj = ld_hint<H>(A.d2 + j, ps);
    lj = A.lu / dj;
    uj = A.uu / dj;
  } else if (A.ub == 2) {
    lj = A.lu;
    uj = A.uu;
  } else {
    lj = ld_hint<H>(A.l + j, ps);
    uj = ld_hint<H>(A.u + j, ps);
  }
}

// Controller folded into a step kernel (mode 0 off, 1 line search after the
// y-step, 2 beta after the G^T step).
struct CtrlFuse {
  int mode;
  unsigned* ticket;
  PdcsCtrl* C;
  const double* partA;  // x-group partials (mode 1)
  int capA;
  const double* partB;  // y-group (mode 1) or T-group (mode 2) partials
  int capB;
  double* red;
  const int* err;
};
template <int U = 1>
__device__ void ctrl_ls_body(PdcsCtrl*, const double*, int, const double*, int, double*, const double*);
template <int U = 1>
__device__ void ctrl_beta_body(PdcsCtrl*, const double*, int, const double*, const int*,
                               const double*);
__device__ __forceinline__ void fused_ctrl(const CtrlFuse& F);

// gate: 0 = always run, 1 = skip when stopped, 2 = skip when stopped or the
// current trial was rejected.
// Programmatic dependent launch (the step kernels of one trial, launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): wait for the previous
// kernel's grid to complete and its writes to be visible -- before ANY global
// access, in every CTA, so completion stays transitive along the stream.  No
// explicit launch_dependents: the next grid is launched when all of this
// grid's CTAs have exited (an early trigger placed the next grid's CTAs on
// the SMs with free slots first and unbalanced the one-wave grids: C5 612 vs
// 684 it/s).  A no-op for an ordinary launch.
__device__ __forceinline__ void pdl_enter() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ bool gated(const PdcsCtrl* c, int gate) {
  if (gate == 0) return false;
  if (c->stop) return true;
  return gate == 2 && !c->accepted;
}

__device__ __forceinline__ int dual_kind(int k) {
  switch (k) {
    case PDCS_ZERO: return PDCS_FREE;
    case PDCS_FREE: return PDCS_ZERO;
    case PDCS_EXP: return PDCS_DUAL_EXP;
    case PDCS_DUAL_EXP: return PDCS_EXP;
    default: return k;
  }
}

// Reductions whose bit is set in these masks are maxima, the rest sums.
constexpr unsigned MET_MAXMASK = (1u << PDCS_MET_RVMAX) | (1u << PDCS_MET_HMAX) |
                                 (1u << PDCS_MET_GXMAX) | (1u << PDCS_MET_RPMAX) |
                                 (1u << PDCS_MET_V1MAX) | (1u << PDCS_MET_V2MAX) |
                                 (1u << PDCS_MET_CMAX) | (1u << PDCS_MET_GTYMAX);
constexpr unsigned RAY_MAXMASK = (1u << 0) | (1u << 1) | (1u << 5) | (1u << 6) | (1u << 7);

// Block reduction of NQ quantities; bit q of maxmask selects max (else sum).
template <int NQ>
__device__ __forceinline__ void block_store_mask(double (&v)[NQ], unsigned maxmask, double* part,
                                                 int cap, int slot) {
  __shared__ double sh[NQ * 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    double t = v[q];
    const bool mx = (maxmask >> q) & 1u;
    for (int off = 16; off > 0; off >>= 1) {
      double o = __shfl_down_sync(0xffffffffu, t, off);
      t = mx ? nanmax(t, o) : t + o;
    }
    if (lane == 0) sh[q * 32 + wid] = t;
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const bool mx = (maxmask >> q) & 1u;
      double t = lane < nw ? sh[q * 32 + lane] : 0.0;
      for (int off = 16; off > 0; off >>= 1) {
        double o = __shfl_down_sync(0xffffffffu, t, off);
        t = mx ? nanmax(t, o) : t + o;
      }
      if (lane == 0) part[q * cap + slot] = t;
    }
  }
  __syncthreads();
}

// Reduce partial columns [0, nslots) of NQ rows into out[q] (one CTA).
__global__ void k_finalize(const double* part, int cap, int nslots, int nq, unsigned maxmask,
                           double* out) {
  __shared__ double sh[33];
  CtaGrp g(sh);
  for (int q = 0; q < nq; ++q) {
    const bool mx = (maxmask >> q) & 1u;
    double t = 0.0;
    for (int s = threadIdx.x; s < nslots; s += blockDim.x) {
      double v = part[q * cap + s];
      t = mx ? nanmax(t, v) : t + v;
    }
    t = mx ? g.max(t) : g.sum(t);
    if (threadIdx.x == 0) out[q] = t;
  }
}

// ---------------------------------------------------------------------------
// SpMV
// ---------------------------------------------------------------------------
template <int VW>
__device__ __forceinline__ double row_dot(const int* __restrict__ rp, const int* __restrict__ ci,
                                          const double* __restrict__ va,
                                          const double* __restrict__ x, int row, int sub,
                                          int nrows, int long_t, const double* longv,
                                          bool& lng, uint64_t pk) {
  double s = 0.0;
  lng = false;
  if (row < nrows) {
    const uint64_t ps = policy_stream();
    const int b = ld_hint(rp + row, ps), e = ld_hint(rp + row + 1, ps);
    if (e - b > long_t) {
      lng = true;
      if (sub == 0) s = longv[row];
    } else if (VW == 1) {
      // thread per row: issue four index loads, then four gathers, then
      // accumulate in index order (the sum order of scipy's csr_matvec)
      int j = b;
      for (; j + 4 <= e; j += 4) {
        const int c0 = ld_hint(ci + j, ps), c1 = ld_hint(ci + j + 1, ps);
        const int c2 = ld_hint(ci + j + 2, ps), c3 = ld_hint(ci + j + 3, ps);
        const double a0 = ld_hint(va + j, ps), a1 = ld_hint(va + j + 1, ps);
        const double a2 = ld_hint(va + j + 2, ps), a3 = ld_hint(va + j + 3, ps);
        const double x0 = ld_hint(x + c0, pk), x1 = ld_hint(x + c1, pk);
        const double x2 = ld_hint(x + c2, pk), x3 = ld_hint(x + c3, pk);
        s += a0 * x0;
        s += a1 * x1;
        s += a2 * x2;
        s += a3 * x3;
      }
      for (; j < e; ++j) s += ld_hint(va + j, ps) * ld_hint(x + ld_hint(ci + j, ps), pk);
    } else {
      for (int j = b + sub; j < e; j += VW) s += ld_hint(va + j, ps) * ld_hint(x + ld_hint(ci + j, ps), pk);
    }
  }
  if (VW > 1) {
#pragma unroll
    for (int off = VW / 2; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off, VW);
  }
  return s;
}

// Generic SpMV for short rows; long rows are already in y (written by
// k_long_partial) and are left untouched.
template <int VW>
__global__ void __launch_bounds__(BS) k_spmv(int nrows, const int* __restrict__ rp,
                                             const int* __restrict__ ci,
                                             const double* __restrict__ va,
                                             const double* __restrict__ x, double* y,
                                             int long_t, const PdcsCtrl* ctrl, int gate) {
  if (ctrl && gated(ctrl, gate)) return;
  const int lane = threadIdx.x & 31, sub = lane & (VW - 1);
  constexpr int RPW = 32 / VW;
  const int wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int wt = gridDim.x * (blockDim.x >> 5);
  for (int base = wg * RPW; base < nrows; base += wt * RPW) {
    const int row = base + lane / VW;
    bool lng;
    double s = row_dot<VW>(rp, ci, va, x, row, sub, nrows, long_t, y, lng, policy_stream());
    if (sub == 0 && row < nrows && !lng) y[row] = s;
  }
}

// Chunks of the long rows, one CTA reduction each; the last chunk of a row
// to finish (per-row ticket) adds the row's chunk sums in chunk order and
// writes y[row] -- no second launch, and the sum order is fixed.
// q = (row, begin, end, index of the row in the long-row list | LONG_DENSE
// when the chunk's columns are consecutive: C4's dense factor rows read no
// column indices and stream x).
constexpr int LONG_DENSE = 1 << 30;
__global__ void k_chunk_dense(int4* ch, int nch, const int* __restrict__ ci) {
  for (int c = blockIdx.x; c < nch; c += gridDim.x) {
    const int4 q = ch[c];
    const int c0 = ci[q.y];
    int ok = 1;
    for (int j = q.y + threadIdx.x; j < q.z; j += blockDim.x) ok &= ci[j] == c0 + (j - q.y);
    ok = __syncthreads_and(ok);
    if (threadIdx.x == 0 && ok) ch[c].w = q.w | LONG_DENSE;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(BS, 8) k_long_partial(const int4* __restrict__ ch, int nch, const int* __restrict__ ci,
                               const double* __restrict__ va, const double* __restrict__ x,
                               double* out, const PdcsCtrl* ctrl, int gate, const int* __restrict__ first,
                               unsigned* cnt, double* y) {
  if (gated(ctrl, gate)) return;
  __shared__ double sh[33];
  CtaGrp g(sh);
  for (int c = blockIdx.x; c < nch; c += gridDim.x) {
    const int4 q = ch[c];
    // eight independent gathers in flight per thread: the column loads of a
    // group first, then the gathers (the chain ci -> x is latency bound)
    constexpr int U = 8;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    const int bd = blockDim.x;
    int j = q.y + threadIdx.x;
    if (q.w & LONG_DENSE) {
      const double* xs = x + (__ldg(ci + q.y) - q.y);  // x index = column of j
      for (; j + (U - 1) * bd < q.z; j += U * bd) {
#pragma unroll
        for (int u = 0; u < U; ++u) acc[u & 3] += __ldg(va + j + u * bd) * __ldg(xs + j + u * bd);
      }
      for (; j < q.z; j += bd) acc[0] += __ldg(va + j) * __ldg(xs + j);
    } else {
      for (; j + (U - 1) * bd < q.z; j += U * bd) {
        int cc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) cc[u] = __ldg(ci + j + u * bd);
#pragma unroll
        for (int u = 0; u < U; ++u) acc[u & 3] += __ldg(va + j + u * bd) * __ldg(x + cc[u]);
      }
      for (; j < q.z; j += bd) acc[0] += __ldg(va + j) * __ldg(x + __ldg(ci + j));
    }
    const double s = g.sum((acc[0] + acc[1]) + (acc[2] + acc[3]));
    if (threadIdx.x == 0) {
      out[c] = s;
      const int i = q.w & (LONG_DENSE - 1), f = first[i], nc = first[i + 1] - f;
      if (nc == 1) {
        y[q.x] = s;
      } else {
        __threadfence();
        if (atomicAdd(cnt + i, 1u) == (unsigned)(nc - 1)) {
          __threadfence();
          double t = 0.0;
          for (int k = f; k < f + nc; ++k) t += __ldcg(out + k);
          y[q.x] = t;
          cnt[i] = 0u;
        }
      }
    }
    __syncthreads();
  }
}

// Panel build: entries per (panel, row); long rows get none.
__global__ void k_panel_count(int nrows, const int* __restrict__ rp, const int* __restrict__ ci,
                              int long_t, int np, int width, int* cnt) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
    const int b = rp[r], e = rp[r + 1];
    const bool lng = e - b > long_t;
    int j = b;
    for (int p = 0; p < np; ++p) {
      const long long lim = (long long)(p + 1) * width;
      int c = 0;
      while (!lng && j < e && ci[j] < lim) { ++c; ++j; }
      cnt[(long long)p * nrows + r] = c;
    }
  }
}
// Panel build: scatter column indices and CSR positions in panel-major order.
__global__ void k_panel_scatter(int nrows, const int* __restrict__ rp, const int* __restrict__ ci,
                                int long_t, int np, int width, const int* __restrict__ po, int* pci,
                                int* pperm) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
    const int b = rp[r], e = rp[r + 1];
    if (e - b > long_t) continue;
    int j = b;
    for (int p = 0; p < np; ++p) {
      const long long lim = (long long)(p + 1) * width;
      int pos = po[(long long)p * nrows + r];
      while (j < e && ci[j] < lim) {
        pci[pos] = ci[j];
        pperm[pos] = j;
        ++pos;
        ++j;
      }
    }
  }
}

// Row reductions used by the preconditioner: OP 0 = max |a_ij| (order free),
// OP 1 = sum |a_ij| (sequential in index order, like scipy's csr sum).
template <int OP>
__global__ void k_rowred_short(int nrows, const int* __restrict__ rp,
                               const double* __restrict__ va, double* out, int long_t) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
    const int b = rp[r], e = rp[r + 1];
    if (e - b > long_t) continue;
    double s = 0.0;
    for (int j = b; j < e; ++j) {
      double a = fabs(va[j]);
      s = OP == 0 ? (a > s ? a : s) : s + a;
    }
    out[r] = s;
  }
}

template <int OP>
__global__ void k_rowred_long_partial(const int4* __restrict__ ch, int nch,
                                      const double* __restrict__ va, double* out) {
  __shared__ double sh[33];
  CtaGrp g(sh);
  for (int c = blockIdx.x; c < nch; c += gridDim.x) {
    const int4 q = ch[c];
    double s = 0.0;
    for (int j = q.y + threadIdx.x; j < q.z; j += blockDim.x) {
      double a = fabs(va[j]);
      s = OP == 0 ? (a > s ? a : s) : s + a;
    }
    s = OP == 0 ? g.max(s) : g.sum(s);
    if (threadIdx.x == 0) out[c] = s;
  }
}

template <int OP>
__global__ void k_rowred_long_final(const int* rows, const int* first, int nl, const double* part,
                                    double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nl) return;
  double s = 0.0;
  for (int c = first[i]; c < first[i + 1]; ++c) s = OP == 0 ? (part[c] > s ? part[c] : s) : s + part[c];
  out[rows[i]] = s;
}

// ---------------------------------------------------------------------------
// Elementwise helpers
// ---------------------------------------------------------------------------
__global__ void k_fill(double* p, int n, double v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = v;
}
// Row-length statistics of a CSR for the SpMV plan (integer sums: exact and
// order-free, so the atomics are deterministic): [0] sum of short-row
// lengths, [1] sum of their squares, [2] short rows, [3] long rows (> long_t).
__global__ void k_row_stats(const int* __restrict__ rp, int nrows, int long_t,
                            unsigned long long* out) {
  unsigned long long s1 = 0, s2 = 0, cnt = 0, nl = 0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
    const unsigned long long len = (unsigned long long)(rp[r + 1] - rp[r]);
    if ((long long)len > long_t) {
      ++nl;
    } else {
      s1 += len;
      s2 += len * len;
      ++cnt;
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    s1 += __shfl_down_sync(0xffffffffu, s1, off);
    s2 += __shfl_down_sync(0xffffffffu, s2, off);
    cnt += __shfl_down_sync(0xffffffffu, cnt, off);
    nl += __shfl_down_sync(0xffffffffu, nl, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out + 0, s1);
    atomicAdd(out + 1, s2);
    atomicAdd(out + 2, cnt);
    atomicAdd(out + 3, nl);
  }
}

// Long rows (> long_t entries) in ascending order with their [begin, end).
struct IsLongRow {
  const int* rp;
  int long_t;
  __host__ __device__ bool operator()(int r) const { return rp[r + 1] - rp[r] > long_t; }
};

__global__ void k_row_extents(const int* __restrict__ rp, const int* rows, int n, int2* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = make_int2(rp[rows[i]], rp[rows[i] + 1]);
}

__global__ void k_iota_rows(const int* rp, int nrows, int* rowid) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x)
    for (int j = rp[r]; j < rp[r + 1]; ++j) rowid[j] = r;
}
__global__ void k_iota(int* p, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = i;
}
__global__ void k_count_cols(const int* ci, int nnz, int* cnt) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += gridDim.x * blockDim.x)
    atomicAdd(cnt + ci[i], 1);
}
__global__ void k_transpose_scatter(const int* perm, const int* rowid, const double* val, int nnz,
                                    int* tcol, double* tval) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += gridDim.x * blockDim.x) {
    const int q = perm[p];
    tcol[p] = rowid[q];
    if (val) tval[p] = val[q];
  }
}
__global__ void k_gather(double* dst, const double* src, const int* perm, int nnz) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += gridDim.x * blockDim.x)
    dst[p] = src[perm[p]];
}
// d *= r, r = 1/sqrt(v) for v > 0 else 1 (scaling.py:40-45)
__global__ void k_inv_sqrt_mul(const double* v, double* r, double* d, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double vi = v[i];
    double ri = vi > 0.0 ? 1.0 / sqrt(vi) : 1.0;
    r[i] = ri;
    d[i] = d[i] * ri;
  }
}
// vals = (r_row * vals) * c_col  (the association of diag(r) @ A @ diag(c))
__global__ void k_scale_vals(double* va, const double* src, const int* rowid, const int* ci,
                             const double* r, const double* c, int nnz) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += gridDim.x * blockDim.x)
    va[p] = (r[rowid[p]] * src[p]) * c[ci[p]];
}
__global__ void k_clip(double* d, int n, double lo, double hi) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    d[i] = clampv(d[i], lo, hi);
}
// geometric mean of each block's scale slice (scaling.py:48-62): warp per block
__global__ void k_geo_mean(const PdcsBlock* tab, int nb, double* d) {
  const int lane = threadIdx.x & 31;
  const int wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int wt = gridDim.x * (blockDim.x >> 5);
  for (int b = wg; b < nb; b += wt) {
    const PdcsBlock B = tab[b];
    double s = 0.0;
    for (int i = lane; i < B.dim; i += 32) s += log(d[B.start + i]);
    s = warp_sum(s);
    const double gm = exp(s / (double)B.dim);
    __syncwarp();
    for (int i = lane; i < B.dim; i += 32) d[B.start + i] = gm;
  }
}
// scaled instance vectors (scaling.py:115-135)
__global__ void k_scale_x(KArgs A, int asis) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < A.n; j += gridDim.x * blockDim.x) {
    double* c = const_cast<double*>(A.c);
    c[j] = asis ? A.c0[j] : A.c0[j] * A.d2[j];
    if (j < A.nbox) {
      const_cast<double*>(A.l)[j] = asis ? A.l0[j] : A.l0[j] / A.d2[j];
      const_cast<double*>(A.u)[j] = asis ? A.u0[j] : A.u0[j] / A.d2[j];
    }
  }
}
__global__ void k_scale_y(KArgs A, int asis) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.m; i += gridDim.x * blockDim.x)
    const_cast<double*>(A.h)[i] = asis ? A.h0[i] : A.h0[i] * A.d1[i];
}

__global__ void k_stats(KArgs A, const double* gval, int nnz, const double* rowsum, double* part,
                        int cap) {
  double acc[6] = {0, 0, 0, 0, 0, 0};
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int j = tid; j < A.n; j += nt) {
    double c = A.c[j];
    acc[0] += fabs(c);
    acc[2] += c * c;
  }
  for (int i = tid; i < A.m; i += nt) {
    double h = A.h[i];
    acc[1] += fabs(h);
    acc[3] += h * h;
    acc[5] = nanmax(acc[5], rowsum[i]);
  }
  for (int p = tid; p < nnz; p += nt) acc[4] = nanmax(acc[4], fabs(gval[p]));
  block_store_mask<6>(acc, 0x30u, part, cap, blockIdx.x);
}

// ---------------------------------------------------------------------------
// Cone-block kernels (segmented projections + fused epilogues)
// ---------------------------------------------------------------------------
enum { OP_PROJECT = 0, OP_STEP_X = 1, OP_STEP_Y = 2, OP_TLAM = 3 };
template <int OP> struct OpNQ { static constexpr int v = 1; };
template <> struct OpNQ<OP_STEP_X> { static constexpr int v = GX_N; };
template <> struct OpNQ<OP_STEP_Y> { static constexpr int v = GY_N; };
template <> struct OpNQ<OP_TLAM> { static constexpr int v = GT_N; };

struct BlkParams {
  const double* in;
  double* out;
  const double* scale;
  int dualize;
  int smode;  // -1: use the block's own smode
  RootCfg rc;  // ProjectionSettings of the standalone projection API
};

struct ThreadGrp {
  int rank = 0, size = 1;
  __device__ double sum(double v) const { return v; }
  __device__ double max(double v) const { return v; }
  __device__ int all(int v) const { return v; }
  __device__ void sync() const {}
};

template <class Grp, int OP>
__device__ __forceinline__ void do_block(const Grp& g, const PdcsBlock& b, const KArgs& A,
                                         const BlkParams& P, double* acc) {
  const int s = b.start, dim = b.dim;
  if (OP == OP_PROJECT) {
    const int kind = P.dualize ? dual_kind(b.kind) : b.kind;
    const int sm = P.smode >= 0 ? P.smode : b.smode;
    proj_segment(g, kind, sm, P.in + s, P.out + s, sm ? P.scale + s : nullptr, dim, A.err, P.rc);
    g.sync();
  } else if (OP == OP_STEP_X) {
    proj_segment(g, b.kind, PDCS_SCALE_DIRECT, A.xh + s, A.xh + s, A.d2 + s, dim, A.err);
    g.sync();
    for (int i = g.rank; i < dim; i += g.size) {
      const int j = s + i;
      const double xn = A.x[j], p = A.xh[j];
      A.xt[j] = 2.0 * p - xn;
      const double d = p - xn;
      acc[GX_XX] += xn * xn;
      acc[GX_DXDX] += d * d;
      acc[GX_CX] += A.c[j] * p;
    }
  } else if (OP == OP_STEP_Y) {
    proj_segment(g, dual_kind(b.kind), PDCS_SCALE_DIRECT, A.yh + s, A.yh + s, A.d1 + s, dim, A.err);
    for (int i = g.rank; i < dim; i += g.size) A.ty0[s + i] = A.gxh[s + i] - A.h[s + i];
    g.sync();
    proj_segment(g, b.kind, PDCS_SCALE_INVERT, A.ty0 + s, A.ty0 + s, A.d1 + s, dim, A.err);
    g.sync();
    for (int i = g.rank; i < dim; i += g.size) {
      const int r = s + i;
      const double yn = A.y[r], p = A.yh[r], hi = A.h[r];
      const double dy = p - yn;
      acc[GY_YY] += yn * yn;
      acc[GY_DYDY] += dy * dy;
      acc[GY_INTER] += dy * (A.w[r] - A.gx[r]);
      const double res = A.gxh[r] - hi;
      const double viol = res - A.ty0[r];
      acc[GY_RP2] += viol * viol;
      acc[GY_YH] += p * hi;
    }
  } else if (OP == OP_TLAM) {
    for (int i = g.rank; i < dim; i += g.size) A.tx0[s + i] = A.c[s + i] - A.gth[s + i];
    g.sync();
    proj_segment(g, dual_kind(b.kind), PDCS_SCALE_INVERT, A.tx0 + s, A.tx0 + s, A.d2 + s, dim, A.err);
    g.sync();
    for (int i = g.rank; i < dim; i += g.size) {
      const double lam = A.c[s + i] - A.gth[s + i];
      const double v = lam - A.tx0[s + i];
      acc[GT_RD2] += v * v;
    }
  }
}

// Exponential-cone blocks (always 3-dimensional, block-uniform scale): one
// thread per block with straight-line code, no generic segment machinery.
__device__ __forceinline__ void exp_or_dual(int kind, const double* v, double* o, int* err,
                                            double* rho = nullptr, RootCfg rc = RootCfg()) {
  if (kind == PDCS_EXP) proj_exp3(v[0], v[1], v[2], o, err, rho, rc);
  else proj_dual_exp3(v[0], v[1], v[2], o, err, rho, rc);
}

__device__ __forceinline__ bool exp_or_dual_fast(int kind, const double* v, double* o, int* err,
                                                 double* rho) {
  if (kind == PDCS_EXP) return proj_exp3_fast(v[0], v[1], v[2], o, err, rho);
  return proj_dual_exp3_fast(v[0], v[1], v[2], o, err, rho);
}

template <int OP, int MINB = 4>
__global__ void __launch_bounds__(BS, MINB) k_blk_exp(const PdcsBlock* tab, int nb, KArgs A, BlkParams P,
                                                double* part, int cap, int slot0, int gate) {
  if (gated(A.ctrl, gate)) return;
  constexpr int NQ = OpNQ<OP>::v;
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  int err = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) {
    const PdcsBlock b = tab[i];
    const int s = b.start;
    double v[3], o[3];
    if (OP == OP_PROJECT) {
      for (int q = 0; q < 3; ++q) v[q] = P.in[s + q];
      exp_or_dual(P.dualize ? dual_kind(b.kind) : b.kind, v, o, &err, nullptr, P.rc);
      for (int q = 0; q < 3; ++q) P.out[s + q] = o[q];
    } else if (OP == OP_STEP_X) {
      for (int q = 0; q < 3; ++q) v[q] = A.xh[s + q];
      exp_or_dual(b.kind, v, o, &err);
      for (int q = 0; q < 3; ++q) {
        const int j = s + q;
        const double xn = A.x[j], p = o[q];
        A.xh[j] = p;
        A.xt[j] = 2.0 * p - xn;
        const double d = p - xn;
        acc[GX_XX] += xn * xn;
        acc[GX_DXDX] += d * d;
        acc[GX_CX] += A.c[j] * p;
      }
    } else if (OP == OP_STEP_Y) {
      for (int q = 0; q < 3; ++q) v[q] = A.yh[s + q];
      double* rho = A.exp_rho ? A.exp_rho + 2 * (size_t)i : nullptr;  // warm starts
      exp_or_dual(dual_kind(b.kind), v, o, &err, rho);
      double res[3], rp[3];
      for (int q = 0; q < 3; ++q) res[q] = A.gxh[s + q] - A.h[s + q];
      exp_or_dual(b.kind, res, rp, &err, rho ? rho + 1 : nullptr);
      for (int q = 0; q < 3; ++q) {
        const int r = s + q;
        const double yn = A.y[r], p = o[q], hi = A.h[r];
        A.yh[r] = p;
        const double dy = p - yn;
        acc[GY_YY] += yn * yn;
        acc[GY_DYDY] += dy * dy;
        acc[GY_INTER] += dy * (A.w[r] - A.gx[r]);
        const double viol = res[q] - rp[q];
        acc[GY_RP2] += viol * viol;
        acc[GY_YH] += p * hi;
      }
    } else if (OP == OP_TLAM) {
      for (int q = 0; q < 3; ++q) v[q] = A.c[s + q] - A.gth[s + q];
      exp_or_dual(dual_kind(b.kind), v, o, &err);
      for (int q = 0; q < 3; ++q) {
        const double dv = v[q] - o[q];
        acc[GT_RD2] += dv * dv;
      }
    }
  }
  if (err) set_err(A.err, err);
  if (OP != OP_PROJECT) block_store_mask<NQ>(acc, 0u, part, cap, slot0 + blockIdx.x);
}

// Exponential-cone blocks of the y-step in two launches (C3: 1M blocks).  In
// one thread-per-block kernel the warps of the common case -- cheap cases
// and the warm-started Newton -- wait for the few lanes whose blocks need the
// reference's bracket + safeguarded Newton + bisection (up to 100 h
// evaluations).  So:
//  (1) k_exp_y_fast: CTA c owns blocks [c*per, (c+1)*per).  A block whose two
//      projections (y_hat onto the dual kind, the residual onto the kind)
//      are both decided by the fast path is finished here; otherwise nothing
//      of it is written and its index is queued, in block order, in CTA c's
//      queue (warp ballots + a CTA prefix: deterministic).
//  (2) k_exp_y_slow: CTA c runs the full projections of its queue -- exactly
//      the computation k_blk_exp<OP_STEP_Y> does for those blocks.
// Each block's result is the single-kernel result bit for bit; the line-search
// sums are per-CTA partials in fixed slots (deterministic).
__device__ __forceinline__ void exp_y_finish(const KArgs& A, int s, const double* o,
                                             const double* res, const double* rp, double* acc) {
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int r = s + q;
    const double yn = A.y[r], p = o[q], hi = A.h[r];
    A.yh[r] = p;
    const double dy = p - yn;
    acc[GY_YY] += yn * yn;
    acc[GY_DYDY] += dy * dy;
    acc[GY_INTER] += dy * (A.w[r] - A.gx[r]);
    const double viol = res[q] - rp[q];
    acc[GY_RP2] += viol * viol;
    acc[GY_YH] += p * hi;
  }
}

template <int MINB>
__global__ void __launch_bounds__(BS, MINB) k_exp_y_fast(const PdcsBlock* tab, int nb, int per, KArgs A,
                                                   int* queue, int* qcount, double* part, int cap,
                                                   int slot0, int gate) {
  if (gated(A.ctrl, gate)) return;
  __shared__ int wcnt[BS / 32];
  double acc[GY_N] = {0.0, 0.0, 0.0, 0.0, 0.0};
  int err = 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int b0 = blockIdx.x * per, b1 = min(nb, b0 + per);
  int qn = 0;
  for (int c = b0; c < b1; c += BS) {
    const int i = c + threadIdx.x;
    bool miss = false;
    if (i < b1) {
      const PdcsBlock b = tab[i];
      const int s = b.start;
      double v[3], o[3], res[3], rp[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        v[q] = A.yh[s + q];
        res[q] = A.gxh[s + q] - A.h[s + q];
      }
      double rho0 = A.exp_rho[2 * (size_t)i], rho1 = A.exp_rho[2 * (size_t)i + 1];
      int e = 0;
      const bool ok = exp_or_dual_fast(dual_kind(b.kind), v, o, &e, &rho0) &&
                      exp_or_dual_fast(b.kind, res, rp, &e, &rho1);
      if (ok) {
        A.exp_rho[2 * (size_t)i] = rho0;
        A.exp_rho[2 * (size_t)i + 1] = rho1;
        exp_y_finish(A, s, o, res, rp, acc);
        err |= e;
      } else {
        miss = true;
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, miss);
    if (lane == 0) wcnt[wid] = __popc(bal);
    __syncthreads();
    int off = qn, tot = 0;
#pragma unroll
    for (int w = 0; w < BS / 32; ++w) {
      const int cw = wcnt[w];
      if (w < wid) off += cw;
      tot += cw;
    }
    if (miss) queue[b0 + off + __popc(bal & ((1u << lane) - 1u))] = i;
    qn += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) qcount[blockIdx.x] = qn;
  if (err) set_err(A.err, err);
  block_store_mask<GY_N>(acc, 0u, part, cap, slot0 + blockIdx.x);
}

__global__ void __launch_bounds__(BS, 2) k_exp_y_slow(const PdcsBlock* tab, int per, KArgs A,
                                                   const int* queue, const int* qcount, double* part,
                                                   int cap, int slot0, int gate) {
  if (gated(A.ctrl, gate)) return;
  double acc[GY_N] = {0.0, 0.0, 0.0, 0.0, 0.0};
  int err = 0;
  const int cnt = qcount[blockIdx.x];
  for (int k = threadIdx.x; k < cnt; k += BS) {
    const int i = queue[blockIdx.x * per + k];
    const PdcsBlock b = tab[i];
    const int s = b.start;
    double v[3], o[3], res[3], rp[3];
    for (int q = 0; q < 3; ++q) {
      v[q] = A.yh[s + q];
      res[q] = A.gxh[s + q] - A.h[s + q];
    }
    double* rho = A.exp_rho + 2 * (size_t)i;
    exp_or_dual(dual_kind(b.kind), v, o, &err, rho);
    exp_or_dual(b.kind, res, rp, &err, rho + 1);
    exp_y_finish(A, s, o, res, rp, acc);
  }
  if (err) set_err(A.err, err);
  block_store_mask<GY_N>(acc, 0u, part, cap, slot0 + blockIdx.x);
}

template <int OP>
__global__ void __launch_bounds__(BS) k_blk_thread(const PdcsBlock* tab, int nb, KArgs A,
                                                   BlkParams P, double* part, int cap, int slot0,
                                                   int gate) {
  if (gated(A.ctrl, gate)) return;
  constexpr int NQ = OpNQ<OP>::v;
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  ThreadGrp g;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x)
    do_block<ThreadGrp, OP>(g, tab[i], A, P, acc);
  if (OP != OP_PROJECT) block_store_mask<NQ>(acc, 0u, part, cap, slot0 + blockIdx.x);
}

// Small blocks (THREAD_CLASS_MAX < dim <= HALF_CLASS_MAX): 16 lanes per
// block, two blocks per warp.
// W lanes per block (16, or 4: shorter reductions, several rows per lane)
template <int OP, int MINB = 1, int W = 16>
__global__ void __launch_bounds__(BS, MINB) k_blk_half(const PdcsBlock* tab, int nb, KArgs A,
                                                 BlkParams P, double* part, int cap, int slot0,
                                                 int gate) {
  if (gated(A.ctrl, gate)) return;
  constexpr int NQ = OpNQ<OP>::v;
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  SubGrp<W> g;
  const int gi = (blockIdx.x * blockDim.x + threadIdx.x) / W;
  const int gn = (gridDim.x * blockDim.x) / W;
  for (int i = gi; i < nb; i += gn) do_block<SubGrp<W>, OP>(g, tab[i], A, P, acc);
  __syncwarp();
  if (OP != OP_PROJECT) block_store_mask<NQ>(acc, 0u, part, cap, slot0 + blockIdx.x);
}

template <int OP>
__global__ void __launch_bounds__(BS) k_blk_warp(const PdcsBlock* tab, int nb, KArgs A,
                                                 BlkParams P, double* part, int cap, int slot0,
                                                 int gate) {
  if (gated(A.ctrl, gate)) return;
  constexpr int NQ = OpNQ<OP>::v;
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  WarpGrp g;
  const int wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int wt = gridDim.x * (blockDim.x >> 5);
  for (int i = wg; i < nb; i += wt) do_block<WarpGrp, OP>(g, tab[i], A, P, acc);
  if (OP != OP_PROJECT) block_store_mask<NQ>(acc, 0u, part, cap, slot0 + blockIdx.x);
}

template <int OP>
__global__ void __launch_bounds__(CTA_BLOCK_THREADS) k_blk_cta(const PdcsBlock* tab, int nb,
                                                               KArgs A, BlkParams P, double* part,
                                                               int cap, int slot0, int gate) {
  if (gated(A.ctrl, gate)) return;
  constexpr int NQ = OpNQ<OP>::v;
  __shared__ double sh[33];
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  CtaGrp g(sh);
  for (int i = blockIdx.x; i < nb; i += gridDim.x) do_block<CtaGrp, OP>(g, tab[i], A, P, acc);
  if (OP != OP_PROJECT) block_store_mask<NQ>(acc, 0u, part, cap, slot0 + blockIdx.x);
}

// ---------------------------------------------------------------------------
// Fused step kernels of one line-search trial
// ---------------------------------------------------------------------------

// x-space: pending Halpern/average of the previous iteration, then the primal
// candidate x_hat = P_X(x - tau (c - G^T y)), x~ = 2 x_hat - x and the
// reductions ||x||^2, ||x_hat - x||^2, c.x_hat (engine.py:155-161, 207-218,
// 246-277, 602-610).  Cone coordinates are left unprojected for k_blk_*.
template <bool H>
__global__ void __launch_bounds__(BS, 8) k_step_x(KArgs A, double* part, int cap) {
  pdl_enter();
  const PdcsCtrl* C = A.ctrl;
  if (C->stop) return;
  // the Halpern / step coefficients live in shared memory (register pressure)
  __shared__ double kc[8];
  if (threadIdx.x == 0) {
    kc[0] = C->pa; kc[1] = C->pb; kc[2] = C->pbeta; kc[3] = C->peta; kc[4] = C->pW; kc[5] = C->tau;
    kc[6] = 1.0 + C->pbeta; kc[7] = C->pW + C->peta;
  }
  __syncthreads();
  const double &a = kc[0], &b = kc[1], &be = kc[2], &et = kc[3], &W = kc[4], &tau = kc[5];
  const double &opb = kc[6], &tot = kc[7];
  const bool pend = C->pending != 0;
  const bool inject = C->nan_after >= 0 && C->n_primal_proj >= C->nan_after;
  double acc[GX_N] = {0.0, 0.0, 0.0};
  const uint64_t ps = policy_stream(), pk = policy_keep_frac(A.keep_xt);
  for (int j = A.x0 + blockIdx.x * blockDim.x + threadIdx.x; j < A.x1; j += gridDim.x * blockDim.x) {
    double xn, gn;
    if (pend) {
      const double xo = ldc_hint<H>(A.x + j, ps);
      xn = a * (opb * ldc_hint<H>(A.xh + j, ps) - be * xo) + b * ld_hint<H>(A.xa + j, ps);
      const double go = ldc_hint<H>(A.gty + j, ps);
      gn = a * (opb * ld_hint<H>(A.gth + j, ps) - be * go) + b * ld_hint<H>(A.gtya + j, ps);
      st_hint<H>(A.xb + j, (W == 0.0) ? xn : (W * ldc_hint<H>(A.xb + j, ps) + et * xn) / tot, ps);
      st_hint<H>(A.x + j, xn, ps);
      st_hint<H>(A.gty + j, gn, ps);
    } else {
      xn = ldc_hint<H>(A.x + j, ps);
      gn = ldc_hint<H>(A.gty + j, ps);
    }
    const double cj = ld_hint<H>(A.c + j, ps);
    const double v = xn - tau * (cj - gn);
    if (j < A.nbox) {
      double lj, uj;
      box_bounds<H>(A, j, ps, lj, uj);
      double p = clampv(v, lj, uj);
      if (j == 0 && inject) p = __longlong_as_double(0x7ff8000000000000ll);
      st_hint<H>(A.xh + j, p, ps);
      st_hint<H>(A.xt + j, 2.0 * p - xn, pk);
      const double d = p - xn;
      acc[GX_XX] += xn * xn;
      acc[GX_DXDX] += d * d;
      acc[GX_CX] += cj * p;
    } else {
      A.xh[j] = v;
    }
  }
  block_store_mask<GX_N>(acc, 0u, part, cap, blockIdx.x);
}

// ---- tiled CSR-stream SpMV ---------------------------------------------------
// A tile is up to TILE_ROWS consecutive rows holding at most TILE_NNZ entries
// (of the current panel).  Phase 1 streams the tile's (col, val) coalesced and
// issues all of its gathers at once, parking the products in shared memory;
// phase 2 gives each row to one thread, which adds its products in index
// order -- the exact rounding sequence of scipy's csr_matvec (s += a*x).
struct TileSrc {
  const int* tiles;     // [ntiles + 1] first row of each tile
  int ntiles;
  const int* po;        // row offsets of this pass (panel) into ci/va
  const int* ci;
  const double* va;
  const double* wpart;  // partial sums of the previous passes (nullptr: start at 0)
  const int* orig_rp;   // rows longer than long_t in the CSR take longv (nullptr: none)
  int long_t;
};

__device__ __forceinline__ double tile_rows(const TileSrc& S, const double* __restrict__ x,
                                            const double* longv, int r0, int nr, double* prod,
                                            int* rs) {
  const int base = __ldg(S.po + r0);
  const int tnnz = __ldg(S.po + r0 + nr) - base;
  for (int i = threadIdx.x; i <= nr; i += blockDim.x) rs[i] = __ldg(S.po + r0 + i) - base;
  const int* __restrict__ ci = S.ci + base;
  const double* __restrict__ va = S.va + base;
  int k = threadIdx.x;
  for (; k + 3 * BS < tnnz; k += 4 * BS) {
    const int c0 = __ldg(ci + k), c1 = __ldg(ci + k + BS), c2 = __ldg(ci + k + 2 * BS),
              c3 = __ldg(ci + k + 3 * BS);
    const double a0 = __ldg(va + k), a1 = __ldg(va + k + BS), a2 = __ldg(va + k + 2 * BS),
                 a3 = __ldg(va + k + 3 * BS);
    const double x0 = __ldg(x + c0), x1 = __ldg(x + c1), x2 = __ldg(x + c2), x3 = __ldg(x + c3);
    prod[k] = a0 * x0;
    prod[k + BS] = a1 * x1;
    prod[k + 2 * BS] = a2 * x2;
    prod[k + 3 * BS] = a3 * x3;
  }
  for (; k < tnnz; k += BS) prod[k] = __ldg(va + k) * __ldg(x + __ldg(ci + k));
  __syncthreads();
  double s = 0.0;
  const int i = threadIdx.x;
  if (i < nr) {
    const int r = r0 + i;
    const bool lng = S.orig_rp && (__ldg(S.orig_rp + r + 1) - __ldg(S.orig_rp + r)) > S.long_t;
    if (lng) {
      s = longv[r];
    } else {
      if (S.wpart) s = S.wpart[r];
      for (int q = rs[i]; q < rs[i + 1]; ++q) s += prod[q];
    }
  }
  return s;
}

// One partial pass of a panelled SpMV (all panels but the last).
__global__ void __launch_bounds__(BS) k_tile_pass(TileSrc S, const double* __restrict__ x,
                                                  double* wout, const PdcsCtrl* ctrl, int gate) {
  if (gated(ctrl, gate)) return;
  __shared__ double prod[TILE_NNZ];
  __shared__ int rs[TILE_ROWS + 1];
  for (int t = blockIdx.x; t < S.ntiles; t += gridDim.x) {
    const int r0 = __ldg(S.tiles + t), nr = __ldg(S.tiles + t + 1) - r0;
    const double s = tile_rows(S, x, nullptr, r0, nr, prod, rs);
    if (threadIdx.x < nr) wout[r0 + threadIdx.x] = s;
    __syncthreads();
  }
}

// ---- giant SOC blocks in the y-step: the whole grid cooperates ---------------
// A dual SOC block far larger than a CTA (C4: one block of 500,042 rows) is
// projected in three launches: (A) grid-wide partial sums of ||v[1:]||^2 for
// the dual projection of v = y + sigma(h - w) and of the residual
// r = gx_hat - h; (B) one CTA turns them into the SOC case and coefficients
// (cones.py:54-67); (C) the grid applies both projections and accumulates the
// line-search / beta reductions of the block's rows.  Scales are uniform
// (dual SOC blocks are made block-uniform by the preconditioner).
__global__ void __launch_bounds__(BS) k_giant_soc_a(const PdcsBlock* tab, int nb, KArgs A,
                                                    double* gpart, int gcap) {
  if (A.ctrl->stop) return;
  for (int b = 0; b < nb; ++b) {
    const PdcsBlock B = tab[b];
    double acc[2] = {0.0, 0.0};
    for (int i = B.start + 1 + blockIdx.x * blockDim.x + threadIdx.x; i < B.start + B.dim;
         i += gridDim.x * blockDim.x) {
      const double v = A.yh[i];
      const double r = A.gxh[i] - A.h[i];
      acc[0] += v * v;
      acc[1] += r * r;
    }
    block_store_mask<2>(acc, 0u, gpart + (size_t)b * 2 * gcap, gcap, blockIdx.x);
  }
}

// coefficients per block: [mode_v, ratio_v, first_v, mode_r, ratio_r, first_r]
// mode 0 = keep, 1 = zero, 2 = scale (first element = coef, rest * coef/nx)
__global__ void k_giant_soc_b(const PdcsBlock* tab, int nb, KArgs A, const double* gpart, int gcap,
                              int nslots, double* gcoef) {
  if (A.ctrl->stop) return;
  __shared__ double sh[33];
  CtaGrp g(sh);
  for (int b = 0; b < nb; ++b) {
    const PdcsBlock B = tab[b];
    const double* p = gpart + (size_t)b * 2 * gcap;
    double sv = 0.0, sr = 0.0;
    for (int s = threadIdx.x; s < nslots; s += blockDim.x) {
      sv += p[s];
      sr += p[gcap + s];
    }
    sv = g.sum(sv);
    sr = g.sum(sr);
    if (threadIdx.x == 0) {
      const double t[2] = {A.yh[B.start], A.gxh[B.start] - A.h[B.start]};
      const double nx[2] = {sqrt(sv), sqrt(sr)};
      for (int q = 0; q < 2; ++q) {
        double mode = 2.0, ratio = 0.0, first = 0.0;
        if (nx[q] <= t[q]) {
          mode = 0.0;
        } else if (nx[q] <= -t[q]) {
          mode = 1.0;
        } else {
          first = 0.5 * (t[q] + nx[q]);
          ratio = first / nx[q];
        }
        gcoef[b * 8 + 3 * q + 0] = mode;
        gcoef[b * 8 + 3 * q + 1] = ratio;
        gcoef[b * 8 + 3 * q + 2] = first;
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(BS) k_giant_soc_c(const PdcsBlock* tab, int nb, KArgs A,
                                                    const double* gcoef, double* part, int cap,
                                                    int slot0) {
  if (A.ctrl->stop) return;
  double acc[GY_N] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int b = 0; b < nb; ++b) {
    const PdcsBlock B = tab[b];
    const double mv = gcoef[b * 8 + 0], rv = gcoef[b * 8 + 1], fv = gcoef[b * 8 + 2];
    const double mr = gcoef[b * 8 + 3], rr = gcoef[b * 8 + 4], fr = gcoef[b * 8 + 5];
    for (int i = B.start + blockIdx.x * blockDim.x + threadIdx.x; i < B.start + B.dim;
         i += gridDim.x * blockDim.x) {
      const double v = A.yh[i];
      const double hi = A.h[i];
      const double res = A.gxh[i] - hi;
      const bool head = i == B.start;
      const double p = mv == 0.0 ? v : (mv == 1.0 ? 0.0 : (head ? fv : rv * v));
      const double rp = mr == 0.0 ? res : (mr == 1.0 ? 0.0 : (head ? fr : rr * res));
      A.yh[i] = p;
      const double yn = A.y[i];
      const double dy = p - yn;
      acc[GY_YY] += yn * yn;
      acc[GY_DYDY] += dy * dy;
      acc[GY_INTER] += dy * (A.w[i] - A.gx[i]);
      const double viol = res - rp;
      acc[GY_RP2] += viol * viol;
      acc[GY_YH] += p * hi;
    }
  }
  block_store_mask<GY_N>(acc, 0u, part, cap, slot0 + blockIdx.x);
}

// Giant SOC blocks in plain projections (check path: gap probes, metrics,
// project_set): the same three grid-wide phases on out = P_SOC(in).  Giant
// blocks are uniform-scale SOC blocks, so every scaled or dualised form of the
// projection is the plain SOC projection.
__global__ void __launch_bounds__(BS) k_giant_proj_a(const PdcsBlock* tab, int nb,
                                                     const double* __restrict__ in, double* gpart,
                                                     int gcap) {
  for (int b = 0; b < nb; ++b) {
    const PdcsBlock B = tab[b];
    double acc[1] = {0.0};
    for (int i = B.start + 1 + blockIdx.x * blockDim.x + threadIdx.x; i < B.start + B.dim;
         i += gridDim.x * blockDim.x) {
      const double v = in[i];
      acc[0] += v * v;
    }
    block_store_mask<1>(acc, 0u, gpart + (size_t)b * 2 * gcap, gcap, blockIdx.x);
  }
}

__global__ void k_giant_proj_b(const PdcsBlock* tab, int nb, const double* in, const double* gpart,
                               int gcap, int nslots, double* gcoef) {
  __shared__ double sh[33];
  CtaGrp g(sh);
  for (int b = 0; b < nb; ++b) {
    const PdcsBlock B = tab[b];
    const double* p = gpart + (size_t)b * 2 * gcap;
    double sv = 0.0;
    for (int s = threadIdx.x; s < nslots; s += blockDim.x) sv += p[s];
    sv = g.sum(sv);
    if (threadIdx.x == 0) {
      const double t = in[B.start], nx = sqrt(sv);
      double mode = 2.0, ratio = 0.0, first = 0.0;
      if (nx <= t) {
        mode = 0.0;
      } else if (nx <= -t) {
        mode = 1.0;
      } else {
        first = 0.5 * (t + nx);
        ratio = first / nx;
      }
      gcoef[b * 8 + 0] = mode;
      gcoef[b * 8 + 1] = ratio;
      gcoef[b * 8 + 2] = first;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(BS) k_giant_proj_c(const PdcsBlock* tab, int nb, const double* in,
                                                     double* out, const double* gcoef) {
  for (int b = 0; b < nb; ++b) {
    const PdcsBlock B = tab[b];
    const double mv = gcoef[b * 8 + 0], rv = gcoef[b * 8 + 1], fv = gcoef[b * 8 + 2];
    for (int i = B.start + blockIdx.x * blockDim.x + threadIdx.x; i < B.start + B.dim;
         i += gridDim.x * blockDim.x) {
      const double v = in[i];
      out[i] = mv == 0.0 ? v : (mv == 1.0 ? 0.0 : (i == B.start ? fv : rv * v));
    }
  }
}

// ---- per-row epilogues of the fused step kernels -----------------------------
struct YCoef {
  bool pend;
  double a, b, be, et, W, sigma, opb, tot;
};

__device__ __forceinline__ YCoef y_coef(const PdcsCtrl* C) {
  YCoef k;
  k.pend = C->pending != 0;
  k.a = C->pa; k.b = C->pb; k.be = C->pbeta; k.et = C->peta; k.W = C->pW; k.sigma = C->sigma;
  k.opb = 1.0 + k.be;
  k.tot = k.W + k.et;
  return k;
}

// y-space row r with dot = (G^ x~)_r: pending Halpern/average, then
// y_hat = P_Y(y + sigma (h - w)), gx_hat = (w + gx)/2 and the reductions
// ||y||^2, ||dy||^2, dy.(w - gx), the beta residual ||r - P_{K_d*} r||^2 of
// r = gx_hat - h, and y_hat.h.  Block rows are left for k_blk_*.
template <bool H>
__device__ __forceinline__ void y_epilogue(const KArgs& A, const YCoef& k, int r, double dot,
                                           double* acc, uint64_t ps, uint64_t pk) {
  double yn, gn;
  if (k.pend) {
    const double yo = ldc_hint<H>(A.y + r, ps);
    yn = k.a * (k.opb * ldc_hint<H>(A.yh + r, ps) - k.be * yo) + k.b * ld_hint<H>(A.ya + r, ps);
    const double go = ldc_hint<H>(A.gx + r, ps);
    gn = k.a * (k.opb * ldc_hint<H>(A.gxh + r, ps) - k.be * go) + k.b * ld_hint<H>(A.gxa + r, ps);
    st_hint<H>(A.yb + r, (k.W == 0.0) ? yn : (k.W * ldc_hint<H>(A.yb + r, ps) + k.et * yn) / k.tot, ps);
    st_hint<H>(A.y + r, yn, ps);
    st_hint<H>(A.gx + r, gn, ps);
  } else {
    yn = ldc_hint<H>(A.y + r, ps);
    gn = ldc_hint<H>(A.gx + r, ps);
  }
  const double hi = ld_hint<H>(A.h + r, ps);
  const double v = yn + k.sigma * (hi - dot);
  const double gh = 0.5 * (dot + gn);
  st_hint<H>(A.gxh + r, gh, ps);
  if (r < A.m_elem) {
    const bool zero = r < A.m_zero;
    const double p = zero ? v : pos_part(v);
    st_hint<H>(A.yh + r, p, pk);
    const double dy = p - yn;
    acc[GY_YY] += yn * yn;
    acc[GY_DYDY] += dy * dy;
    acc[GY_INTER] += dy * (dot - gn);
    const double res = gh - hi;
    const double viol = zero ? res : res - pos_part(res);
    acc[GY_RP2] += viol * viol;
    acc[GY_YH] += p * hi;
  } else {
    A.yh[r] = v;
    A.w[r] = dot;
  }
}

// x-space row j with dot = (G^T y_hat)_j: stores gth and the box part of the
// dual residual of beta, ||lam1 - P_Lambda lam1||^2, and the bound terms of
// the dual objective (model.py:182-237, termination.py:113-119).
template <bool H, bool STORE = true>
__device__ __forceinline__ void t_epilogue(const KArgs& A, int j, double dot, double* acc,
                                           uint64_t ps) {
  if (STORE) st_hint<H>(A.gth + j, dot, ps);
  if (j < A.nbox) {
    const double lam = ld_hint<H>(A.c + j, ps) - dot;
    double lj, uj;
    box_bounds<H>(A, j, ps, lj, uj);
    const bool lf = isfinite(lj), uf = isfinite(uj);
    const double pr = (!lf && !uf) ? 0.0 : (!lf ? neg_clip(lam) : (!uf ? pos_part(lam) : lam));
    const double v = lam - pr;
    acc[GT_RD2] += v * v;
    if (lf) acc[GT_LSUM] += lj * pos_part(lam);
    if (uf) acc[GT_USUM] += uj * pos_part(-lam);
  }
}

// Sharded mode: the x-space epilogue of the G^T step after the all-reduce
// of the G^T y_hat partial sums (accepted trials only).
__global__ void __launch_bounds__(BS) k_t_epilogue(KArgs A, double* part, int cap) {
  const PdcsCtrl* C = A.ctrl;
  if (C->stop || !C->accepted) return;
  double acc[GT_N] = {0.0, 0.0, 0.0};
  for (int j = A.x0 + blockIdx.x * blockDim.x + threadIdx.x; j < A.x1; j += gridDim.x * blockDim.x)
    t_epilogue<false>(A, j, A.gth[j], acc, 0);
  block_store_mask<GT_N>(acc, 0u, part, cap, blockIdx.x);
}

// ---- tiled (CSR-stream) step kernels -----------------------------------------
// SOC: the dual SOC blocks (block-uniform scales, each inside one tile: the
// tiles are cut at block boundaries) are projected here, in the tile, instead
// of by k_blk_half after the kernel (C2: 10k SOC(11) blocks).  `rowhead[r]` is
// the first row of row r's block (or -1).  For a block with rows [b, b+d):
// v = y + sigma (h - w) is projected onto the SOC (the dual kind, cones.py:
// 436-443), the residual gx_hat - h onto K_d* = SOC (cones.py:523-530) --
// both plain SOC projections under uniform scales (cones.py:54-67) -- with the
// norms of the tails summed by the head row's thread in index order.
template <bool SOC>
__global__ void __launch_bounds__(BS, 5) k_step_y(KArgs A, TileSrc S, double* part, int cap,
                                                  CtrlFuse F, const int* __restrict__ rowhead) {
  const PdcsCtrl* C = A.ctrl;
  if (C->stop) return;
  __shared__ double prod[TILE_NNZ];
  __shared__ int rs[TILE_ROWS + 1];
  __shared__ YCoef ks;  // coefficients in shared memory (register pressure)
  __shared__ double sv[SOC ? TILE_ROWS : 1], sr[SOC ? TILE_ROWS : 1];
  // per head row: (mode 0 keep / 1 zero / 2 scale, head value, tail ratio)
  __shared__ double cv[SOC ? TILE_ROWS : 1][3], cr[SOC ? TILE_ROWS : 1][3];
  if (threadIdx.x == 0) ks = y_coef(C);
  __syncthreads();
  const YCoef& k = ks;
  double acc[GY_N] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int t = blockIdx.x; t < S.ntiles; t += gridDim.x) {
    const int r0 = __ldg(S.tiles + t), nr = __ldg(S.tiles + t + 1) - r0;
    const double dot = tile_rows(S, A.xt, A.w, r0, nr, prod, rs);
    const int i = threadIdx.x, r = r0 + i;
    if (!SOC || r >= A.m_elem || i >= nr) {
      if (i < nr && (!SOC || r < A.m_elem)) y_epilogue<false>(A, k, r, dot, acc, 0, 0);
    }
    if (SOC) {
      // block rows: pending Halpern, pre-projection values into shared memory
      const bool blk = i < nr && r >= A.m_elem;
      double yn = 0.0, hi = 0.0, v = 0.0, res = 0.0, gn = 0.0;
      int head = -1;
      if (blk) {
        if (k.pend) {
          const double yo = A.y[r];
          yn = k.a * (k.opb * A.yh[r] - k.be * yo) + k.b * A.ya[r];
          const double go = A.gx[r];
          gn = k.a * (k.opb * A.gxh[r] - k.be * go) + k.b * A.gxa[r];
          A.yb[r] = (k.W == 0.0) ? yn : (k.W * A.yb[r] + k.et * yn) / k.tot;
          A.y[r] = yn;
          A.gx[r] = gn;
        } else {
          yn = A.y[r];
          gn = A.gx[r];
        }
        hi = A.h[r];
        v = yn + k.sigma * (hi - dot);
        const double gh = 0.5 * (dot + gn);
        A.gxh[r] = gh;
        A.w[r] = dot;
        res = gh - hi;
        sv[i] = v;
        sr[i] = res;
        head = __ldg(rowhead + r) - r0;
      }
      __syncthreads();
      if (blk && head == i) {
        // the block's rows are [r, r + d): d from the next head or the tile end
        int d = 1;
        while (i + d < nr && __ldg(rowhead + r + d) == r) ++d;
        double nv = 0.0, nres = 0.0;
        for (int j = 1; j < d; ++j) {
          nv += sv[i + j] * sv[i + j];
          nres += sr[i + j] * sr[i + j];
        }
        nv = sqrt(nv);
        nres = sqrt(nres);
        const double tv = sv[i], tr = sr[i];
        // cones.py:54-67: keep if ||x|| <= t, zero if ||x|| <= -t, else
        // ((t + ||x||)/2) (1, x/||x||) -- the tail as coef/||x|| * x
        if (nv <= tv) { cv[i][0] = 0.0; } else if (nv <= -tv) { cv[i][0] = 1.0; }
        else { cv[i][0] = 2.0; cv[i][1] = 0.5 * (tv + nv); cv[i][2] = cv[i][1] / nv; }
        if (nres <= tr) { cr[i][0] = 0.0; } else if (nres <= -tr) { cr[i][0] = 1.0; }
        else { cr[i][0] = 2.0; cr[i][1] = 0.5 * (tr + nres); cr[i][2] = cr[i][1] / nres; }
      }
      __syncthreads();
      if (blk) {
        const double mv = cv[head][0], mr = cr[head][0];
        double p, rp;
        if (mv == 0.0) p = v;
        else if (mv == 1.0) p = 0.0;
        else p = head == i ? cv[head][1] : cv[head][2] * v;
        if (mr == 0.0) rp = res;
        else if (mr == 1.0) rp = 0.0;
        else rp = head == i ? cr[head][1] : cr[head][2] * res;
        A.yh[r] = p;
        const double dy = p - yn;
        acc[GY_YY] += yn * yn;
        acc[GY_DYDY] += dy * dy;
        acc[GY_INTER] += dy * (dot - gn);
        const double viol = res - rp;
        acc[GY_RP2] += viol * viol;
        acc[GY_YH] += p * hi;
      }
    }
    __syncthreads();
  }
  block_store_mask<GY_N>(acc, 0u, part, cap, blockIdx.x);
  fused_ctrl(F);
}

__global__ void __launch_bounds__(BS, 4) k_step_t(KArgs A, TileSrc S, double* part, int cap,
                                                  CtrlFuse F) {
  const PdcsCtrl* C = A.ctrl;
  if (C->stop || !C->accepted) return;
  __shared__ double prod[TILE_NNZ];
  __shared__ int rs[TILE_ROWS + 1];
  double acc[GT_N] = {0.0, 0.0, 0.0};
  for (int t = blockIdx.x; t < S.ntiles; t += gridDim.x) {
    const int r0 = __ldg(S.tiles + t), nr = __ldg(S.tiles + t + 1) - r0;
    const double dot = tile_rows(S, A.yh, A.gtr, r0, nr, prod, rs);
    if (threadIdx.x < nr) t_epilogue<false>(A, r0 + threadIdx.x, dot, acc, 0);
    __syncthreads();
  }
  block_store_mask<GT_N>(acc, 0u, part, cap, blockIdx.x);
  fused_ctrl(F);
}

// ---- lane-mapped step kernels: VW lanes per row ------------------------------
template <int VW, int GP, bool H = false>
__device__ __forceinline__ double lane_row(const TileSrc& S, const double* __restrict__ x,
                                           const double* longv, int r, int sub, int nrows,
                                           uint64_t ps, uint64_t pk) {
  int b = 0, e = 0;
  double s = 0.0;
  if (r < nrows) {
    const bool lng = S.orig_rp && (__ldg(S.orig_rp + r + 1) - __ldg(S.orig_rp + r)) > S.long_t;
    if (lng) {
      if (sub == 0) s = longv[r];
    } else {
      b = ld_hint<H>(S.po + r, ps);
      e = ld_hint<H>(S.po + r + 1, ps);
      if (S.wpart && sub == 0) s = ld_hint<H>(S.wpart + r, ps);
    }
  }
  if (VW == 1) {
    // groups of up to 4 entries with predicated loads: a row of <= 4 entries
    // (every panel row of a short-row matrix) costs one round of dependent
    // loads instead of one per entry; the adds keep index order
    for (int j = b; j < e; j += 4) {
      const int q = e - j;
      const int c0 = ld_hint<H>(S.ci + j, ps);
      const int c1 = q > 1 ? ld_hint<H>(S.ci + j + 1, ps) : 0;
      const int c2 = q > 2 ? ld_hint<H>(S.ci + j + 2, ps) : 0;
      const int c3 = q > 3 ? ld_hint<H>(S.ci + j + 3, ps) : 0;
      const double a0 = ld_hint<H>(S.va + j, ps);
      const double a1 = q > 1 ? ld_hint<H>(S.va + j + 1, ps) : 0.0;
      const double a2 = q > 2 ? ld_hint<H>(S.va + j + 2, ps) : 0.0;
      const double a3 = q > 3 ? ld_hint<H>(S.va + j + 3, ps) : 0.0;
      const double x0 = ld_gather<GP>(x + c0);
      const double x1 = q > 1 ? ld_gather<GP>(x + c1) : 0.0;
      const double x2 = q > 2 ? ld_gather<GP>(x + c2) : 0.0;
      const double x3 = q > 3 ? ld_gather<GP>(x + c3) : 0.0;
      s += a0 * x0;
      if (q > 1) s += a1 * x1;
      if (q > 2) s += a2 * x2;
      if (q > 3) s += a3 * x3;
    }
  } else {
    for (int j = b + sub; j < e; j += VW)
      s += ld_hint<H>(S.va + j, ps) * ld_gather<GP>(x + ld_hint<H>(S.ci + j, ps));
#pragma unroll
    for (int off = VW / 2; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off, VW);
  }
  return s;
}

// HS: the pass's streams (row offsets, entries, partial sums in and out)
// carry the L2 evict_first policy so the gathered panel stays resident
// (PDCS_TUNE hs=1; C5 lab: 0.505 vs 0.517 ms per y-step, tools/c5_lab.cu)
template <int VW, int GP, bool HS = false>
__global__ void __launch_bounds__(BS) k_lane_pass(TileSrc S, int nrows, const double* __restrict__ x,
                                                  double* wout, const PdcsCtrl* ctrl, int gate,
                                                  float keep) {
  pdl_enter();
  if (gated(ctrl, gate)) return;
  const uint64_t ps = policy_stream(), pk = policy_keep_frac(keep);
  const int lane = threadIdx.x & 31, sub = lane & (VW - 1);
  constexpr int RPW = 32 / VW;
  const int wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int wt = gridDim.x * (blockDim.x >> 5);
  for (int base = wg * RPW; base < nrows; base += wt * RPW) {
    const int r = base + lane / VW;
    const double s = lane_row<VW, GP, HS>(S, x, nullptr, r, sub, nrows, ps, pk);
    if (sub == 0 && r < nrows) st_hint<HS>(wout + r, s, ps);
  }
}

// Class split (mixed row lengths): rows of <= CLS_SHORT entries are summed by
// the epilogue thread itself, in index order, and the product stored back
// (w / gth stay complete for the block kernels after the epilogue); the rows
// of the long class come from the k_rows_pass before it.
constexpr int CLS_SHORT = 6;
struct ShortRows {
  const int* rp;  // nullptr: every product comes from the pass (no class split)
  const int* ci;
  const double* va;
  const double* x;
};
__device__ __forceinline__ double cls_dot(const ShortRows& R, int r, double w, double* out) {
  if (R.rp == nullptr) return w;
  const int b = __ldg(R.rp + r), e = __ldg(R.rp + r + 1);
  if (e - b > CLS_SHORT) return w;
  double s = 0.0;
  for (int j = b; j < e; ++j) s += __ldg(R.va + j) * R.x[__ldg(R.ci + j)];
  out[r] = s;
  return s;
}

// Class split of G^T: the columns past the box (primal cone blocks) are
// projected by the block kernels after the epilogue, which read G^T y_hat
// from gth -- their short rows are summed and stored here.
__device__ __forceinline__ void cls_cone_cols(const KArgs& A, const ShortRows& R) {
  if (R.rp == nullptr) return;
  for (int j = A.nbox + blockIdx.x * blockDim.x + threadIdx.x; j < A.n; j += gridDim.x * blockDim.x)
    cls_dot(R, j, 0.0, A.gth);
}

// x-step of the primal exponential-cone coordinates in the block kernel itself
// (C3p: all 3M of its coordinates): each thread applies the pending Halpern
// update and forms the candidate v = x - tau (c - G^T y) of its block's three
// coordinates, then projects -- v makes no round trip through HBM and the
// x-step kernel only covers the box.  The same arithmetic as k_step_x +
// k_blk_exp<OP_STEP_X>.
template <int MINB>
__global__ void __launch_bounds__(BS, MINB) k_exp_xstep(const PdcsBlock* tab, int nb, KArgs A, double* part,
                                                        int cap, int slot0) {
  const PdcsCtrl* C = A.ctrl;
  if (C->stop) return;
  __shared__ double kc[8];
  if (threadIdx.x == 0) {
    kc[0] = C->pa; kc[1] = C->pb; kc[2] = C->pbeta; kc[3] = C->peta; kc[4] = C->pW; kc[5] = C->tau;
    kc[6] = 1.0 + C->pbeta; kc[7] = C->pW + C->peta;
  }
  __syncthreads();
  const double &a = kc[0], &b = kc[1], &be = kc[2], &et = kc[3], &W = kc[4], &tau = kc[5];
  const double &opb = kc[6], &tot = kc[7];
  const bool pend = C->pending != 0;
  double acc[GX_N] = {0.0, 0.0, 0.0};
  int err = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) {
    const PdcsBlock bk = tab[i];
    const int s = bk.start;
    double v[3], o[3], xv[3], cv[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int j = s + q;
      double xn, gn;
      if (pend) {
        const double xo = A.x[j];
        xn = a * (opb * A.xh[j] - be * xo) + b * A.xa[j];
        const double go = A.gty[j];
        gn = a * (opb * A.gth[j] - be * go) + b * A.gtya[j];
        A.xb[j] = (W == 0.0) ? xn : (W * A.xb[j] + et * xn) / tot;
        A.x[j] = xn;
        A.gty[j] = gn;
      } else {
        xn = A.x[j];
        gn = A.gty[j];
      }
      const double cj = A.c[j];
      v[q] = xn - tau * (cj - gn);
      xv[q] = xn;
      cv[q] = cj;
    }
    exp_or_dual(bk.kind, v, o, &err);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int j = s + q;
      const double p = o[q];
      A.xh[j] = p;
      A.xt[j] = 2.0 * p - xv[q];
      const double d = p - xv[q];
      acc[GX_XX] += xv[q] * xv[q];
      acc[GX_DXDX] += d * d;
      acc[GX_CX] += cv[q] * p;
    }
  }
  if (err) set_err(A.err, err);
  block_store_mask<GX_N>(acc, 0u, part, cap, slot0 + blockIdx.x);
}

// G^T y_hat rows of the primal exponential-cone coordinates and their
// lambda_2 projection in one kernel (C3p): each thread sums its block's three
// rows of G^T (index order, as the lane kernels), stores them in gth and
// projects c - G^T y_hat onto the dual cone for beta's dual residual -- the
// t-step kernel only covers the box.  The same arithmetic as the lane t-step
// + k_blk_exp<OP_TLAM>.
template <int MINB>
__global__ void __launch_bounds__(BS, MINB) k_exp_tstep(const PdcsBlock* tab, int nb, KArgs A, ShortRows R,
                                                        double* part, int cap, int slot0) {
  const PdcsCtrl* C = A.ctrl;
  if (C->stop || !C->accepted) return;
  double acc[GT_N] = {0.0, 0.0, 0.0};
  int err = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) {
    const PdcsBlock bk = tab[i];
    const int s = bk.start;
    double v[3], o[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int j = s + q;
      double d = 0.0;
      for (int k = __ldg(R.rp + j), e = __ldg(R.rp + j + 1); k < e; ++k) d += __ldg(R.va + k) * R.x[__ldg(R.ci + k)];
      A.gth[j] = d;
      v[q] = A.c[j] - d;
    }
    exp_or_dual(dual_kind(bk.kind), v, o, &err);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double dv = v[q] - o[q];
      acc[GT_RD2] += dv * dv;
    }
  }
  if (err) set_err(A.err, err);
  block_store_mask<GT_N>(acc, 0u, part, cap, slot0 + blockIdx.x);
}

// y-step of the exponential-cone rows in the block kernel itself (C3: 3M of
// its 3.001M rows): each thread forms its block's three products of G^ x~
// (index-order sums, as the lane kernels), the pending Halpern update and the
// dual candidate of y_epilogue, then projects -- the rows' v, w and gx_hat
// make no round trip through HBM and the step kernel only covers the
// elementwise rows.  The same arithmetic as y_epilogue + k_blk_exp<OP_STEP_Y>.
template <int MINB>
__global__ void __launch_bounds__(BS, MINB) k_exp_ystep(const PdcsBlock* tab, int nb, KArgs A, ShortRows R,
                                                        double* part, int cap, int slot0) {
  const PdcsCtrl* C = A.ctrl;
  if (C->stop) return;
  __shared__ YCoef ks;
  if (threadIdx.x == 0) ks = y_coef(C);
  __syncthreads();
  const YCoef& k = ks;
  double acc[GY_N] = {0.0, 0.0, 0.0, 0.0, 0.0};
  int err = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) {
    const PdcsBlock b = tab[i];
    const int s = b.start;
    double v[3], o[3], res[3], rp[3], yn[3], dg[3], hv[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int r = s + q;
      double d = 0.0;
      for (int j = __ldg(R.rp + r), e = __ldg(R.rp + r + 1); j < e; ++j) d += __ldg(R.va + j) * R.x[__ldg(R.ci + j)];
      double y0, g0;
      if (k.pend) {
        const double yo = A.y[r];
        y0 = k.a * (k.opb * A.yh[r] - k.be * yo) + k.b * A.ya[r];
        const double go = A.gx[r];
        g0 = k.a * (k.opb * A.gxh[r] - k.be * go) + k.b * A.gxa[r];
        A.yb[r] = (k.W == 0.0) ? y0 : (k.W * A.yb[r] + k.et * y0) / k.tot;
        A.y[r] = y0;
        A.gx[r] = g0;
      } else {
        y0 = A.y[r];
        g0 = A.gx[r];
      }
      const double hi = A.h[r];
      v[q] = y0 + k.sigma * (hi - d);
      const double gh = 0.5 * (d + g0);
      A.gxh[r] = gh;
      A.w[r] = d;
      res[q] = gh - hi;
      yn[q] = y0;
      dg[q] = d - g0;
      hv[q] = hi;
    }
    double* rho = A.exp_rho ? A.exp_rho + 2 * (size_t)i : nullptr;  // warm starts
    exp_or_dual(dual_kind(b.kind), v, o, &err, rho);
    exp_or_dual(b.kind, res, rp, &err, rho ? rho + 1 : nullptr);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double p = o[q];
      A.yh[s + q] = p;
      const double dy = p - yn[q];
      acc[GY_YY] += yn[q] * yn[q];
      acc[GY_DYDY] += dy * dy;
      acc[GY_INTER] += dy * dg[q];
      const double viol = res[q] - rp[q];
      acc[GY_RP2] += viol * viol;
      acc[GY_YH] += p * hv[q];
    }
  }
  if (err) set_err(A.err, err);
  block_store_mask<GY_N>(acc, 0u, part, cap, slot0 + blockIdx.x);
}

// ---- 16-byte (double2) streaming variants of the step epilogues -------------
// The same per-element arithmetic as k_step_x / y_epilogue / t_epilogue, with
// every stream moved as aligned pairs (one 16-byte load or store per two
// elements): twice the bytes in flight per instruction for the HBM-bound
// streams.  Used when every row is elementwise (no cone blocks in the space);
// odd lengths finish with one scalar element.
__device__ __forceinline__ double2 ld2(const double* p, int i) {
  return __ldg(reinterpret_cast<const double2*>(p) + i);
}
__device__ __forceinline__ double2 ldc2(const double* p, int i) {
  return reinterpret_cast<const double2*>(p)[i];
}
__device__ __forceinline__ void st2(double* p, int i, double a, double b) {
  reinterpret_cast<double2*>(p)[i] = make_double2(a, b);
}

// y-space row r (elementwise block) with dot = (G^ x~)_r and the loaded operands
__device__ __forceinline__ void y_elem(const KArgs& A, const YCoef& k, int r, double dot, double y,
                                       double yh, double ya, double yb, double gx, double gxh,
                                       double gxa, double hi, double& o_y, double& o_yb, double& o_gx,
                                       double& o_gxh, double& o_yh, double* acc) {
  double yn, gn;
  if (k.pend) {
    yn = k.a * (k.opb * yh - k.be * y) + k.b * ya;
    gn = k.a * (k.opb * gxh - k.be * gx) + k.b * gxa;
    o_yb = (k.W == 0.0) ? yn : (k.W * yb + k.et * yn) / k.tot;
  } else {
    yn = y;
    gn = gx;
    o_yb = yb;
  }
  o_y = yn;
  o_gx = gn;
  const double v = yn + k.sigma * (hi - dot);
  const double gh = 0.5 * (dot + gn);
  o_gxh = gh;
  const bool zero = r < A.m_zero;
  const double p = zero ? v : pos_part(v);
  o_yh = p;
  const double dy = p - yn;
  acc[GY_YY] += yn * yn;
  acc[GY_DYDY] += dy * dy;
  acc[GY_INTER] += dy * (dot - gn);
  const double res = gh - hi;
  const double viol = zero ? res : res - pos_part(res);
  acc[GY_RP2] += viol * viol;
  acc[GY_YH] += p * hi;
}

__global__ void __launch_bounds__(BS, 4) k_y_epi2(KArgs A, double* part, int cap, CtrlFuse F) {
  pdl_enter();
  const PdcsCtrl* C = A.ctrl;
  if (C->stop) return;
  __shared__ YCoef ks;
  if (threadIdx.x == 0) ks = y_coef(C);
  __syncthreads();
  const YCoef& k = ks;
  double acc[GY_N] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const int np = A.m >> 1;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int q = tid; q < np; q += nt) {
    const double2 w = ldc2(A.w, q), y = ldc2(A.y, q), yh = ldc2(A.yh, q), ya = ld2(A.ya, q),
                  yb = ldc2(A.yb, q), gx = ldc2(A.gx, q), gxh = ldc2(A.gxh, q), gxa = ld2(A.gxa, q),
                  h = ld2(A.h, q);
    double oy0, oyb0, ogx0, ogxh0, oyh0, oy1, oyb1, ogx1, ogxh1, oyh1;
    y_elem(A, k, 2 * q, w.x, y.x, yh.x, ya.x, yb.x, gx.x, gxh.x, gxa.x, h.x, oy0, oyb0, ogx0, ogxh0, oyh0, acc);
    y_elem(A, k, 2 * q + 1, w.y, y.y, yh.y, ya.y, yb.y, gx.y, gxh.y, gxa.y, h.y, oy1, oyb1, ogx1, ogxh1, oyh1,
           acc);
    if (k.pend) {
      st2(A.y, q, oy0, oy1);
      st2(A.yb, q, oyb0, oyb1);
      st2(A.gx, q, ogx0, ogx1);
    }
    st2(A.gxh, q, ogxh0, ogxh1);
    st2(A.yh, q, oyh0, oyh1);
  }
  if ((A.m & 1) && tid == 0) {
    const int r = A.m - 1;
    double oy, oyb, ogx, ogxh, oyh;
    y_elem(A, k, r, A.w[r], A.y[r], A.yh[r], A.ya[r], A.yb[r], A.gx[r], A.gxh[r], A.gxa[r], A.h[r], oy, oyb,
           ogx, ogxh, oyh, acc);
    if (k.pend) {
      A.y[r] = oy;
      A.yb[r] = oyb;
      A.gx[r] = ogx;
    }
    A.gxh[r] = ogxh;
    A.yh[r] = oyh;
  }
  block_store_mask<GY_N>(acc, 0u, part, cap, blockIdx.x);
  fused_ctrl(F);
}

// x-space coordinate j of k_step_x (box-only, uniform box) with loaded operands
__device__ __forceinline__ void x_elem(const KArgs& A, bool pend, bool inject, const double* kc, double x,
                                       double xh, double xa, double xb, double gty, double gth,
                                       double gtya, double cj, double dj, double& o_x, double& o_xb,
                                       double& o_gty, double& o_xh, double& o_xt, double* acc) {
  const double &a = kc[0], &b = kc[1], &be = kc[2], &et = kc[3], &W = kc[4], &tau = kc[5];
  const double &opb = kc[6], &tot = kc[7];
  double xn, gn;
  if (pend) {
    xn = a * (opb * xh - be * x) + b * xa;
    gn = a * (opb * gth - be * gty) + b * gtya;
    o_xb = (W == 0.0) ? xn : (W * xb + et * xn) / tot;
  } else {
    xn = x;
    gn = gty;
    o_xb = xb;
  }
  o_x = xn;
  o_gty = gn;
  const double v = xn - tau * (cj - gn);
  double lj, uj;
  if (A.ub == 2) {
    lj = A.lu;
    uj = A.uu;
  } else {
    lj = A.lu / dj;
    uj = A.uu / dj;
  }
  double p = clampv(v, lj, uj);
  if (inject) p = __longlong_as_double(0x7ff8000000000000ll);  // debug NaN hook (coordinate 0)
  o_xh = p;
  o_xt = 2.0 * p - xn;
  const double d = p - xn;
  acc[GX_XX] += xn * xn;
  acc[GX_DXDX] += d * d;
  acc[GX_CX] += cj * p;
}

// k_step_x over a uniform box covering all of x-space (single GPU, no NaN
// injection), pairs of coordinates per 16-byte access
__global__ void __launch_bounds__(BS, 4) k_step_x2(KArgs A, double* part, int cap) {
  pdl_enter();
  const PdcsCtrl* C = A.ctrl;
  if (C->stop) return;
  __shared__ double kc[8];
  if (threadIdx.x == 0) {
    kc[0] = C->pa; kc[1] = C->pb; kc[2] = C->pbeta; kc[3] = C->peta; kc[4] = C->pW; kc[5] = C->tau;
    kc[6] = 1.0 + C->pbeta; kc[7] = C->pW + C->peta;
  }
  __syncthreads();
  const bool pend = C->pending != 0;
  const bool inject = C->nan_after >= 0 && C->n_primal_proj >= C->nan_after;
  double acc[GX_N] = {0.0, 0.0, 0.0};
  const int np = A.n >> 1;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int q = tid; q < np; q += nt) {
    const double2 x = ldc2(A.x, q), gty = ldc2(A.gty, q), c = ld2(A.c, q);
    const double2 d = A.ub == 1 ? ld2(A.d2, q) : make_double2(1.0, 1.0);
    double2 xh, xa, xb, gth, gtya;
    if (pend) {
      xh = ldc2(A.xh, q); xa = ld2(A.xa, q); xb = ldc2(A.xb, q); gth = ldc2(A.gth, q); gtya = ld2(A.gtya, q);
    } else {
      xh = xa = xb = gth = gtya = make_double2(0.0, 0.0);
    }
    double ox0, oxb0, og0, oxh0, oxt0, ox1, oxb1, og1, oxh1, oxt1;
    x_elem(A, pend, inject && q == 0, kc, x.x, xh.x, xa.x, xb.x, gty.x, gth.x, gtya.x, c.x, d.x, ox0, oxb0, og0,
           oxh0, oxt0, acc);
    x_elem(A, pend, false, kc, x.y, xh.y, xa.y, xb.y, gty.y, gth.y, gtya.y, c.y, d.y, ox1, oxb1, og1, oxh1, oxt1,
           acc);
    if (pend) {
      st2(A.xb, q, oxb0, oxb1);
      st2(A.x, q, ox0, ox1);
      st2(A.gty, q, og0, og1);
    }
    st2(A.xh, q, oxh0, oxh1);
    st2(A.xt, q, oxt0, oxt1);
  }
  if ((A.n & 1) && tid == 0) {
    const int j = A.n - 1;
    double ox, oxb, og, oxh, oxt;
    x_elem(A, pend, inject && j == 0, kc, A.x[j], A.xh[j], A.xa[j], A.xb[j], A.gty[j], A.gth[j], A.gtya[j],
           A.c[j], A.ub == 1 ? A.d2[j] : 1.0, ox, oxb, og, oxh, oxt, acc);
    if (pend) {
      A.xb[j] = oxb;
      A.x[j] = ox;
      A.gty[j] = og;
    }
    A.xh[j] = oxh;
    A.xt[j] = oxt;
  }
  block_store_mask<GX_N>(acc, 0u, part, cap, blockIdx.x);
}

// x-space box coordinate j with dot = (G^T y_hat)_j (t_epilogue without the store)
__device__ __forceinline__ void t_elem(const KArgs& A, double dot, double cj, double dj, double* acc) {
  double lj, uj;
  if (A.ub == 2) {
    lj = A.lu;
    uj = A.uu;
  } else {
    lj = A.lu / dj;
    uj = A.uu / dj;
  }
  const double lam = cj - dot;
  const bool lf = isfinite(lj), uf = isfinite(uj);
  const double pr = (!lf && !uf) ? 0.0 : (!lf ? neg_clip(lam) : (!uf ? pos_part(lam) : lam));
  const double v = lam - pr;
  acc[GT_RD2] += v * v;
  if (lf) acc[GT_LSUM] += lj * pos_part(lam);
  if (uf) acc[GT_USUM] += uj * pos_part(-lam);
}

// needs a uniform box over all of x-space (ub != 0, nbox == n)
__global__ void __launch_bounds__(BS, 5) k_t_epi2(KArgs A, double* part, int cap, CtrlFuse F, ShortRows R) {
  pdl_enter();
  const PdcsCtrl* C = A.ctrl;
  if (C->stop || !C->accepted) return;
  double acc[GT_N] = {0.0, 0.0, 0.0};
  const int np = A.nbox >> 1;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int q = tid; q < np; q += nt) {
    const double2 g = ldc2(A.gth, q), c = ld2(A.c, q);
    const double2 d = A.ub == 1 ? ld2(A.d2, q) : make_double2(1.0, 1.0);
    t_elem(A, cls_dot(R, 2 * q, g.x, A.gth), c.x, d.x, acc);
    t_elem(A, cls_dot(R, 2 * q + 1, g.y, A.gth), c.y, d.y, acc);
  }
  if ((A.nbox & 1) && tid == 0) {
    const int j = A.nbox - 1;
    t_elem(A, cls_dot(R, j, A.gth[j], A.gth), A.c[j], A.ub == 1 ? A.d2[j] : 1.0, acc);
  }
  cls_cone_cols(A, R);
  block_store_mask<GT_N>(acc, 0u, part, cap, blockIdx.x);
  fused_ctrl(F);
}

// Row-class pass of a mixed-length matrix (C2: rows of 1-2 and of ~48
// entries): the rows of the long class, listed in `rows`, VW lanes per row,
// product into out[row].  The epilogue then streams over all rows and sums
// the short ones itself (cls_dot).
template <int VW>
__global__ void __launch_bounds__(BS) k_rows_pass(const int* __restrict__ rows, int nr, const int* __restrict__ rp,
                                                  const int* __restrict__ ci, const double* __restrict__ va,
                                                  const double* __restrict__ x, double* out, const PdcsCtrl* ctrl,
                                                  int gate) {
  pdl_enter();
  if (gated(ctrl, gate)) return;
  const int lane = threadIdx.x & 31, sub = lane & (VW - 1);
  constexpr int RPW = 32 / VW, U = 4;
  const int wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int wt = gridDim.x * (blockDim.x >> 5);
  // the next row's extent is loaded while this row's entries are summed: the
  // rows -> rp -> (ci, va) -> x chain is latency bound, not bandwidth bound
  int i = wg * RPW + lane / VW;
  int r = 0, b = 0, e = 0;
  if (i < nr) {
    r = __ldg(rows + i);
    b = __ldg(rp + r);
    e = __ldg(rp + r + 1);
  }
  for (int base = wg * RPW; base < nr; base += wt * RPW) {
    const int in = i + wt * RPW;
    int rn = 0, bn = 0, en = 0;
    if (in < nr) {
      rn = __ldg(rows + in);
      bn = __ldg(rp + rn);
      en = __ldg(rp + rn + 1);
    }
    double s = 0.0;
    // U entries per lane in flight: their column and value loads, then the gathers
    for (int j = b + sub; j < e; j += U * VW) {
      int c[U];
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int jj = j + u * VW;
        c[u] = jj < e ? __ldg(ci + jj) : -1;
        v[u] = jj < e ? __ldg(va + jj) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c[u] >= 0) s += v[u] * __ldg(x + c[u]);
    }
    if (VW > 1) {
#pragma unroll
      for (int off = VW / 2; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off, VW);
    }
    if (sub == 0 && i < nr) out[r] = s;
    i = in;
    r = rn;
    b = bn;
    e = en;
  }
}

// Split step (PDCS_TUNE split=1, matrices without chunked long rows): every
// panel is a gather-only pass, the last one writing the whole product
// (G^ x~ into w, G^T y_hat into gth), and the epilogue is a pure stream over
// the y- (x-) space -- the gathered panel no longer competes in L2 with the
// 13 epilogue streams (C5 lab: 0.486 vs 0.517 ms per y-step with hs=1).
template <bool H>
__global__ void __launch_bounds__(BS, 8) k_y_epi(KArgs A, double* part, int cap, CtrlFuse F, ShortRows R) {
  pdl_enter();
  const PdcsCtrl* C = A.ctrl;
  if (C->stop) return;
  __shared__ YCoef ks;
  if (threadIdx.x == 0) ks = y_coef(C);
  __syncthreads();
  const YCoef& k = ks;
  const uint64_t ps = policy_stream(), pky = policy_keep_frac(A.keep_yh);
  double acc[GY_N] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < A.m; r += gridDim.x * blockDim.x)
    y_epilogue<H>(A, k, r, cls_dot(R, r, ld_hint<H>(A.w + r, ps), A.w), acc, ps, pky);
  block_store_mask<GY_N>(acc, 0u, part, cap, blockIdx.x);
  fused_ctrl(F);
}

// Class-split y-step epilogue fused with the dual cone blocks of <= 16 rows
// (C2's SOC(11)): CTAs [0, ga) stream the elementwise rows; the others give
// each block to a 16-lane group, which finishes the epilogue of the block's
// rows (v into yh, the product into w, gx_hat) and projects the block right
// away (do_block) -- the block kernel's launch and its second pass over the
// block rows go away, and a block's rows are written and read by one group.
template <int MINB>
__global__ void __launch_bounds__(BS, MINB) k_y_epi_blk(KArgs A, double* part, int cap, ShortRows R,
                                                        const PdcsBlock* tab, int nb, int ga) {
  pdl_enter();
  const PdcsCtrl* C = A.ctrl;
  if (C->stop) return;
  __shared__ YCoef ks;
  if (threadIdx.x == 0) ks = y_coef(C);
  __syncthreads();
  const YCoef& k = ks;
  double acc[GY_N] = {0.0, 0.0, 0.0, 0.0, 0.0};
  if ((int)blockIdx.x < ga) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < A.m_elem; r += ga * blockDim.x)
      y_epilogue<false>(A, k, r, cls_dot(R, r, A.w[r], A.w), acc, 0, 0);
  } else {
    SubGrp<16> g;
    const BlkParams P{};
    const int gi = (((int)blockIdx.x - ga) * blockDim.x + threadIdx.x) >> 4;
    const int gn = (((int)gridDim.x - ga) * blockDim.x) >> 4;
    for (int i = gi; i < nb; i += gn) {
      const PdcsBlock b = tab[i];
      for (int q = g.rank; q < b.dim; q += g.size) {
        const int r = b.start + q;
        y_epilogue<false>(A, k, r, cls_dot(R, r, A.w[r], A.w), acc, 0, 0);
      }
      g.sync();
      do_block<SubGrp<16>, OP_STEP_Y>(g, b, A, P, acc);
    }
    __syncwarp();
  }
  block_store_mask<GY_N>(acc, 0u, part, cap, blockIdx.x);
}

template <bool H>
__global__ void __launch_bounds__(BS, 8) k_t_epi(KArgs A, double* part, int cap, CtrlFuse F, ShortRows R) {
  pdl_enter();
  const PdcsCtrl* C = A.ctrl;
  if (C->stop || !C->accepted) return;
  const uint64_t ps = policy_stream();
  double acc[GT_N] = {0.0, 0.0, 0.0};
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < A.nbox; j += gridDim.x * blockDim.x)
    t_epilogue<H, false>(A, j, cls_dot(R, j, ld_hint<H>(A.gth + j, ps), A.gth), acc, ps);
  cls_cone_cols(A, R);
  block_store_mask<GT_N>(acc, 0u, part, cap, blockIdx.x);
  fused_ctrl(F);
}

template <int VW, int GP>
__global__ void __launch_bounds__(BS, 6) k_step_y_lane(KArgs A, int nrows, TileSrc S, double* part,
                                                       int cap, CtrlFuse F) {
  pdl_enter();
  const PdcsCtrl* C = A.ctrl;
  if (C->stop) return;
  // the Halpern / step coefficients live in shared memory, not in 16
  // registers per thread: 40 registers, 6 CTAs per SM
  __shared__ YCoef ks;
  if (threadIdx.x == 0) ks = y_coef(C);
  __syncthreads();
  const YCoef& k = ks;
  const uint64_t ps = policy_stream(), pkx = policy_keep_frac(A.keep_xt),
                 pky = policy_keep_frac(A.keep_yh);
  double acc[GY_N] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const int lane = threadIdx.x & 31, sub = lane & (VW - 1);
  constexpr int RPW = 32 / VW;
  const int wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int wt = gridDim.x * (blockDim.x >> 5);
  for (int base = wg * RPW; base < nrows; base += wt * RPW) {
    const int r = base + lane / VW;
    const double dot = lane_row<VW, GP>(S, A.xt, A.w, r, sub, nrows, ps, pkx);
    if (sub == 0 && r < nrows) y_epilogue<false>(A, k, r, dot, acc, ps, pky);
  }
  block_store_mask<GY_N>(acc, 0u, part, cap, blockIdx.x);
  fused_ctrl(F);
}

template <int VW, int GP>
__global__ void __launch_bounds__(BS, 8) k_step_t_lane(KArgs A, int nrows, TileSrc S, double* part,
                                                       int cap, CtrlFuse F) {
  pdl_enter();
  const PdcsCtrl* C = A.ctrl;
  if (C->stop || !C->accepted) return;
  const uint64_t ps = policy_stream(), pky = policy_keep_frac(A.keep_yh);
  double acc[GT_N] = {0.0, 0.0, 0.0};
  const int lane = threadIdx.x & 31, sub = lane & (VW - 1);
  constexpr int RPW = 32 / VW;
  const int wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int wt = gridDim.x * (blockDim.x >> 5);
  for (int base = wg * RPW; base < nrows; base += wt * RPW) {
    const int j = base + lane / VW;
    const double dot = lane_row<VW, GP>(S, A.yh, A.gtr, j, sub, nrows, ps, pky);
    if (sub == 0 && j < nrows) t_epilogue<false>(A, j, dot, acc, ps);
  }
  block_store_mask<GT_N>(acc, 0u, part, cap, blockIdx.x);
  fused_ctrl(F);
}

// Sums of NQ partial rows p[q * cap + 0 .. n) by one CTA: all rows' loads are
// in flight together and the tree reductions share one pair of barriers.
// Thread 0 receives the sums (the controllers below run on thread 0).
template <int NQ, int U = 1>
__device__ __forceinline__ void cta_sum_rows(const double* p, int cap, int n, double (&out)[NQ]) {
  __shared__ double sh[NQ][32];
  // U independent accumulator sets keep U NQ L2 loads in flight per thread
  // (the standalone controllers: U = 4; folded into a step kernel: U = 1, so
  // the step kernel's register budget is not spent on the controller)
  double tu[U][NQ];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int q = 0; q < NQ; ++q) tu[u][q] = 0.0;
  const int bd = blockDim.x;
  int s0 = threadIdx.x;
  for (; s0 + (U - 1) * bd < n; s0 += U * bd) {
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < NQ; ++q) tu[u][q] += __ldcg(p + (size_t)q * cap + s0 + u * bd);  // L2: other CTAs wrote them
  }
  for (; s0 < n; s0 += bd) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) tu[0][q] += __ldcg(p + (size_t)q * cap + s0);
  }
  double t[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    t[q] = tu[0][q];
#pragma unroll
    for (int u = 1; u < U; ++u) t[q] += tu[u][q];
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    for (int off = 16; off > 0; off >>= 1) t[q] += __shfl_down_sync(0xffffffffu, t[q], off);
    if (lane == 0) sh[q][wid] = t[q];
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      double v = lane < nw ? sh[q][lane] : 0.0;
      for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
      out[q] = v;
    }
  }
}

// Line-search controller (engine.py:183-243), run by one whole CTA.
// yred (sharded mode): the y-space sums already all-reduced across ranks.
// The line-search sums of both spaces in one pass: the x- and y-space partial
// rows are loaded together and share one pair of barriers (the controller
// kernel is latency bound: two sequential reductions cost a round trip each).
template <int NA, int NB>
__device__ __forceinline__ void cta_sum_rows2(const double* pa, int capa, int na, const double* pb, int capb,
                                              int nb, double (&oa)[NA], double (&ob)[NB]) {
  __shared__ double sh[NA + NB][32];
  double t[NA + NB];
#pragma unroll
  for (int q = 0; q < NA + NB; ++q) t[q] = 0.0;
  const int bd = blockDim.x, n = na > nb ? na : nb;
  for (int s0 = threadIdx.x; s0 < n; s0 += bd) {
    if (s0 < na) {
#pragma unroll
      for (int q = 0; q < NA; ++q) t[q] += __ldcg(pa + (size_t)q * capa + s0);
    }
    if (s0 < nb) {
#pragma unroll
      for (int q = 0; q < NB; ++q) t[NA + q] += __ldcg(pb + (size_t)q * capb + s0);
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int q = 0; q < NA + NB; ++q) {
    for (int off = 16; off > 0; off >>= 1) t[q] += __shfl_down_sync(0xffffffffu, t[q], off);
    if (lane == 0) sh[q][wid] = t[q];
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int q = 0; q < NA + NB; ++q) {
      double v = lane < nw ? sh[q][lane] : 0.0;
      for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
      if (q < NA) oa[q < NA ? q : 0] = v;
      else ob[q >= NA ? q - NA : 0] = v;
    }
  }
}

template <int U>
__device__ void ctrl_ls_body(PdcsCtrl* C, const double* partX, int capX, const double* partY,
                             int capY, double* red, const double* yred) {
  double sx[GX_N], sy[GY_N];
  if (yred) {  // sharded: y sums then x sums, already all-reduced over the ranks
#pragma unroll
    for (int q = 0; q < GY_N; ++q) sy[q] = yred[q];
#pragma unroll
    for (int q = 0; q < GX_N; ++q) sx[q] = yred[GY_N + q];
  } else {
    cta_sum_rows2<GX_N, GY_N>(partX, capX, capX, partY, capY, capY, sx, sy);
  }
  if (threadIdx.x != 0) return;
  const double xx = sx[GX_XX], dxdx = sx[GX_DXDX], cx = sx[GX_CX];
  const double yy = sy[GY_YY], dydy = sy[GY_DYDY], inter = sy[GY_INTER], rp2 = sy[GY_RP2],
               yh = sy[GY_YH];
  if (C->new_iter) {
    C->k_bar += 1;
    C->new_iter = 0;
    C->trials = 0;
  }
  C->n_primal_proj += 1;
  C->n_trials_total += 1;
  C->pending = 0;
  red[0] = cx; red[1] = rp2; red[2] = yh;
  const double omega = C->omega, eta = C->eta_try;
  double nxt = eta;
  bool accept = true;
  if (C->adaptive) {
    const double noise = 1e-14 * (1.0 + sqrt(omega * xx + yy / omega));
    const double mov = omega * dxdx + dydy / omega;
    const double itr = fabs(inter) / 2.0;
    C->movement = mov;
    C->interaction = itr;
    if (isnan(mov) || isnan(itr)) {
      C->error = PDCS_ERR_NAN_LINESEARCH;
      C->k_bar -= C->trials;
      C->stop = 1;
      C->reason = PDCS_STOP_ERROR;
      return;
    }
    const double bar = (itr == 0.0 || sqrt(mov) <= noise) ? INFINITY : mov / (2.0 * itr);
    C->eta_bar = bar;
    const double kb1 = (double)C->k_bar + 1.0;
    const double shrink = 1.0 - pow(kb1, -0.3);
    const double grow = 1.0 + pow(kb1, -0.6);
    const double cand = isinf(bar) ? (shrink > 0.0 ? INFINITY : 0.0) : shrink * bar;
    nxt = dmin(dmax(1e-12, dmin(cand, grow * eta)), 1e14);
    accept = eta < bar;
  }
  if (accept) {
    C->accepted = 1;
    C->eta = eta;
    C->eta_hat = nxt;
  } else {
    C->accepted = 0;
    C->eta_try = nxt;
    C->k_bar += 1;
    C->trials += 1;
    C->tau = nxt / omega;
    C->sigma = nxt * omega;
    if (C->trials >= 60) {
      C->error = PDCS_ERR_TRIAL_CAP;
      C->k_bar -= C->trials;
      C->stop = 1;
      C->reason = PDCS_STOP_ERROR;
    }
  }
}

// The standalone controllers work on a shared-memory copy of the control
// block (one parallel load and store instead of thread 0's chain of
// dependent global read-modify-writes).
__device__ __forceinline__ void ctrl_to_smem(PdcsCtrl* sc, const PdcsCtrl* C) {
  constexpr int NW = sizeof(PdcsCtrl) / sizeof(long long);
  for (int i = threadIdx.x; i < NW; i += blockDim.x)
    reinterpret_cast<long long*>(sc)[i] = reinterpret_cast<const long long*>(C)[i];
  __syncthreads();
}
__device__ __forceinline__ void ctrl_from_smem(PdcsCtrl* C, const PdcsCtrl* sc) {
  constexpr int NW = sizeof(PdcsCtrl) / sizeof(long long);
  __syncthreads();
  for (int i = threadIdx.x; i < NW; i += blockDim.x)
    reinterpret_cast<long long*>(C)[i] = reinterpret_cast<const long long*>(sc)[i];
}

__global__ void k_ctrl_ls(PdcsCtrl* C, const double* partX, int capX, const double* partY,
                          int capY, double* red, const double* yred) {
  __shared__ PdcsCtrl sc;
  ctrl_to_smem(&sc, C);
  if (sc.stop) return;
  ctrl_ls_body<4>(&sc, partX, capX, partY, capY, red, yred);
  ctrl_from_smem(C, &sc);
}

// Reflection parameter, Halpern coefficients, averaging weight and the stop
// tests of an accepted iteration (engine.py:590-628, termination.py:150-160),
// run by one whole CTA.
template <int U>
__device__ void ctrl_beta_body(PdcsCtrl* C, const double* partT, int capT, const double* red,
                               const int* err, const double* tred) {
  double st[GT_N];
  if (tred) {  // sharded: all-reduced over the ranks
#pragma unroll
    for (int q = 0; q < GT_N; ++q) st[q] = tred[q];
  } else {
    cta_sum_rows<GT_N, U>(partT, capT, capT, st);
  }
  if (threadIdx.x != 0) return;
  const double rd2 = st[GT_RD2], ls = st[GT_LSUM], us = st[GT_USUM];
  int e = *err;
  if (tred && e == 0 && tred[GT_N] > 0.0)  // another rank's projection failed
    e = (int)dmin(tred[GT_N], (double)PDCS_ERR_BETA);
  if (e) {  // numerical failure inside a projection (exp non-finite, rsoc bracket)
    C->error = e;
    C->stop = 1;
    C->reason = PDCS_STOP_ERROR;
    C->accepted = 0;
    return;
  }
  double beta;
  const double cx = red[0], rp2 = red[1], yh = red[2];
  const double po = cx, dob = yh + ls - us;
  C->p_obj = po;
  C->d_obj = dob;
  if (C->use_fixed_beta) {
    beta = C->fixed_beta;
  } else {
    const double abs_p = sqrt(rp2), abs_d = sqrt(rd2), gap = fabs(po - dob);
    const double e1 = abs_p / (1.0 + C->h1), e2 = abs_d / (1.0 + C->c1);
    const double e3 = gap / (1.0 + fabs(po) + fabs(dob));
    const double err_max = dmax(dmax(e1, e2), e3);
    C->max_err = err_max;
    if (isnan(e1) || isnan(e2) || isnan(e3)) {
      C->error = PDCS_ERR_BETA;
      C->stop = 1;
      C->reason = PDCS_STOP_ERROR;
      C->accepted = 0;
      return;
    }
    beta = err_max <= 0.0 ? 1.0 : dmin(dmax(-0.1 * log10(err_max) + 0.2, 0.0), 1.0);
  }
  C->beta = beta;
  const double k = (double)C->k;
  C->pa = (k + 1.0) / (k + 2.0);
  C->pb = 1.0 / (k + 2.0);
  C->pbeta = beta;
  C->peta = C->eta;
  C->pW = C->W;
  C->W = (C->W == 0.0) ? C->eta : C->W + C->eta;
  C->pending = 1;
  C->accepted = 0;
  C->k += 1;
  C->n_accepted_total += 1;
  C->new_iter = 1;
  C->eta_try = C->eta_hat;
  C->tau = C->eta_hat / C->omega;
  C->sigma = C->eta_hat * C->omega;
  const int64_t kb = C->k_bar;
  if (kb >= C->max_iter) { C->stop = 1; C->reason = PDCS_STOP_MAXITER; }
  else if (kb % C->check_freq == 0) { C->stop = 1; C->reason = PDCS_STOP_CHECK; }
  else if (kb >= C->k_bar_stop) { C->stop = 1; C->reason = PDCS_STOP_BATCH; }
  else if (C->print_freq > 0 && kb % C->print_freq == 0) { C->stop = 1; C->reason = PDCS_STOP_PRINT; }
}

// sharded mode: the rank's projection error code as a double for the all-reduce
__global__ void k_err_to_double(const int* err, double* out) { *out = (double)*err; }

__global__ void k_ctrl_beta(PdcsCtrl* C, const double* partT, int capT, const double* red,
                            const int* err, const double* tred) {
  __shared__ PdcsCtrl sc;
  ctrl_to_smem(&sc, C);
  if (sc.stop || !sc.accepted) return;
  ctrl_beta_body<4>(&sc, partT, capT, red, err, tred);
  ctrl_from_smem(C, &sc);
}

// Controller folded into the last CTA of the kernel that writes the final
// reduction partials (saves a launch per controller when no cone-block kernel
// follows).  The ticket counts finished CTAs; the last one, after a fence,
// sees every partial.
__device__ __forceinline__ bool last_cta(unsigned* ticket) {
  __shared__ int is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}

__device__ __forceinline__ void fused_ctrl(const CtrlFuse& F) {
  if (!F.mode || !last_cta(F.ticket)) return;
  if (F.mode == 1) ctrl_ls_body<1>(F.C, F.partA, F.capA, F.partB, F.capB, F.red, nullptr);
  else ctrl_beta_body<1>(F.C, F.partB, F.capB, F.red, F.err, nullptr);
  if (threadIdx.x == 0) *F.ticket = 0u;
}

// Apply the pending Halpern/average update outside the loop (check path).
__global__ void k_flush_x(KArgs A) {
  const PdcsCtrl* C = A.ctrl;
  if (!C->pending) return;
  const double a = C->pa, b = C->pb, be = C->pbeta, et = C->peta, W = C->pW;
  const double opb = 1.0 + be, tot = W + et;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < A.n; j += gridDim.x * blockDim.x) {
    const double xo = A.x[j];
    const double xn = a * (opb * A.xh[j] - be * xo) + b * A.xa[j];
    const double go = A.gty[j];
    A.gty[j] = a * (opb * A.gth[j] - be * go) + b * A.gtya[j];
    A.xb[j] = (W == 0.0) ? xn : (W * A.xb[j] + et * xn) / tot;
    A.x[j] = xn;
  }
}
__global__ void k_flush_y(KArgs A) {
  const PdcsCtrl* C = A.ctrl;
  if (!C->pending) return;
  const double a = C->pa, b = C->pb, be = C->pbeta, et = C->peta, W = C->pW;
  const double opb = 1.0 + be, tot = W + et;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < A.m; r += gridDim.x * blockDim.x) {
    const double yo = A.y[r];
    const double yn = a * (opb * A.yh[r] - be * yo) + b * A.ya[r];
    const double go = A.gx[r];
    A.gx[r] = a * (opb * A.gxh[r] - be * go) + b * A.gxa[r];
    A.yb[r] = (W == 0.0) ? yn : (W * A.yb[r] + et * yn) / tot;
    A.y[r] = yn;
  }
}
__global__ void k_clear_pending(PdcsCtrl* C) { C->pending = 0; }

// Batched engines: copy every member's control block into one array (one
// device-to-host copy per batch-graph replay instead of one per engine).
__global__ void k_gather_ctrl(PdcsCtrl* const* src, PdcsCtrl* dst, int n) {
  constexpr int W = sizeof(PdcsCtrl) / sizeof(int64_t);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n * W; i += gridDim.x * blockDim.x) {
    const int e = i / W, w = i % W;
    reinterpret_cast<int64_t*>(dst + e)[w] = reinterpret_cast<const int64_t*>(src[e])[w];
  }
}

// ---------------------------------------------------------------------------
// Check path
// ---------------------------------------------------------------------------
// Fill the block regions with the vectors whose cone projections the metric
// passes need.  mode 0 = scaled, 1 = original.
__global__ void k_met_fill(KArgs A, int mode, const double* gx, const double* gty) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int j = A.nbox + tid; j < A.n; j += nt) {
    double g = gty[j], c = A.c[j];
    if (mode == 1) { g = g / A.d2[j]; c = A.c0[j]; }
    A.tx1[j] = c - g;
  }
  for (int i = A.m_elem + tid; i < A.m; i += nt) {
    double g = gx[i], h = A.h[i];
    if (mode == 1) { g = g / A.d1[i]; h = A.h0[i]; }
    A.ty1[i] = g - h;
  }
}

// compute_errors reductions (termination.py:91-147), split in a y pass and
// an x pass writing disjoint slot ranges.
__global__ void k_met_y(KArgs A, int mode, const double* y, const double* gx, double* part, int cap,
                        int slot0) {
  double acc[PDCS_NMET];
#pragma unroll
  for (int q = 0; q < PDCS_NMET; ++q) acc[q] = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.m; i += gridDim.x * blockDim.x) {
    double yi = y[i], gi = gx[i], hi;
    acc[PDCS_MET_NONFINITE] += isfinite(yi) ? 0.0 : 1.0;
    if (mode == 1) {
      const double d = A.d1[i];
      yi = yi * d;
      gi = gi / d;
      hi = A.h0[i];
    } else {
      hi = A.h[i];
    }
    const double r = gi - hi;
    const double rp = i < A.m_zero ? 0.0 : (i < A.m_elem ? pos_part(r) : A.ty1[i]);
    const double v = r - rp;
    acc[PDCS_MET_RV2] += v * v;
    acc[PDCS_MET_RVMAX] = nanmax(acc[PDCS_MET_RVMAX], fabs(v));
    acc[PDCS_MET_HMAX] = nanmax(acc[PDCS_MET_HMAX], fabs(hi));
    acc[PDCS_MET_GXMAX] = nanmax(acc[PDCS_MET_GXMAX], fabs(gi));
    acc[PDCS_MET_RPMAX] = nanmax(acc[PDCS_MET_RPMAX], fabs(rp));
    acc[PDCS_MET_YH] += yi * hi;
    acc[PDCS_MET_H1] += fabs(hi);
    acc[PDCS_MET_YY] += yi * yi;
  }
  block_store_mask<PDCS_NMET>(acc, MET_MAXMASK, part, cap, slot0 + blockIdx.x);
}

__global__ void k_met_x(KArgs A, int mode, const double* x, const double* gty, double* part, int cap,
                        int slot0) {
  double acc[PDCS_NMET];
#pragma unroll
  for (int q = 0; q < PDCS_NMET; ++q) acc[q] = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < A.n; j += gridDim.x * blockDim.x) {
    double xi = x[j], gi = gty[j], cj;
    acc[PDCS_MET_NONFINITE] += isfinite(xi) ? 0.0 : 1.0;
    if (mode == 1) {
      const double d = A.d2[j];
      xi = xi * d;
      gi = gi / d;
      cj = A.c0[j];
    } else {
      cj = A.c[j];
    }
    const double lam = cj - gi;
    if (j < A.nbox) {
      const double lj = mode == 1 ? A.l0[j] : A.l[j];
      const double uj = mode == 1 ? A.u0[j] : A.u[j];
      const bool lf = isfinite(lj), uf = isfinite(uj);
      const double pr = (!lf && !uf) ? 0.0 : (!lf ? neg_clip(lam) : (!uf ? pos_part(lam) : lam));
      const double v = lam - pr;
      acc[PDCS_MET_V1SQ] += v * v;
      acc[PDCS_MET_V1MAX] = nanmax(acc[PDCS_MET_V1MAX], fabs(v));
      if (lf) acc[PDCS_MET_LSUM] += lj * pos_part(lam);
      if (uf) acc[PDCS_MET_USUM] += uj * pos_part(-lam);
    } else {
      const double v = lam - A.tx1[j];
      acc[PDCS_MET_V2SQ] += v * v;
      acc[PDCS_MET_V2MAX] = nanmax(acc[PDCS_MET_V2MAX], fabs(v));
    }
    acc[PDCS_MET_CMAX] = nanmax(acc[PDCS_MET_CMAX], fabs(cj));
    acc[PDCS_MET_GTYMAX] = nanmax(acc[PDCS_MET_GTYMAX], fabs(gi));
    acc[PDCS_MET_CX] += cj * xi;
    acc[PDCS_MET_C1] += fabs(cj);
    acc[PDCS_MET_XX] += xi * xi;
  }
  block_store_mask<PDCS_NMET>(acc, MET_MAXMASK, part, cap, slot0 + blockIdx.x);
}

// Infeasibility rays on the original instance (termination.py:230-273).
__global__ void k_ray_fill(KArgs A, const double* x, const double* gx, const double* gty,
                           double xn, double yn) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int j = A.nbox + tid; j < A.n; j += nt) {
    const double g = gty[j] / A.d2[j];
    A.tx1[j] = (-g) / yn;
    A.tx2[j] = (x[j] * A.d2[j]) / xn;
  }
  for (int i = A.m_elem + tid; i < A.m; i += nt) A.ty1[i] = (gx[i] / A.d1[i]) / xn;
}

__global__ void k_ray_y(KArgs A, const double* y, const double* gx, double xn, double* part, int cap,
                        int slot0) {
  double acc[PDCS_NRAY];
#pragma unroll
  for (int q = 0; q < PDCS_NRAY; ++q) acc[q] = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.m; i += gridDim.x * blockDim.x) {
    const double d = A.d1[i];
    const double yi = y[i] * d;
    const double gh = (gx[i] / d) / xn;
    const double rp = i < A.m_zero ? 0.0 : (i < A.m_elem ? pos_part(gh) : A.ty1[i]);
    acc[5] = nanmax(acc[5], fabs(gh - rp));
    acc[2] += yi * A.h0[i];
  }
  block_store_mask<PDCS_NRAY>(acc, RAY_MAXMASK, part, cap, slot0 + blockIdx.x);
}

__global__ void k_ray_x(KArgs A, const double* x, const double* gty, double xn, double yn,
                        double* part, int cap, int slot0) {
  double acc[PDCS_NRAY];
#pragma unroll
  for (int q = 0; q < PDCS_NRAY; ++q) acc[q] = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < A.n; j += gridDim.x * blockDim.x) {
    const double d = A.d2[j];
    const double g = gty[j] / d;
    const double lam = (-g) / yn;
    const double xh = (x[j] * d) / xn;
    if (j < A.nbox) {
      const double lj = A.l0[j], uj = A.u0[j];
      const bool lf = isfinite(lj), uf = isfinite(uj);
      const double pr = (!lf && !uf) ? 0.0 : (!lf ? neg_clip(lam) : (!uf ? pos_part(lam) : lam));
      acc[0] = nanmax(acc[0], fabs(lam - pr));
      if (lf) acc[3] += lj * pos_part(lam);
      if (uf) acc[4] += uj * pos_part(-lam);
      const double rec = (lf && uf) ? 0.0 : (lf ? pos_part(xh) : (uf ? neg_clip(xh) : xh));
      acc[6] = nanmax(acc[6], fabs(xh - rec));
    } else {
      acc[1] = nanmax(acc[1], fabs(lam - A.tx1[j]));
      acc[7] = nanmax(acc[7], fabs(xh - A.tx2[j]));
    }
    acc[8] += A.c0[j] * xh;
  }
  block_store_mask<PDCS_NRAY>(acc, RAY_MAXMASK, part, cap, slot0 + blockIdx.x);
}

// Normalized-gap probe z(t) (restart.py:62-77): elementwise parts.
__global__ void k_gap_x(KArgs A, const double* x, const double* gty, double ttau) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < A.n; j += gridDim.x * blockDim.x) {
    const double b1 = gty[j] - A.c[j];
    const double v = x[j] + ttau * b1;
    A.tx0[j] = j < A.nbox ? clampv(v, A.l[j], A.u[j]) : v;
  }
}
__global__ void k_gap_y(KArgs A, const double* y, const double* gx, double tsig) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.m; i += gridDim.x * blockDim.x) {
    const double b2 = A.h[i] - gx[i];
    const double v = y[i] + tsig * b2;
    A.ty0[i] = i < A.m_zero ? v : (i < A.m_elem ? pos_part(v) : v);
  }
}
__global__ void k_gap_red(KArgs A, const double* x, const double* y, const double* gx,
                          const double* gty, double* part, int cap) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int j = tid; j < A.n; j += nt) {
    const double zx = A.tx0[j], xj = x[j];
    const double dx = xj - zx;
    acc[0] += dx * dx;
    acc[2] += (gty[j] - A.c[j]) * (zx - xj);
  }
  for (int i = tid; i < A.m; i += nt) {
    const double zy = A.ty0[i], yi = y[i];
    const double dy = yi - zy;
    acc[1] += dy * dy;
    acc[3] += (A.h[i] - gx[i]) * (zy - yi);
  }
  block_store_mask<4>(acc, 0u, part, cap, blockIdx.x);
}

// Up to GAP_K gap probes in ONE pass over the iterate (problems without cone
// blocks): the reads of x, G^T y, c, l, u, y, G x, h are shared by all t,
// only the projections and sums are per t.  Per probe k the sums of
// k_gap_x/k_gap_y/k_gap_red: part rows [2k] ||x - zx||^2, [2k+1] b1.(zx - x)
// (x pass), [2 GAP_K + 2k] ||y - zy||^2, [2 GAP_K + 2k + 1] b2.(zy - y).
constexpr int GAP_K = 16;
struct GapTs {
  double tt[GAP_K];  // t_k tau
  double ts[GAP_K];  // t_k sigma
  int k;
};

__global__ void __launch_bounds__(BS) k_gap_multi(KArgs A, const double* __restrict__ x,
                                                  const double* __restrict__ y,
                                                  const double* __restrict__ gx,
                                                  const double* __restrict__ gty, GapTs T,
                                                  double* part, int cap) {
  double acc[2 * GAP_K];
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
#pragma unroll
  for (int q = 0; q < 2 * GAP_K; ++q) acc[q] = 0.0;
  for (int j = tid; j < A.n; j += nt) {
    const double b1 = gty[j] - A.c[j], xj = x[j];
    const bool box = j < A.nbox;
    const double lj = box ? A.l[j] : 0.0, uj = box ? A.u[j] : 0.0;
#pragma unroll
    for (int k = 0; k < GAP_K; ++k) {
      if (k < T.k) {
        const double v = xj + T.tt[k] * b1;
        const double z = box ? clampv(v, lj, uj) : v;
        const double d = xj - z;
        acc[2 * k] += d * d;
        acc[2 * k + 1] += b1 * (z - xj);
      }
    }
  }
  block_store_mask<2 * GAP_K>(acc, 0u, part, cap, blockIdx.x);
#pragma unroll
  for (int q = 0; q < 2 * GAP_K; ++q) acc[q] = 0.0;
  for (int i = tid; i < A.m; i += nt) {
    const double b2 = A.h[i] - gx[i], yi = y[i];
    const bool zero = i < A.m_zero, elem = i < A.m_elem;
#pragma unroll
    for (int k = 0; k < GAP_K; ++k) {
      if (k < T.k) {
        const double v = yi + T.ts[k] * b2;
        const double z = zero ? v : (elem ? pos_part(v) : v);
        const double d = yi - z;
        acc[2 * k] += d * d;
        acc[2 * k + 1] += b2 * (z - yi);
      }
    }
  }
  block_store_mask<2 * GAP_K>(acc, 0u, part + (size_t)2 * GAP_K * cap, cap, blockIdx.x);
}

// Reduce partial row q (columns [0, nslots)) into out[q]; one CTA per row.
__global__ void k_finalize_rows(const double* part, int cap, int nslots, double* out) {
  __shared__ double sh[33];
  CtaGrp g(sh);
  const int q = blockIdx.x;
  double t = 0.0;
  for (int s = threadIdx.x; s < nslots; s += blockDim.x) t += part[(size_t)q * cap + s];
  t = g.sum(t);
  if (threadIdx.x == 0) out[q] = t;
}

__global__ void k_dot_diff(const double* a, const double* b, const double* c, const double* d,
                           int n, double* part, int cap) {
  double acc[1] = {0.0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double u = b ? a[i] - b[i] : a[i];
    const double v = d ? c[i] - d[i] : c[i];
    acc[0] += u * v;
  }
  block_store_mask<1>(acc, 0u, part, cap, blockIdx.x);
}

__global__ void k_dist2(const double* a, const double* b, int n, double* part, int cap) {
  double acc[1] = {0.0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double d = b ? a[i] - b[i] : a[i];
    acc[0] += d * d;
  }
  block_store_mask<1>(acc, 0u, part, cap, blockIdx.x);
}

// Elementwise part of the set projections (cones.py:498-549); block parts by
// k_blk_*<OP_PROJECT>.  which: 0 P_X, 1 P_Y, 2 K_d* residual, 3 K_p* (cone
// part, box copied), 4 K_p (cone part, box copied).
__global__ void k_proj_elem(KArgs A, int which, const double* in, double* out) {
  if (which == 0 || which == 3 || which == 4) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < A.n; j += gridDim.x * blockDim.x) {
      const double v = in[j];
      out[j] = (which == 0 && j < A.nbox) ? clampv(v, A.l[j], A.u[j]) : v;
    }
  } else {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.m; i += gridDim.x * blockDim.x) {
      const double v = in[i];
      double o = v;
      if (i < A.m_zero) o = which == 1 ? v : 0.0;
      else if (i < A.m_elem) o = pos_part(v);
      out[i] = o;
    }
  }
}

__global__ void k_step_input(KArgs A, int space, const double* v, const double* g, double step,
                             double* out) {
  const int n = space == 0 ? A.n : A.m;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = space == 0 ? v[i] - step * (A.c[i] - g[i]) : v[i] + step * (A.h[i] - g[i]);
}
__global__ void k_axpby(int n, double a, const double* p, double b, const double* q, double d,
                        double* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = (q ? a * p[i] + b * q[i] : a * p[i]) / d;
}
__global__ void k_box(int n, const double* in, const double* l, const double* u, double* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = clampv(in[i], l[i], u[i]);
}
// result assembly on the work instance (engine.py:663-680)
__global__ void k_unscale(KArgs A, const double* x, const double* y, const double* gx,
                          const double* gty, double* xo, double* yo, double* slack, double* lam) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int j = tid; j < A.n; j += nt) {
    const double d = A.d2[j];
    xo[j] = x[j] * d;
    lam[j] = A.c0[j] - gty[j] / d;
  }
  for (int i = tid; i < A.m; i += nt) {
    const double d = A.d1[i];
    yo[i] = y[i] * d;
    slack[i] = gx[i] / d - A.h0[i];
  }
}

}  // namespace pdcs

namespace pdcs {

// ---------------------------------------------------------------------------
// Persistent trials for small instances (C1 class: thousands of rows, no cone
// blocks, one column panel).  A trial of the graph path is three ~8 us
// kernels bound by launch and grid-drain latency; here ONE cooperative launch
// (one CTA per SM) runs every trial up to the batch end with grid-wide
// barriers between the phases:
//   X (primal step) | sync | Y (G^ x~ + dual step) | sync | line search |
//   [accepted] T (G^T y_hat + beta partials) | sync | beta
// Every CTA keeps an identical copy of the control block in shared memory and
// runs both controllers redundantly on the same partial sums read in the same
// order (bit-identical decisions, no extra barrier); CTA 0 writes it back at
// the end.  The arithmetic per element is the graph path's (k_step_x,
// y_epilogue, t_epilogue, ctrl_*_body).  Vectors written in one phase and read
// by other CTAs in the next are loaded coherently (ld.global / .cg).
// ---------------------------------------------------------------------------
template <int VWY, int VWT>
__global__ void __launch_bounds__(BS, 1) k_persist(KArgs A, TileSrc SY, TileSrc ST, double* pX, double* pY,
                                                   double* pT, int cap, long long max_trials) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ PdcsCtrl sc;
  __shared__ double sred[16];
  constexpr int NW = sizeof(PdcsCtrl) / sizeof(long long);
  for (int i = threadIdx.x; i < NW; i += blockDim.x)
    reinterpret_cast<long long*>(&sc)[i] = reinterpret_cast<const long long*>(A.ctrl)[i];
  __syncthreads();
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gstride = gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  const int wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), wt = gridDim.x * (blockDim.x >> 5);
  long long trials = 0;
  while (!sc.stop && trials < max_trials) {
    ++trials;
    {  // X: pending Halpern + primal candidate (k_step_x)
      const bool pend = sc.pending != 0;
      const bool inject = sc.nan_after >= 0 && sc.n_primal_proj >= sc.nan_after;
      const double a = sc.pa, b = sc.pb, be = sc.pbeta, et = sc.peta, W = sc.pW, tau = sc.tau;
      const double opb = 1.0 + be, tot = W + et;
      double acc[GX_N] = {0.0, 0.0, 0.0};
      for (int j = gtid; j < A.n; j += gstride) {
        double xn, gn;
        if (pend) {
          const double xo = A.x[j];
          xn = a * (opb * A.xh[j] - be * xo) + b * __ldg(A.xa + j);
          const double go = A.gty[j];
          // G^T y_hat was written by other CTAs in the last T phase: L2 load
          gn = a * (opb * __ldcg(A.gth + j) - be * go) + b * __ldg(A.gtya + j);
          A.xb[j] = (W == 0.0) ? xn : (W * A.xb[j] + et * xn) / tot;
          A.x[j] = xn;
          A.gty[j] = gn;
        } else {
          xn = A.x[j];
          gn = A.gty[j];
        }
        const double cj = __ldg(A.c + j);
        const double v = xn - tau * (cj - gn);
        double lj, uj;
        box_bounds<false>(A, j, 0, lj, uj);
        double p = clampv(v, lj, uj);
        if (j == 0 && inject) p = __longlong_as_double(0x7ff8000000000000ll);
        A.xh[j] = p;
        A.xt[j] = 2.0 * p - xn;
        const double d = p - xn;
        acc[GX_XX] += xn * xn;
        acc[GX_DXDX] += d * d;
        acc[GX_CX] += cj * p;
      }
      block_store_mask<GX_N>(acc, 0u, pX, cap, blockIdx.x);
    }
    grid.sync();
    {  // Y: w = G^ x~ and the dual candidate (k_step_y_lane)
      const YCoef k = y_coef(&sc);
      double acc[GY_N] = {0.0, 0.0, 0.0, 0.0, 0.0};
      constexpr int RPW = 32 / VWY;
      const int sub = lane & (VWY - 1);
      for (int base = wg * RPW; base < A.m; base += wt * RPW) {
        const int r = base + lane / VWY;
        const double dot = lane_row<VWY, 3>(SY, A.xt, nullptr, r, sub, A.m, 0, 0);
        if (sub == 0 && r < A.m) y_epilogue<false>(A, k, r, dot, acc, 0, 0);
      }
      block_store_mask<GY_N>(acc, 0u, pY, cap, blockIdx.x);
    }
    grid.sync();
    ctrl_ls_body<1>(&sc, pX, cap, pY, cap, sred, nullptr);
    __syncthreads();
    if (sc.stop) break;
    if (!sc.accepted) {
      grid.sync();  // the partials are rewritten by the next trial's X
      continue;
    }
    {  // T: G^T y_hat and the beta partials (k_step_t_lane)
      double acc[GT_N] = {0.0, 0.0, 0.0};
      constexpr int RPW = 32 / VWT;
      const int sub = lane & (VWT - 1);
      for (int base = wg * RPW; base < A.n; base += wt * RPW) {
        const int j = base + lane / VWT;
        const double dot = lane_row<VWT, 3>(ST, A.yh, nullptr, j, sub, A.n, 0, 0);
        if (sub == 0 && j < A.n) t_epilogue<false>(A, j, dot, acc, 0);
      }
      block_store_mask<GT_N>(acc, 0u, pT, cap, blockIdx.x);
    }
    grid.sync();
    ctrl_beta_body<1>(&sc, pT, cap, sred, A.err, nullptr);
    __syncthreads();
  }
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < NW; i += blockDim.x)
      reinterpret_cast<long long*>(A.ctrl)[i] = reinterpret_cast<const long long*>(&sc)[i];
  }
}

}  // namespace pdcs
