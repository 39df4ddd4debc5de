// Kernels of libpdcs.  Included by pdcs_engine.cu only.
#pragma once
#include "pdcs_internal.cuh"

namespace pdcs {

// All engine pointers, passed by value to kernels.
struct KArgs {
  int n, m, nbox, m_zero, m_elem;
  const double *c, *h, *l, *u, *c0, *h0, *l0, *u0, *d1, *d2;
  double *x, *y, *xh, *yh, *xb, *yb, *xa, *ya;
  double *gx, *gty, *gxa, *gtya, *w, *gxh, *gth, *gtr, *xt;
  double *tx0, *tx1, *tx2, *ty0, *ty1, *ty2;
  PdcsCtrl* ctrl;
  int* err;
};

// gate: 0 = always run, 1 = skip when stopped, 2 = skip when stopped or the
// current trial was rejected.
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
                                          bool& lng) {
  double s = 0.0;
  lng = false;
  if (row < nrows) {
    const int b = __ldg(rp + row), e = __ldg(rp + row + 1);
    if (e - b > long_t) {
      lng = true;
      if (sub == 0) s = longv[row];
    } else {
      for (int j = b + sub; j < e; j += VW) s += __ldg(va + j) * __ldg(x + __ldg(ci + j));
    }
  }
  if (VW > 1) {
#pragma unroll
    for (int off = VW / 2; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off, VW);
  }
  return s;
}

// Generic SpMV for short rows; long rows are already in y (written by
// k_long_final) and are left untouched.
template <int VW>
__global__ void __launch_bounds__(BS) k_spmv(int nrows, const int* __restrict__ rp,
                                             const int* __restrict__ ci,
                                             const double* __restrict__ va,
                                             const double* __restrict__ x, double* y,
                                             int long_t) {
  const int lane = threadIdx.x & 31, sub = lane & (VW - 1);
  constexpr int RPW = 32 / VW;
  const int wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int wt = gridDim.x * (blockDim.x >> 5);
  for (int base = wg * RPW; base < nrows; base += wt * RPW) {
    const int row = base + lane / VW;
    bool lng;
    double s = row_dot<VW>(rp, ci, va, x, row, sub, nrows, long_t, y, lng);
    if (sub == 0 && row < nrows && !lng) y[row] = s;
  }
}

__global__ void k_long_partial(const int4* __restrict__ ch, int nch, const int* __restrict__ ci,
                               const double* __restrict__ va, const double* __restrict__ x,
                               double* out, const PdcsCtrl* ctrl, int gate) {
  if (gated(ctrl, gate)) return;
  __shared__ double sh[33];
  CtaGrp g(sh);
  for (int c = blockIdx.x; c < nch; c += gridDim.x) {
    const int4 q = ch[c];
    double s = 0.0;
    for (int j = q.y + threadIdx.x; j < q.z; j += blockDim.x) s += va[j] * x[ci[j]];
    s = g.sum(s);
    if (threadIdx.x == 0) out[c] = s;
  }
}

__global__ void k_long_final(const int* __restrict__ rows, const int* __restrict__ first, int nl,
                             const double* __restrict__ part, double* y, const PdcsCtrl* ctrl,
                             int gate) {
  if (gated(ctrl, gate)) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nl) return;
  double s = 0.0;
  for (int c = first[i]; c < first[i + 1]; ++c) s += part[c];
  y[rows[i]] = s;
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
    proj_segment(g, kind, sm, P.in + s, P.out + s, sm ? P.scale + s : nullptr, dim, A.err);
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
__global__ void __launch_bounds__(BS) k_step_x(KArgs A, double* part, int cap) {
  const PdcsCtrl* C = A.ctrl;
  if (C->stop) return;
  const bool pend = C->pending != 0;
  const double a = C->pa, b = C->pb, be = C->pbeta, et = C->peta, W = C->pW, tau = C->tau;
  const double opb = 1.0 + be, tot = W + et;
  const bool inject = C->nan_after >= 0 && C->n_primal_proj >= C->nan_after;
  double acc[GX_N] = {0.0, 0.0, 0.0};
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < A.n; j += gridDim.x * blockDim.x) {
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
    const double v = xn - tau * (cj - gn);
    if (j < A.nbox) {
      double p = clampv(v, A.l[j], A.u[j]);
      if (j == 0 && inject) p = __longlong_as_double(0x7ff8000000000000ll);
      A.xh[j] = p;
      A.xt[j] = 2.0 * p - xn;
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

// y-space fused with w = G^ x~: pending Halpern/average, then
// y_hat = P_Y(y + sigma (h - w)), gx_hat = (w + gx)/2 and the reductions
// ||y||^2, ||dy||^2, dy.(w - gx), the beta residual ||r - P_{K_d*} r||^2 of
// r = gx_hat - h, and y_hat.h.  Block rows are left for k_blk_*.
template <int VW>
__global__ void __launch_bounds__(BS) k_step_y(KArgs A, int nrows, const int* __restrict__ rp,
                                               const int* __restrict__ ci,
                                               const double* __restrict__ va, int long_t,
                                               double* part, int cap) {
  const PdcsCtrl* C = A.ctrl;
  if (C->stop) return;
  const bool pend = C->pending != 0;
  const double a = C->pa, b = C->pb, be = C->pbeta, et = C->peta, W = C->pW, sigma = C->sigma;
  const double opb = 1.0 + be, tot = W + et;
  double acc[GY_N] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const int lane = threadIdx.x & 31, sub = lane & (VW - 1);
  constexpr int RPW = 32 / VW;
  const int wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int wt = gridDim.x * (blockDim.x >> 5);
  for (int base = wg * RPW; base < nrows; base += wt * RPW) {
    const int r = base + lane / VW;
    bool lng;
    const double dot = row_dot<VW>(rp, ci, va, A.xt, r, sub, nrows, long_t, A.w, lng);
    if (sub == 0 && r < nrows) {
      double yn, gn;
      if (pend) {
        const double yo = A.y[r];
        yn = a * (opb * A.yh[r] - be * yo) + b * A.ya[r];
        const double go = A.gx[r];
        gn = a * (opb * A.gxh[r] - be * go) + b * A.gxa[r];
        A.yb[r] = (W == 0.0) ? yn : (W * A.yb[r] + et * yn) / tot;
        A.y[r] = yn;
        A.gx[r] = gn;
      } else {
        yn = A.y[r];
        gn = A.gx[r];
      }
      const double hi = A.h[r];
      const double v = yn + sigma * (hi - dot);
      const double gh = 0.5 * (dot + gn);
      A.gxh[r] = gh;
      if (r < A.m_elem) {
        const bool zero = r < A.m_zero;
        const double p = zero ? v : pos_part(v);
        A.yh[r] = p;
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
  }
  block_store_mask<GY_N>(acc, 0u, part, cap, blockIdx.x);
}

// x-space fused with gth = G^T y_hat (accepted trials only): stores gth and the
// box part of the dual residual of beta: ||lam1 - P_Lambda lam1||^2 and the
// bound terms of the dual objective (model.py:182-237, termination.py:113-119).
template <int VW>
__global__ void __launch_bounds__(BS) k_step_t(KArgs A, int nrows, const int* __restrict__ rp,
                                               const int* __restrict__ ci,
                                               const double* __restrict__ va, int long_t,
                                               double* part, int cap) {
  const PdcsCtrl* C = A.ctrl;
  if (C->stop || !C->accepted) return;
  double acc[GT_N] = {0.0, 0.0, 0.0};
  const int lane = threadIdx.x & 31, sub = lane & (VW - 1);
  constexpr int RPW = 32 / VW;
  const int wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int wt = gridDim.x * (blockDim.x >> 5);
  for (int base = wg * RPW; base < nrows; base += wt * RPW) {
    const int j = base + lane / VW;
    bool lng;
    const double dot = row_dot<VW>(rp, ci, va, A.yh, j, sub, nrows, long_t, A.gtr, lng);
    if (sub == 0 && j < nrows) {
      A.gth[j] = dot;
      if (j < A.nbox) {
        const double lam = A.c[j] - dot;
        const double lj = A.l[j], uj = A.u[j];
        const bool lf = isfinite(lj), uf = isfinite(uj);
        const double pr = (!lf && !uf) ? 0.0 : (!lf ? neg_clip(lam) : (!uf ? pos_part(lam) : lam));
        const double v = lam - pr;
        acc[GT_RD2] += v * v;
        if (lf) acc[GT_LSUM] += lj * pos_part(lam);
        if (uf) acc[GT_USUM] += uj * pos_part(-lam);
      }
    }
  }
  block_store_mask<GT_N>(acc, 0u, part, cap, blockIdx.x);
}

__device__ __forceinline__ double cta_sum_range(const double* p, int n, CtaGrp& g) {
  double t = 0.0;
  for (int s = threadIdx.x; s < n; s += blockDim.x) t += p[s];
  return g.sum(t);
}

// Line-search controller (engine.py:183-243): one CTA.
__global__ void k_ctrl_ls(PdcsCtrl* C, const double* partX, int capX, const double* partY,
                          int capY, double* red) {
  if (C->stop) return;
  __shared__ double sh[33];
  CtaGrp g(sh);
  const double xx = cta_sum_range(partX + GX_XX * capX, capX, g);
  const double dxdx = cta_sum_range(partX + GX_DXDX * capX, capX, g);
  const double cx = cta_sum_range(partX + GX_CX * capX, capX, g);
  const double yy = cta_sum_range(partY + GY_YY * capY, capY, g);
  const double dydy = cta_sum_range(partY + GY_DYDY * capY, capY, g);
  const double inter = cta_sum_range(partY + GY_INTER * capY, capY, g);
  const double rp2 = cta_sum_range(partY + GY_RP2 * capY, capY, g);
  const double yh = cta_sum_range(partY + GY_YH * capY, capY, g);
  if (threadIdx.x != 0) return;
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

// Reflection parameter, Halpern coefficients, averaging weight and the stop
// tests of an accepted iteration (engine.py:590-628, termination.py:150-160).
__global__ void k_ctrl_beta(PdcsCtrl* C, const double* partT, int capT, const double* red,
                            const int* err) {
  if (C->stop || !C->accepted) return;
  __shared__ double sh[33];
  CtaGrp g(sh);
  const double rd2 = cta_sum_range(partT + GT_RD2 * capT, capT, g);
  const double ls = cta_sum_range(partT + GT_LSUM * capT, capT, g);
  const double us = cta_sum_range(partT + GT_USUM * capT, capT, g);
  if (threadIdx.x != 0) return;
  if (*err) {  // numerical failure inside a projection (exp non-finite, rsoc bracket)
    C->error = *err;
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
