// Device-side building blocks of libpdcs: NaN-propagating selects, deterministic
// reductions, and the cone projections (box, SOC, rescaled SOC, exponential and
// dual exponential cone).  Compiled with --fmad=false so that elementwise
// expressions round exactly like the numpy reference (each * and + rounds).
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/pdcs.h"

namespace pdcs {

constexpr int BS = 256;         // threads per CTA for streaming kernels
constexpr int NSM = 148;        // B200 SMs
constexpr int MAX_GRID = NSM * 8;

// ---------------------------------------------------------------------------
// NaN-propagating selects (np.maximum / np.clip propagate NaN; fmax does not,
// SURVEY 8(a') item 11).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double pos_part(double v) { return v < 0.0 ? 0.0 : v; }
__device__ __forceinline__ double neg_clip(double v) { return v > 0.0 ? 0.0 : v; }
__device__ __forceinline__ double clampv(double v, double lo, double hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}
// max for infinity norms: NaN wins (np.max propagates NaN)
__device__ __forceinline__ double nanmax(double a, double b) {
  return (a != a) ? a : ((b != b) ? b : (a > b ? a : b));
}
__device__ __forceinline__ double dmin(double a, double b) { return a < b ? a : b; }
__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }

// ---------------------------------------------------------------------------
// L2 eviction-priority hints.  Streams touched once per iteration (CSR
// values/indices, state vectors) are loaded and stored evict_first so that the
// randomly gathered vectors (x~ for G^ x~, y_hat for G^T y_hat) and the
// freshly written y_hat / x~ keep their lines in the 126 MB L2.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t policy_stream() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_keep() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// evict_last for a fraction of the lines (the rest evict_first): used when the
// gathered vector is larger than the L2 set-aside, so a stable subset stays.
__device__ __forceinline__ uint64_t policy_keep_frac(float f) {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, %1;" : "=l"(p) : "f"(f));
  return p;
}
// Measured on B200 (profiles/r01_*): with the hot SpMVs tiled so each
// gathered slice fits in L2, plain LRU beats these policies, and a persisting
// set-aside steals bandwidth from the streams -- so the hints compile to
// plain loads/stores unless PDCS_L2_HINTS is defined.
// The hints are a template switch of the step kernels (HINT) so both forms
// can be measured; kL2Hints is the default of the plain helpers.
constexpr bool kL2Hints = false;
template <bool H = kL2Hints>
__device__ __forceinline__ double ld_hint(const double* a, uint64_t pol) {
  if (!H) return __ldg(a);
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
template <bool H = kL2Hints>
__device__ __forceinline__ int ld_hint(const int* a, uint64_t pol) {
  if (!H) return __ldg(a);
  int v;
  asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
// Gather load with an explicit L2 fill size: GP = 0 plain, 1 = 64 B, 2 = 128 B
// (random 8-byte gathers otherwise pull larger lines from HBM).
// GP 3: coherent L2 load (ld.global.cg) for a vector the same kernel writes
// (the persistent trial kernel gathers x~ / y_hat produced by other CTAs)
template <int GP>
__device__ __forceinline__ double ld_gather(const double* a) {
  if (GP == 0) return __ldg(a);
  if (GP == 3) return __ldcg(a);
  double v;
  if (GP == 1) asm("ld.global.nc.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(a));
  else asm("ld.global.nc.L2::128B.f64 %0, [%1];" : "=d"(v) : "l"(a));
  return v;
}

// coherent (non-.nc) load for buffers the same kernel also writes
template <bool H = kL2Hints>
__device__ __forceinline__ double ldc_hint(const double* a, uint64_t pol) {
  if (!H) return *a;
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
template <bool H = kL2Hints>
__device__ __forceinline__ void st_hint(double* a, double v, uint64_t pol) {
  if (!H) {
    *a = v;
    return;
  }
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}

// ---------------------------------------------------------------------------
// Deterministic reductions.  Sums go down a fixed shuffle tree to lane 0 and
// are broadcast from there, so every lane sees the bit-identical value.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  return __shfl_sync(0xffffffffu, v, 0);
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = nanmax(v, __shfl_down_sync(0xffffffffu, v, off));
  return __shfl_sync(0xffffffffu, v, 0);
}
__device__ __forceinline__ int warp_and(int v) { return __all_sync(0xffffffffu, v); }

// Block-wide reduction of NS sums and NM maxima; result written by thread 0
// into partials (layout [q][cap]) at column `slot`.  blockDim.x must be a
// multiple of 32 and <= 1024.
template <int NS, int NM>
__device__ __forceinline__ void block_store(double (&s)[NS], double (&mx)[NM], double* part_s,
                                            double* part_m, int cap, int slot) {
  __shared__ double sh[(NS + NM > 0 ? NS + NM : 1) * 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    double v = s[q];
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    if (lane == 0) sh[q * 32 + wid] = v;
  }
#pragma unroll
  for (int q = 0; q < NM; ++q) {
    double v = mx[q];
    for (int off = 16; off > 0; off >>= 1) v = nanmax(v, __shfl_down_sync(0xffffffffu, v, off));
    if (lane == 0) sh[(NS + q) * 32 + wid] = v;
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      double v = lane < nw ? sh[q * 32 + lane] : 0.0;
      for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
      if (lane == 0) part_s[q * cap + slot] = v;
    }
#pragma unroll
    for (int q = 0; q < NM; ++q) {
      double v = lane < nw ? sh[(NS + q) * 32 + lane] : 0.0;
      for (int off = 16; off > 0; off >>= 1) v = nanmax(v, __shfl_down_sync(0xffffffffu, v, off));
      if (lane == 0) part_m[q * cap + slot] = v;
    }
  }
  __syncthreads();
}

// Cooperative group abstractions for segment (cone block) work: a warp or a
// whole CTA handles one block; reductions return the same value to all
// members.
struct WarpGrp {
  int rank, size;
  __device__ WarpGrp() : rank(threadIdx.x & 31), size(32) {}
  __device__ double sum(double v) const { return warp_sum(v); }
  __device__ double max(double v) const { return warp_max(v); }
  __device__ int all(int v) const { return warp_and(v); }
  __device__ void sync() const { __syncwarp(); }
};

// W lanes of a warp per block (32 / W blocks side by side).  Every collective
// names only the group's lanes, so the groups of one warp may diverge
// (different branches or trip counts) without waiting on each other.
template <int W>
struct SubGrp {
  int rank, size;
  unsigned mask;
  __device__ SubGrp()
      : rank(threadIdx.x & (W - 1)), size(W),
        mask((W == 32 ? 0xffffffffu : ((1u << W) - 1u)) << ((threadIdx.x & 31) & ~(W - 1))) {}
  __device__ double sum(double v) const {
#pragma unroll
    for (int off = W / 2; off > 0; off >>= 1) v += __shfl_down_sync(mask, v, off, W);
    return __shfl_sync(mask, v, 0, W);
  }
  __device__ double max(double v) const {
#pragma unroll
    for (int off = W / 2; off > 0; off >>= 1) v = nanmax(v, __shfl_down_sync(mask, v, off, W));
    return __shfl_sync(mask, v, 0, W);
  }
  __device__ int all(int v) const { return (__ballot_sync(mask, v) & mask) == mask; }
  __device__ void sync() const { __syncwarp(mask); }
};

struct CtaGrp {
  int rank, size;
  double* sh;  // >= 33 doubles of shared scratch
  __device__ CtaGrp(double* s) : rank(threadIdx.x), size(blockDim.x), sh(s) {}
  __device__ double sum(double v) const {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    if (wid == 0) {
      double t = lane < nw ? sh[lane] : 0.0;
      for (int off = 16; off > 0; off >>= 1) t += __shfl_down_sync(0xffffffffu, t, off);
      if (lane == 0) sh[32] = t;
    }
    __syncthreads();
    return sh[32];
  }
  __device__ double max(double v) const {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int off = 16; off > 0; off >>= 1) v = nanmax(v, __shfl_down_sync(0xffffffffu, v, off));
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    if (wid == 0) {
      double t = lane < nw ? sh[lane] : 0.0;
      for (int off = 16; off > 0; off >>= 1) t = nanmax(t, __shfl_down_sync(0xffffffffu, t, off));
      if (lane == 0) sh[32] = t;
    }
    __syncthreads();
    return sh[32];
  }
  __device__ int all(int v) const { return __syncthreads_and(v); }
  __device__ void sync() const { __syncthreads(); }
};

// ---------------------------------------------------------------------------
// Exponential cone, K_exp = cl{(a,b,c): b > 0, c >= b exp(a/b)}
// (reference cones.py:74-331).  One thread per 3-vector.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double exp_guard(double x) { return x >= 709.0 ? INFINITY : exp(x); }

__device__ inline bool exp_member(double a, double b, double c) {
  if (b > 0.0) {
    double q = a / b;
    if (q < 709.0 && c >= 0.0 && c >= b * exp(q)) return true;
  }
  return (b >= 0.0 && b <= 0.0) && a <= 0.0 && c >= 0.0;
}

__device__ inline bool dual_exp_member(double u, double v, double w) {
  if (u > 0.0) return false;
  if (u >= 0.0) return v >= 0.0 && w >= 0.0;
  if (w <= 0.0) return false;
  return u * log(-u / w) - u + v >= 0.0;
}

// exp(rho) and exp(-rho) for the root search's function evaluations: the
// second as the correctly rounded reciprocal of the first while both are
// normal (|rho| < 700), one exp instead of two -- the exp calls are the
// largest share of the exp-cone kernel's instructions (ncu source page,
// profiles/r02_sweeps.txt).  The root itself is then tested and used
// through exp_from_rho, which keeps both exponentials as the reference has.
__device__ __forceinline__ void exp_pair(double rho, double& ep, double& en) {
  ep = exp_guard(rho);
  en = fabs(rho) < 700.0 ? __drcp_rn(ep) : exp_guard(-rho);
}

__device__ inline double exp_h(double r, double s, double t, double rho) {
  double qd = rho * (rho - 1.0) + 1.0;
  double ep, en;
  exp_pair(rho, ep, en);
  double ca = (rho - 1.0) * r + s, cb = r - rho * s;
  double t1 = (isfinite(ep) || ca != 0.0) ? ca * ep : 0.0;
  double t2 = (isfinite(en) || cb != 0.0) ? cb * en : 0.0;
  return t1 - t2 - qd * t;
}

// exp_h and its derivative at the same rho, sharing the two exponentials
// (the Newton step needs both).
__device__ inline void exp_hdh(double r, double s, double t, double rho, double& f, double& df) {
  double ep, en;
  exp_pair(rho, ep, en);
  const double qd = rho * (rho - 1.0) + 1.0;
  const double ca = (rho - 1.0) * r + s, cb = r - rho * s;
  const double t1 = (isfinite(ep) || ca != 0.0) ? ca * ep : 0.0;
  const double t2 = (isfinite(en) || cb != 0.0) ? cb * en : 0.0;
  f = t1 - t2 - qd * t;
  df = (rho * r + s) * ep + (r - (rho - 1.0) * s) * en - (2.0 * rho - 1.0) * t;
}

__device__ inline void exp_bracket(double r, double s, double t, double pdist, double ddist,
                                   double& lo_out, double& hi_out) {
  double lo = -1e15, hi = 1e15;
  double sm = dmin(s, 0.0), rm = dmin(r, 0.0);
  double dp = sqrt(dmax(pdist * pdist - sm * sm, 0.0));
  double dd = sqrt(dmax(ddist * ddist - rm * rm, 0.0));
  if (t > 0.0) {
    double rt = sqrt(r * r + s * s - r * s);
    double ps = (r > s) ? (r - s + rt) / r : -s / (r - s - rt);
    double pp = ((ps - 1.0) * r + s) / (ps * (ps - 1.0) + 1.0);
    lo = dmax(lo, log(t / pp));
  } else if (t < 0.0) {
    double rt = sqrt(r * r + s * s - r * s);
    double ps = (s > r) ? (r - rt) / s : (r - s) / (r + rt);
    double dpp = (r - ps * s) / (ps * (ps - 1.0) + 1.0);
    hi = dmin(hi, -log(-t / dpp));
  }
  if (r > 0.0) {
    double base = 1.0 - s / r;
    lo = dmax(lo, base);
    double tpu = dmax(1e-12, dmin(dd, dp + t));
    double pw = exp_guard(lo) / (lo * (lo - 1.0) + 1.0);
    if (lo < 2.0) pw = dmin(pw, exp(2.0) / 3.0);
    if (pw > 0.0) hi = dmin(hi, dmax(lo, base + tpu / r / pw));
  }
  if (s > 0.0) {
    double base = r / s;
    hi = dmin(hi, base);
    double tdl = -dmax(1e-12, dmin(dp, dd - t));
    double dw = -exp_guard(-hi) / (hi * (hi - 1.0) + 1.0);
    if (hi > -1.0) dw = dmax(dw, -2.718281828459045 / 3.0);
    if (dw < 0.0) lo = dmax(lo, dmin(hi, base - tdl / s / dw));
  }
  if (lo > hi) { lo = hi = 0.5 * (lo + hi); }
  if (lo != hi) {
    double fl = exp_h(r, s, t, lo), fu = exp_h(r, s, t, hi);
    if (fl * fu > 0.0) {
      if (fabs(fl) < fabs(fu)) hi = lo; else lo = hi;
    }
  }
  lo_out = lo;
  hi_out = hi;
}

// Root-finding controls of the projections (ProjectionSettings, cones.py:24-32):
// tol = root_tol, iters = max_root_iters.  The solver always uses the defaults
// (the reference's engine never passes settings); the standalone projection
// API passes the caller's.
struct RootCfg {
  double tol = 1e-12;
  int iters = 100;
};

// x0: optional Newton start (the block's root from the previous PDHG trial);
// NaN or outside (lo, hi) means the reference's midpoint start.
// cones.py:225-265: min(20, iters) damped Newton steps, then bisection up to
// `iters` evaluations in total, stopping at tol relative width.
__device__ inline double exp_root(double r, double s, double t, double lo, double hi,
                                  double x0 = NAN, RootCfg rc = RootCfg()) {
  const int newton = rc.iters < 20 ? rc.iters : 20, total = rc.iters;
  double x = (x0 > lo && x0 < hi) ? x0 : 0.5 * (lo + hi);
  bool done = false;
  for (int i = 0; i < newton; ++i) {
    double f, df;
    exp_hdh(r, s, t, x, f, df);
    if (fabs(f) <= 1e-15) { done = true; break; }
    if (f < 0.0) lo = x; else hi = x;
    if (hi <= lo) return 0.5 * (lo + hi);
    if (!isfinite(f) || df < 1e-13) break;
    double xn = x - f / df;
    if (fabs(xn - x) <= 1e-15 * dmax(1.0, fabs(xn))) {
      x = dmin(dmax(xn, lo), hi);
      done = true;
      break;
    }
    if (xn >= hi) x = dmin(0.5 * x + 0.95 * hi, hi);
    else if (xn <= lo) x = dmax(0.5 * x + 0.95 * lo, lo);
    else x = xn;
  }
  if (done) return dmin(dmax(x, lo), hi);
  for (int i = 0; i < total - newton; ++i) {
    x = 0.5 * (lo + hi);
    if (exp_h(r, s, t, x) < 0.0) lo = x; else hi = x;
    if (hi - lo <= rc.tol * dmax(1.0, fabs(hi))) break;
  }
  return 0.5 * (lo + hi);
}

// Returns false when the root gives no valid point (reference returns None).
__device__ inline bool exp_from_rho(double r, double s, double t, double rho, double* p,
                                    double* dist) {
  double qd = rho * (rho - 1.0) + 1.0;
  double en = exp_guard(-rho);
  double lin_a = (rho - 1.0) * r + s;
  double lin_b = (r - rho * s) * en + qd * t;
  double cond_a = fabs(rho - 1.0) * fabs(r) + fabs(s);
  double cond_b = (fabs(r - rho * s) * en + qd * fabs(t)) * en;
  if (cond_a <= cond_b) {
    double ep = exp_guard(rho);
    if (lin_a <= 0.0 || !isfinite(ep)) return false;
    p[0] = rho * lin_a / qd; p[1] = lin_a / qd; p[2] = ep * lin_a / qd;
  } else {
    double lin = lin_b * en;
    if (lin <= 0.0) return false;
    p[0] = rho * lin / qd; p[1] = lin / qd; p[2] = lin_b / qd;
  }
  double d0 = p[0] - r, d1 = p[1] - s, d2 = p[2] - t;
  *dist = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
  return true;
}

// Cheap cases of the projection onto K_exp (cones.py:298-320): non-finite
// input (error), member, polar member, the flat piece, and the heuristics'
// early exit.  Returns true with o set when one of them decides; otherwise
// leaves the heuristic primal point and both heuristic distances in H for the
// root stage.
struct ExpHeur {
  double vp0, vp1, vp2, pdist, ddist;
};

__device__ __forceinline__ bool exp_cheap(double r, double s, double t, double* o, int* err,
                                          ExpHeur& H) {
  if (!(isfinite(r) && isfinite(s) && isfinite(t))) {
    *err = PDCS_ERR_EXP_NONFINITE;
    o[0] = r; o[1] = s; o[2] = t;
    return true;
  }
  // exp(r/s) serves both the membership test (cones.py:80-88) and the primal
  // heuristic (cones.py:102-113): computed once (the same operations, so the
  // same bits as computing it twice)
  const double ers = s > 0.0 ? exp_guard(r / s) : 0.0;
  const bool member = s > 0.0 ? (r / s < 709.0 && t >= 0.0 && t >= s * ers)
                              : ((s >= 0.0 && s <= 0.0) && r <= 0.0 && t >= 0.0);
  if (member) { o[0] = r; o[1] = s; o[2] = t; return true; }
  if (dual_exp_member(-r, -s, -t)) { o[0] = 0.0; o[1] = 0.0; o[2] = 0.0; return true; }
  if (r <= 0.0 && s <= 0.0) { o[0] = r; o[1] = 0.0; o[2] = t < 0.0 ? 0.0 : t; return true; }
  // primal heuristic (cones.py:102-113)
  double vp0 = dmin(r, 0.0), vp1 = 0.0, vp2 = dmax(t, 0.0);
  double pdist = sqrt((r - vp0) * (r - vp0) + s * s + (t - vp2) * (t - vp2));
  if (s > 0.0) {
    double tp = s * ers;
    if (isfinite(tp)) {
      tp = dmax(t, tp);
      if (tp - t < pdist) { vp0 = r; vp1 = s; vp2 = tp; pdist = tp - t; }
    }
  }
  // polar heuristic (cones.py:116-126)
  double vd0 = 0.0, vd1 = dmin(s, 0.0), vd2 = dmin(t, 0.0);
  double ddist = sqrt(r * r + (s - vd1) * (s - vd1) + (t - vd2) * (t - vd2));
  if (r > 0.0) {
    double td = -r * exp_guard(s / r - 1.0);
    if (isfinite(td)) {
      td = dmin(t, td);
      if (t - td < ddist) { vd0 = r; vd1 = s; vd2 = td; ddist = t - td; }
    }
  }
  double tol = 1e-12 * dmax(dmax(1.0, fabs(r)), dmax(fabs(s), fabs(t)));
  double merr = dmax(dmax(fabs(vp0 + vd0 - r), fabs(vp1 + vd1 - s)), fabs(vp2 + vd2 - t));
  double inner = vp0 * vd0 + vp1 * vd1 + vp2 * vd2;
  if (dmin(pdist, ddist) <= tol || (merr <= tol && inner <= tol)) {
    o[0] = vp0; o[1] = vp1; o[2] = vp2;
    return true;
  }
  H.vp0 = vp0; H.vp1 = vp1; H.vp2 = vp2; H.pdist = pdist; H.ddist = ddist;
  return false;
}

// Warm start: up to 3 plain Newton steps from the previous trial's root,
// with the reference's own stopping tests.  The converged root is used only
// if it lies inside the cheap bracket bounds (rho >= 1 - s/r for r > 0,
// rho <= r/s for s > 0, cones.py:200-211) and gives a valid point no farther
// than the primal heuristic; h's root in the full bracket is unique, so such
// a root is the one the reference finds.  Returns true (o set, *rho_io
// updated) on success; anything else goes to exp_rooted.
__device__ __forceinline__ bool exp_warm(double r, double s, double t, const ExpHeur& H, double* o,
                                         double* rho_io) {
  if (!isfinite(*rho_io)) return false;
  double x = *rho_io, rho = NAN;
  for (int i = 0; i < 3; ++i) {
    double f, df;
    exp_hdh(r, s, t, x, f, df);
    if (!isfinite(f) || !(df >= 1e-13)) break;
    if (fabs(f) <= 1e-15) { rho = x; break; }
    const double xn = x - f / df;
    if (fabs(xn - x) <= 1e-15 * dmax(1.0, fabs(xn))) { rho = xn; break; }
    x = xn;
  }
  if (!isfinite(rho) || (r > 0.0 && rho < 1.0 - s / r) || (s > 0.0 && rho > r / s)) return false;
  double pr[3], dr;
  if (!exp_from_rho(r, s, t, rho, pr, &dr) || !(dr <= H.pdist)) return false;
  *rho_io = rho;
  o[0] = pr[0]; o[1] = pr[1]; o[2] = pr[2];
  return true;
}

// The reference's root stage (cones.py:321-326): bracket, safeguarded Newton
// + bisection (started from the warm root when it lies inside the bracket),
// the candidate from the root, else the primal heuristic point.
__device__ inline void exp_rooted(double r, double s, double t, const ExpHeur& H, double* o,
                                  double* rho_io, RootCfg rc) {
  double lo, hi;
  exp_bracket(r, s, t, H.pdist, H.ddist, lo, hi);
  const double rho = exp_root(r, s, t, lo, hi, rho_io ? *rho_io : NAN, rc);
  if (rho_io) *rho_io = rho;
  double pr[3], dr;
  if (exp_from_rho(r, s, t, rho, pr, &dr) && dr <= H.pdist) {
    o[0] = pr[0]; o[1] = pr[1]; o[2] = pr[2];
    return;
  }
  o[0] = H.vp0; o[1] = H.vp1; o[2] = H.vp2;
}

// Euclidean projection of (r, s, t) onto K_exp (cones.py:298-326).  Sets *err
// for non-finite input (the reference raises NumericalError).
// rho_io (optional): warm start for the Newton root-find, updated with the
// root found -- consecutive PDHG trials project nearby points, so Newton
// starts next to its root instead of at the bracket midpoint.
__device__ inline void proj_exp3(double r, double s, double t, double* o, int* err,
                                 double* rho_io = nullptr, RootCfg rc = RootCfg()) {
  ExpHeur H;
  if (exp_cheap(r, s, t, o, err, H)) return;
  if (rho_io && exp_warm(r, s, t, H, o, rho_io)) return;
  exp_rooted(r, s, t, H, o, rho_io, rc);
}

// proj_exp3 without the root stage: true when the cheap cases or the warm
// start decide (o set, *rho_io updated), false when the bracket + root search
// is needed (o and *rho_io then undefined / untouched).
__device__ __forceinline__ bool proj_exp3_fast(double r, double s, double t, double* o, int* err,
                                               double* rho_io) {
  ExpHeur H;
  if (exp_cheap(r, s, t, o, err, H)) return true;
  return exp_warm(r, s, t, H, o, rho_io);
}

// Dual cone via Moreau: P_{K*}(v) = v + P_K(-v) (cones.py:329-331).
__device__ inline void proj_dual_exp3(double r, double s, double t, double* o, int* err,
                                      double* rho_io = nullptr, RootCfg rc = RootCfg()) {
  double q[3];
  proj_exp3(-r, -s, -t, q, err, rho_io, rc);
  o[0] = r + q[0]; o[1] = s + q[1]; o[2] = t + q[2];
}

__device__ __forceinline__ bool proj_dual_exp3_fast(double r, double s, double t, double* o, int* err,
                                                    double* rho_io) {
  double q[3];
  if (!proj_exp3_fast(-r, -s, -t, q, err, rho_io)) return false;
  o[0] = r + q[0]; o[1] = s + q[1]; o[2] = t + q[2];
  return true;
}

__device__ inline void set_err(int* gerr, int code) {
  if (code && gerr) atomicCAS(gerr, 0, code);
}

// ---------------------------------------------------------------------------
// Segment projection by a cooperating group (warp or CTA): block of `dim`
// elements at in[0..dim), written to out[0..dim) (may alias in).  `sc` is the
// block's scale slice (or nullptr), smode selects none/direct/inverse.
// Kinds: FREE, ZERO, NONNEG, SOC (plain or rescaled), EXP, DUAL_EXP.
// ---------------------------------------------------------------------------
template <class G>
__device__ inline double rsoc_phi(const G& g, const double* in, const double* sc, int smode,
                                  int dim, double a0inv_base, double mu, double t0) {
  // phi(mu) = sum a_i^2 y_i^2 / (1 + 2 mu a_i^2)^2 - (t0 / (1 - 2 mu))^2  (cones.py:347-350)
  double acc = 0.0;
  for (int i = 1 + g.rank; i < dim; i += g.size) {
    double di = smode == PDCS_SCALE_INVERT ? 1.0 / sc[i] : sc[i];
    double a = di / a0inv_base;
    double a2 = a * a;
    double y = in[i];
    double ay2 = a2 * y * y;
    double den = 1.0 + 2.0 * mu * a2;
    acc += ay2 / (den * den);
  }
  double s = g.sum(acc);
  double tt = t0 / (1.0 - 2.0 * mu);
  return s - tt * tt;
}

template <class G>
__device__ inline void proj_rescaled_soc(const G& g, const double* in, double* out,
                                         const double* sc, int smode, int dim, int* gerr,
                                         RootCfg rc = RootCfg()) {
  double d0 = smode == PDCS_SCALE_INVERT ? 1.0 / sc[0] : sc[0];
  double t0 = in[0];
  // membership tests (cones.py:372-375)
  double s_ay2 = 0.0, s_ya2 = 0.0;
  for (int i = 1 + g.rank; i < dim; i += g.size) {
    double di = smode == PDCS_SCALE_INVERT ? 1.0 / sc[i] : sc[i];
    double a = di / d0;
    double a2 = a * a;
    double y = in[i];
    s_ay2 += a2 * y * y;
    double q = y / a;
    s_ya2 += q * q;
  }
  s_ay2 = g.sum(s_ay2);
  s_ya2 = g.sum(s_ya2);
  if (t0 >= 0.0 && t0 * t0 >= s_ay2) {
    for (int i = g.rank; i < dim; i += g.size) out[i] = in[i];
    return;
  }
  if (t0 <= 0.0 && t0 * t0 >= s_ya2) {
    for (int i = g.rank; i < dim; i += g.size) out[i] = 0.0;
    return;
  }
  if (t0 == 0.0) {
    double acc = 0.0;
    for (int i = 1 + g.rank; i < dim; i += g.size) {
      double di = smode == PDCS_SCALE_INVERT ? 1.0 / sc[i] : sc[i];
      double a = di / d0;
      double zb = in[i] / (1.0 + a * a);
      double az = a * zb;
      acc += az * az;
    }
    double nrm = sqrt(g.sum(acc));
    g.sync();
    for (int i = 1 + g.rank; i < dim; i += g.size) {
      double di = smode == PDCS_SCALE_INVERT ? 1.0 / sc[i] : sc[i];
      double a = di / d0;
      out[i] = in[i] / (1.0 + a * a);
    }
    if (g.rank == 0) out[0] = nrm;
    return;
  }
  // bracket (cones.py:387-412)
  double lo = 0.0, hi = 0.0;
  bool ok = false;
  if (t0 > 0.0) {
    lo = 0.0;
    for (int j = 1; j < 53; ++j) {
      double cand = 0.5 * (1.0 - ldexp(1.0, -j));
      if (rsoc_phi(g, in, sc, smode, dim, d0, cand, t0) < 0.0) { hi = cand; ok = true; break; }
    }
  } else {
    for (int j = 1; j < 53; ++j) {
      double cand = 0.5 * (1.0 + ldexp(1.0, -j));
      if (rsoc_phi(g, in, sc, smode, dim, d0, cand, t0) < 0.0) { lo = cand; ok = true; break; }
    }
    if (ok) {
      ok = false;
      hi = 1.0;
      for (int j = 0; j < 80; ++j) {
        if (rsoc_phi(g, in, sc, smode, dim, d0, hi, t0) > 0.0) { ok = true; break; }
        hi *= 2.0;
      }
    }
  }
  if (!ok) {
    if (g.rank == 0) set_err(gerr, PDCS_ERR_RSOC_BRACKET);
    for (int i = g.rank; i < dim; i += g.size) out[i] = in[i];
    return;
  }
  // Brent's method with xtol = 1e-16, rtol = 8.9e-16, maxiter = max_root_iters
  // (the classic algorithm scipy's brentq implements; not converging within
  // maxiter raises in scipy, so it is a numerical error here, cones.py:414-425).
  const double xtol = 1e-16, rtol = 8.9e-16;
  double xpre = lo, xcur = hi, xblk = 0.0, fblk = 0.0, spre = 0.0, scur = 0.0;
  double fpre = rsoc_phi(g, in, sc, smode, dim, d0, xpre, t0);
  double fcur = rsoc_phi(g, in, sc, smode, dim, d0, xcur, t0);
  double mu = xcur;
  bool conv = true;
  if (fpre == 0.0) {
    mu = xpre;
  } else if (fcur != 0.0) {
    conv = false;
    for (int it = 0; it < rc.iters; ++it) {
      if (fpre != 0.0 && fcur != 0.0 && (signbit(fpre) != signbit(fcur))) {
        xblk = xpre; fblk = fpre; spre = scur = xcur - xpre;
      }
      if (fabs(fblk) < fabs(fcur)) {
        xpre = xcur; xcur = xblk; xblk = xpre;
        fpre = fcur; fcur = fblk; fblk = fpre;
      }
      double delta = (xtol + rtol * fabs(xcur)) / 2.0;
      double sbis = (xblk - xcur) / 2.0;
      if (fcur == 0.0 || fabs(sbis) < delta) { conv = true; break; }
      if (fabs(spre) > delta && fabs(fcur) < fabs(fpre)) {
        double stry;
        if (xpre == xblk) {
          stry = -fcur * (xcur - xpre) / (fcur - fpre);
        } else {
          double dpre = (fpre - fcur) / (xpre - xcur);
          double dblk = (fblk - fcur) / (xblk - xcur);
          stry = -fcur * (fblk * dblk - fpre * dpre) / (dblk * dpre * (fblk - fpre));
        }
        if (2.0 * fabs(stry) < dmin(fabs(spre), 3.0 * fabs(sbis) - delta)) {
          spre = scur; scur = stry;
        } else {
          spre = sbis; scur = sbis;
        }
      } else {
        spre = sbis; scur = sbis;
      }
      xpre = xcur; fpre = fcur;
      if (fabs(scur) > delta) xcur += scur;
      else xcur += (sbis > 0.0 ? delta : -delta);
      fcur = rsoc_phi(g, in, sc, smode, dim, d0, xcur, t0);
    }
    mu = xcur;
  }
  if (!conv && g.rank == 0) set_err(gerr, PDCS_ERR_RSOC_ROOT);
  g.sync();
  for (int i = 1 + g.rank; i < dim; i += g.size) {
    double di = smode == PDCS_SCALE_INVERT ? 1.0 / sc[i] : sc[i];
    double a = di / d0;
    out[i] = in[i] / (1.0 + 2.0 * mu * (a * a));
  }
  if (g.rank == 0) out[0] = t0 / (1.0 - 2.0 * mu);
}

template <class G>
__device__ inline void proj_segment(const G& g, int kind, int smode, const double* in,
                                    double* out, const double* sc, int dim, int* gerr,
                                    RootCfg rc = RootCfg()) {
  switch (kind) {
    case PDCS_FREE:
      for (int i = g.rank; i < dim; i += g.size) out[i] = in[i];
      return;
    case PDCS_ZERO:
      for (int i = g.rank; i < dim; i += g.size) out[i] = 0.0;
      return;
    case PDCS_NONNEG:
      for (int i = g.rank; i < dim; i += g.size) out[i] = pos_part(in[i]);
      return;
    case PDCS_EXP:
    case PDCS_DUAL_EXP: {
      if (g.rank == 0) {
        double o[3];
        int e = 0;
        if (kind == PDCS_EXP) proj_exp3(in[0], in[1], in[2], o, &e, nullptr, rc);
        else proj_dual_exp3(in[0], in[1], in[2], o, &e, nullptr, rc);
        set_err(gerr, e);
        out[0] = o[0]; out[1] = o[1]; out[2] = o[2];
      }
      g.sync();
      return;
    }
    case PDCS_SOC: {
      int uniform = 1;
      if (smode != PDCS_SCALE_NONE) {
        double s0 = sc[0];
        int u = 1;
        for (int i = g.rank; i < dim; i += g.size) u &= (sc[i] == s0);
        uniform = g.all(u);
      }
      if (!uniform) {
        proj_rescaled_soc(g, in, out, sc, smode, dim, gerr, rc);
        g.sync();
        return;
      }
      double acc = 0.0;
      for (int i = 1 + g.rank; i < dim; i += g.size) acc += in[i] * in[i];
      double nx = sqrt(g.sum(acc));
      double t = in[0];
      g.sync();
      if (nx <= t) {
        for (int i = g.rank; i < dim; i += g.size) out[i] = in[i];
      } else if (nx <= -t) {
        for (int i = g.rank; i < dim; i += g.size) out[i] = 0.0;
      } else {
        double coef = 0.5 * (t + nx);
        double ratio = coef / nx;
        for (int i = 1 + g.rank; i < dim; i += g.size) out[i] = ratio * in[i];
        if (g.rank == 0) out[0] = coef;
      }
      g.sync();
      return;
    }
    default:
      return;
  }
}

}  // namespace pdcs
