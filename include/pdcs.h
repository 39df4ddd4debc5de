/*
 * pdcs.h -- C ABI of libpdcs.so, the B200 (sm_100a) engine behind the
 * drop-in `paper_2603_15504_b200` solver package.
 *
 * The reference (conic_pdhg 0.1.0, /root/reference/pkg/src/conic_pdhg) has no
 * C ABI: its "operator API" is the Python surface `solve(problem, options)`
 * (engine.py:683-689) and the seams below it.  Every entry point here
 * replaces one of those seams; the replaced reference symbol is cited on each
 * declaration.  The Python package keeps the reference's names and calls
 * these entry points through ctypes.
 *
 * Conventions
 *  - All pointers named d_* / in / out are DEVICE pointers owned by the caller
 *    (the Python layer allocates them as torch CUDA tensors).  The library
 *    never frees caller memory.  Host pointers are named h_*.
 *  - `stream` is a cudaStream_t passed as void*.  NULL = legacy default stream.
 *  - Return codes: 0 ok, 1 CUDA error, 2 bad argument, 3 numerical failure.
 *    `pdcs_last_error()` returns a thread-local message for the last failure.
 *  - Vectors are FP64, sparse indices are int32, CSR with sorted column
 *    indices and no duplicates (the canonical scipy layout the reference
 *    builds in linalg.py:35-39).
 *  - An engine handle is used by one host thread at a time.
 */
#ifndef PDCS_H
#define PDCS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PDCS_ABI_VERSION 1

/* Cone kinds (model.py:28-37).  RSOC never reaches the library: it is
 * rotated to SOC in presolve exactly as model.py:262-304 does. */
enum {
  PDCS_FREE = 0,
  PDCS_ZERO = 1,
  PDCS_NONNEG = 2,
  PDCS_SOC = 3,
  PDCS_EXP = 4,
  PDCS_DUAL_EXP = 5
};

/* Scale modes of a projected block: project onto {z : diag(s) z in K} with
 * s = nothing / the block's slice of the scale vector / its reciprocal
 * (cones.py:452-549). */
enum { PDCS_SCALE_NONE = 0, PDCS_SCALE_DIRECT = 1, PDCS_SCALE_INVERT = 2 };

/* One cone block of a segmented projection.  `start` indexes the vector the
 * projection is applied to; the scale slice is scale[start : start+dim]. */
typedef struct PdcsBlock {
  int32_t kind;
  int32_t start;
  int32_t dim;
  int32_t smode;
} PdcsBlock;

/* Exit / stop reasons of the device-resident inner loop. */
enum {
  PDCS_STOP_NONE = 0,
  PDCS_STOP_CHECK = 1,     /* k_bar % check_freq == 0 (engine.py:627) */
  PDCS_STOP_MAXITER = 2,   /* k_bar >= max_iter (engine.py:626) */
  PDCS_STOP_BATCH = 3,     /* k_bar >= k_bar_stop (host-requested batch end) */
  PDCS_STOP_PRINT = 4,     /* k_bar % print_freq == 0 (engine.py:628, logging only) */
  PDCS_STOP_ERROR = 5      /* NumericalError inside the step (engine.py:612-620) */
};

enum {
  PDCS_ERR_NONE = 0,
  PDCS_ERR_NAN_LINESEARCH = 1,  /* engine.py:221-228 */
  PDCS_ERR_TRIAL_CAP = 2,       /* engine.py:243 */
  PDCS_ERR_EXP_NONFINITE = 3,   /* cones.py:301-302 */
  PDCS_ERR_RSOC_BRACKET = 4,    /* cones.py:395-412 */
  PDCS_ERR_BETA = 5,            /* non-finite reflection parameter */
  PDCS_ERR_RSOC_ROOT = 6        /* brentq did not converge in max_root_iters (cones.py:414-425) */
};

/* Control block of the device-resident loop (SolverState, engine.py:94-113,
 * plus the pending Halpern/average coefficients).  Lives in device memory;
 * read/written as a whole by pdcs_engine_get_ctrl / pdcs_engine_set_ctrl.
 * Every field is 8 bytes so the layout is trivially portable. */
typedef struct PdcsCtrl {
  int64_t k_bar, k, trials, k_bar_stop, max_iter, check_freq, print_freq;
  int64_t stop, reason, error, new_iter, accepted, pending, adaptive, use_fixed_beta;
  int64_t n_trials_total, n_accepted_total, nan_after, n_primal_proj, spare0;
  double eta_hat, eta_try, eta, omega, beta, W, fixed_beta;
  double tau, sigma;
  double pa, pb, pbeta, peta, pW;
  double c1, h1;
  double movement, interaction, eta_bar, p_obj, d_obj, max_err;
  double spare[4];
} PdcsCtrl;

/* Everything the engine needs.  All d_* are device pointers (caller-owned).
 * Matrix arrays are the SCALED work matrix G^ = D1 G D2 (written by
 * pdcs_precondition from d_g_val0) and its transpose.  Vectors c,h,l,u are the
 * scaled instance; c0,h0,l0,u0 the unscaled work (post-RSOC) instance used by
 * the original-space checks (engine.py:399-404). */
typedef struct PdcsEngineDesc {
  int32_t n, m, num_box, nnz;
  int32_t m_zero;   /* rows [0, m_zero) belong to the ZERO block   */
  int32_t m_elem;   /* rows [m_zero, m_elem) to the NONNEG block; the rest are cone blocks */
  int32_t n_pcones, n_dcones;
  const int32_t* h_pcone_kind; const int32_t* h_pcone_dim;   /* stored primal blocks (host) */
  const int32_t* h_dcone_kind; const int32_t* h_dcone_dim;   /* stored dual blocks (host)   */
  int32_t allow_nonuniform_dual_soc;
  int32_t pad0;
  /* scaled matrix G^ (CSR) and G^T (CSR), plus CSR->CSR^T position map */
  int32_t* d_g_rowptr; int32_t* d_g_colidx; double* d_g_val;
  int32_t* d_gt_rowptr; int32_t* d_gt_colidx; double* d_gt_val;
  int32_t* d_perm;
  const double* d_g_val0;
  /* instance vectors */
  double *d_c, *d_h, *d_l, *d_u;
  const double *d_c0, *d_h0, *d_l0, *d_u0;
  double *d_d1, *d_d2;
  /* iterate state: z, z_hat, z_bar, anchor, previous anchor */
  double *d_x, *d_y, *d_xh, *d_yh, *d_xb, *d_yb, *d_xa, *d_ya, *d_xpa, *d_ypa;
  /* product caches: G x, G^T y, anchors, G x_hat (raw w and (w+gx)/2), G^T y_hat */
  double *d_gx, *d_gty, *d_gxa, *d_gtya, *d_w, *d_gxh, *d_gth, *d_gtr, *d_xt;
  /* scratch (check path) */
  double *d_tx0, *d_tx1, *d_tx2, *d_ty0, *d_ty1, *d_ty2;
} PdcsEngineDesc;

typedef struct PdcsEngine PdcsEngine;

/* ---- library ------------------------------------------------------------ */
const char* pdcs_last_error(void);
int pdcs_abi_version(void);
/* Returns the number of kernels this library launched since load (host-side
 * counter; used by bench.py's gpu_launches). */
int64_t pdcs_launch_count(void);

/* ---- standalone kernels (no engine) ------------------------------------- */

/* y = A x for an r x k CSR.  Replaces SparseMatrix.matvec / .rmatvec
 * (linalg.py:63-73; scipy csr_matvec).  Rows of up to `thread_row_max` nnz
 * are summed sequentially in index order (bit-identical to csr_matvec);
 * longer rows use deterministic lane-split reductions. */
int pdcs_spmv_csr(int32_t nrows, const int32_t* d_rowptr, const int32_t* d_colidx,
                  const double* d_val, const double* d_x, double* d_y, void* stream);

/* CSR of A^T (sorted, stable) plus perm[p] = position in A of entry p of A^T.
 * Replaces the CSC mirror built by SparseMatrix.__init__ (linalg.py:39).
 * Scratch for the stable radix sort is allocated and freed internally. */
int pdcs_transpose_csr(int32_t nrows, int32_t ncols, int32_t nnz, const int32_t* d_rowptr,
                       const int32_t* d_colidx, const double* d_val, int32_t* d_t_rowptr,
                       int32_t* d_t_colidx, double* d_t_val, int32_t* d_perm, void* stream);

/* Segmented projection of `in` onto a product of blocks (elements outside
 * every block are copied).  Replaces project_cone / project_*_set
 * (cones.py:452-549).  h_blocks is a HOST array (copied to the device
 * internally).  h_err receives the numerical error code (PDCS_ERR_*). */
int pdcs_project_segments(int32_t len, const double* d_in, double* d_out, const PdcsBlock* h_blocks,
                          int32_t nblocks, const double* d_scale, int32_t* h_err, void* stream);

/* pdcs_project_segments with explicit root-finding controls: the fields of
 * ProjectionSettings (cones.py:24-32).  root_tol is the exp-cone bisection
 * stopping width (cones.py:263); max_root_iters bounds the exp-cone
 * Newton + bisection evaluations (cones.py:227, 256) and brentq's iterations
 * of the rescaled SOC (cones.py:421; not converging sets PDCS_ERR_RSOC_ROOT).
 * pdcs_project_segments uses the defaults (1e-12, 100). */
int pdcs_project_segments_ex(int32_t len, const double* d_in, double* d_out, const PdcsBlock* h_blocks,
                             int32_t nblocks, const double* d_scale, double root_tol,
                             int32_t max_root_iters, int32_t* h_err, void* stream);

/* out = clip(in, l, u) componentwise, NaN-propagating like np.clip
 * (project_box, cones.py:46-51). */
int pdcs_project_box(int32_t len, const double* d_in, const double* d_l, const double* d_u,
                     double* d_out, void* stream);

/* out = (a p + b q) / d (q may be NULL: out = a p / d).  Building block of
 * reflected_halpern_step / update_weighted_average (engine.py:246-277). */
int pdcs_vec_axpby(int32_t len, double a, const double* d_p, double b, const double* d_q,
                   double d, double* d_out, void* stream);

/* ---- engine --------------------------------------------------------------- */
/* Builds the transpose of the matrix pattern, the cone block tables and the
 * SpMV schedules; allocates the library's small internal workspace (control
 * block, reduction partials, schedules).  `stream` becomes the engine's
 * stream and must not be the legacy default stream (CUDA graphs are captured
 * on it).  Replaces SparseMatrix construction + block_slices. */
int pdcs_engine_create(const PdcsEngineDesc* desc, void* stream, PdcsEngine** out);
void pdcs_engine_destroy(PdcsEngine* e);

/* Ruiz (ruiz_iters rounds) + optional Pock-Chambolle + block uniformity +
 * clamp, then G^ = D1 G D2, c^, h^, l^, u^ (scaling.py:65-135).  With
 * enabled = 0, d1 = d2 = 1 (the identity ScalingPair, engine.py:298-300).
 * With enabled = 2 the caller has already written d1/d2 (as-is mode used by
 * the step-level API: cone scales taken from the problem's ConeSpecs). */
int pdcs_precondition(PdcsEngine* e, int32_t enabled, int32_t ruiz_iters, int32_t use_pock_chambolle);

/* Setup statistics of the scaled instance: out[0]=||c^||_1 out[1]=||h^||_1
 * out[2]=||c^||_2^2 out[3]=||h^||_2^2 out[4]=max|G^_ij| out[5]=max row abs
 * sum (engine.py:322-336, restart.py:180-186). */
int pdcs_stats(PdcsEngine* e, double* h_out);

/* Launch configuration chosen at create: h_out[16] = {vw(G^), vw(G^T), grid
 * step_x, grid step_y, grid step_t, keep fraction x~, keep fraction y_hat,
 * persisting-L2 bytes, long rows of G^, long rows of G^T, primal cone blocks,
 * dual cone blocks, column panels of G^, of G^T, step-kernel lanes per row
 * of G^, of G^T}. */
int pdcs_engine_info(PdcsEngine* e, double* h_out);

int pdcs_engine_get_ctrl(PdcsEngine* e, PdcsCtrl* h_ctrl);
int pdcs_engine_set_ctrl(PdcsEngine* e, const PdcsCtrl* h_ctrl);

/* Runs the inner loop (adaptive_step_pdhg + G^T y_hat + beta + reflected
 * Halpern + weighted average, engine.py:564-611) on the device until the
 * control block's stop flag is set.  Slots are replayed from a CUDA graph of
 * `slots_per_graph` line-search trials. */
int pdcs_run_inner(PdcsEngine* e, int32_t slots_per_graph);

/* ---- batched engines (many C1-class solves per GPU) ----
 * One CUDA graph forks into every member engine's stream (each branch runs
 * `slots` line-search trials of that engine, exactly the pdcs_run_inner
 * sequence), joins, and gathers the members' control blocks.  pdcs_batch_run
 * replays it until every member's device loop has stopped; members the host
 * keeps stopped (ctrl.stop = 1) are gated off.  Members: non-sharded engines,
 * each used by one host thread at a time between runs.  The reference solves
 * one problem per call (engine.py:683-689); results per member are
 * bit-identical to pdcs_run_inner. */
typedef struct PdcsBatch PdcsBatch;
int pdcs_batch_create(PdcsEngine** engines, int32_t n, void* stream, PdcsBatch** out);
int pdcs_batch_run(PdcsBatch* b, int32_t slots_per_graph);
void pdcs_batch_destroy(PdcsBatch* b);

/* Runs `reps` line-search trials eagerly (not from the graph) with CUDA
 * events between the stages and returns the number of stages; h_ms[i] is the
 * mean device time of stage i and h_names[i] its name (static strings).
 * Advances the iteration like pdcs_run_inner would.  For bench.py. */
int pdcs_profile_slot(PdcsEngine* e, int32_t reps, double* h_ms, const char** h_names, int32_t cap);

/* Applies the pending Halpern/average update so z, z_bar, gx, gty are
 * current (the deferred part of engine.py:602-610). */
int pdcs_flush(PdcsEngine* e);

/* out = G^ in (transpose=0, in: x-space) or G^T in (transpose=1). */
int pdcs_engine_spmv(PdcsEngine* e, int32_t transpose, const double* d_in, double* d_out);

/* Metric partial sums for compute_errors (termination.py:91-147).
 * mode 0: scaled instance at (x, y, gx, gty) as given.
 * mode 1: original (unscaled work) instance at x = x~ d2, y = y~ d1,
 *         G x = gx~ / d1, G^T y = gty~ / d2.
 * h_out[PDCS_NMET] receives the reductions listed in pdcs_met_index. */
#define PDCS_NMET 20
enum {
  PDCS_MET_RV2 = 0, PDCS_MET_RVMAX, PDCS_MET_HMAX, PDCS_MET_GXMAX, PDCS_MET_RPMAX, PDCS_MET_YH,
  PDCS_MET_H1, PDCS_MET_V1SQ, PDCS_MET_V1MAX, PDCS_MET_V2SQ, PDCS_MET_V2MAX, PDCS_MET_CMAX,
  PDCS_MET_GTYMAX, PDCS_MET_CX, PDCS_MET_LSUM, PDCS_MET_USUM, PDCS_MET_C1, PDCS_MET_NONFINITE,
  PDCS_MET_XX, PDCS_MET_YY
};
int pdcs_metrics(PdcsEngine* e, int32_t mode, const double* d_x, const double* d_y,
                 const double* d_gx, const double* d_gty, double* h_out);

/* Infeasibility ray quantities on the original instance
 * (termination.py:230-273), with ||x|| and ||y|| (original space) supplied.
 * h_out: [0]=max dual-ray lam1 viol [1]=max lam2 viol [2]=y.h [3]=sum l lam+
 * [4]=sum u lam- [5]=max primal-ray residual viol [6]=max box recession viol
 * [7]=max cone viol [8]=c.x_hat */
#define PDCS_NRAY 9
int pdcs_rays(PdcsEngine* e, const double* d_x, const double* d_y, const double* d_gx,
              const double* d_gty, double xnorm, double ynorm, double* h_out);

/* One normalized-gap probe z(t) (restart.py:62-77): with b1 = gty - c^,
 * b2 = h^ - gx: zx = P_X(x + t tau b1), zy = P_Y(y + t sigma b2).
 * h_out: [0]=||x - zx||^2 [1]=||y - zy||^2 [2]=b1.(zx - x) [3]=b2.(zy - y) */
int pdcs_gap_probe(PdcsEngine* e, const double* d_x, const double* d_y, const double* d_gx,
                   const double* d_gty, double t, double tau, double sigma, double* h_out);

/* k (1..16) gap probes at host values h_ts[0..k) with one read-back; problems
 * without cone blocks evaluate all k in a single pass over the iterate (the
 * search of restart.py:80-132 then needs a pass per 4 bisection levels, not
 * per level).  h_out[4i..4i+3] = pdcs_gap_probe's four sums at t = h_ts[i]
 * (same formulas; summation order of the batched pass). */
int pdcs_gap_probes(PdcsEngine* e, const double* d_x, const double* d_y, const double* d_gx,
                    const double* d_gty, const double* h_ts, int32_t k, double tau, double sigma,
                    double* h_out);

/* h_out[0] = ||a - b||^2 over x-space (space=0) or y-space (space=1);
 * d_b may be NULL (then ||a||^2). */
int pdcs_dist2(PdcsEngine* e, int32_t space, const double* d_a, const double* d_b, double* h_out);
/* h_out[0] = (a - b).(c - d); d_b / d_d may be NULL (treated as 0). */
int pdcs_dot_diff(PdcsEngine* e, int32_t space, const double* d_a, const double* d_b,
                  const double* d_c, const double* d_d, double* h_out);

/* Set projections on the engine's (scaled) instance (cones.py:498-549):
 * which 0 = P_X (primal set), 1 = P_Y (dual set), 2 = K_d* residual set,
 * 3 = K_p* on the cone part (x-space positions >= num_box),
 * 4 = K_p on the cone part. */
int pdcs_project_set(PdcsEngine* e, int32_t which, const double* d_in, double* d_out);
/* pdcs_project_set with the ProjectionSettings fields (cones.py:24-32; see
 * pdcs_project_segments_ex); the set functions of cones.py:498-549 take them. */
int pdcs_project_set_ex(PdcsEngine* e, int32_t which, const double* d_in, double* d_out,
                        double root_tol, int32_t max_root_iters);

/* out = x - tau (c^ - gty) (space 0) or y + sigma (h^ - w) (space 1): the
 * two pre-projection updates of _pdhg_candidate (engine.py:155-161). */
int pdcs_step_input(PdcsEngine* e, int32_t space, const double* d_v, const double* d_g,
                    double step, double* d_out);
/* out = a*p + b*q over x-space (space 0) or y-space (space 1). */
int pdcs_axpby(PdcsEngine* e, int32_t space, double a, const double* d_p, double b,
               const double* d_q, double* d_out);

/* Result assembly on the work instance (engine.py:663-680, scaling.py:138-140):
 * x = x~ d2, y = y~ d1, slack = gx~ / d1 - h0, lam = c0 - gty~ / d2, where
 * gx~ = G^ x~ and gty~ = G^T y~. */
int pdcs_unscale(PdcsEngine* e, const double* d_x, const double* d_y, const double* d_gx,
                 const double* d_gty, double* d_xo, double* d_yo, double* d_slack, double* d_lam);

/* Declare that every box coordinate j < num_box has the same unscaled
 * bounds [lo, hi] (infinities allowed).  The step kernels then form the
 * scaled bounds as lo / d2_j, hi / d2_j -- the same division the scaling
 * kernel performs, so the values are identical -- and stream d2 instead of
 * l^ and u^ (one n-vector instead of two in the x-step and the G^T step).
 * Replaces nothing in the reference (project_box, cones.py:46-51, reads the
 * arrays); an optimisation of the same arithmetic. */
int pdcs_engine_set_uniform_box(PdcsEngine* e, double lo, double hi);

/* Small block-free engines run their trials in one cooperative launch per
 * pdcs_run_inner (chosen at create); on = 0 keeps them on the CUDA-graph path
 * (solves on concurrent host threads: a cooperative launch occupies the GPU). */
int pdcs_engine_set_persist(PdcsEngine* e, int32_t on);

/* ---- multi-GPU ------------------------------------------------
 * A sharded solve gives every rank a contiguous row slice of G^ (cut at dual
 * cone-block boundaries) and a contiguous x-slice (cut at primal cone-block
 * boundaries); every rank keeps full-length x-space buffers.  With a
 * communicator attached, one graph slot (one PDHG trial) adds, inside the
 * CUDA graph:
 *   - after the primal half-step on the x-slice: all-gather of x~ (G_p x~
 *     needs all of it);
 *   - an all-reduce of the 5 y-space + 3 x-space line-search sums;
 *   - after G_p^T y_hat_p over all of x-space: reduce-scatter, each rank
 *     receiving its x-slice of G^T y_hat;
 *   - an all-reduce of the 3 x-space beta sums.
 * Equal x-slices (cut r = r ceil(n / nranks)) use ncclAllGather /
 * ncclReduceScatter; block-aligned unequal slices use grouped per-root
 * broadcasts / reduces.  x-space buffers must then hold
 * nranks * ceil(n / nranks) doubles.  Outside its slice a rank's x-space
 * state goes stale during a batch; pdcs_allgather_x restores full copies
 * (the host calls it after pdcs_flush, before any check).  libnccl is the one
 * the process already loaded (torch's), opened with dlopen. */
int pdcs_comm_unique_id(unsigned char* h_id128);
int pdcs_engine_set_comm(PdcsEngine* e, const unsigned char* h_id128, int32_t rank, int32_t nranks);
/* x-slices of all ranks: h_cuts[0] = 0 <= ... <= h_cuts[nranks] = n.  Required
 * when nranks > 1 (after pdcs_engine_set_comm). */
int pdcs_engine_set_xsplit(PdcsEngine* e, const int32_t* h_cuts, int32_t nranks);
/* Every rank's slice of each x-space device vector d_vecs[0..count) to all
 * ranks (no-op without an x-split). */
int pdcs_allgather_x(PdcsEngine* e, double* const* d_vecs, int32_t count);

/* Debug hook standing in for the reference tests' monkeypatched
 * project_primal_set (T/test_engine.py:300-317): after `after_calls` primal
 * projections inside the loop, x_hat is replaced by NaN.  -1 disables. */
int pdcs_debug_inject_nan(PdcsEngine* e, int64_t after_calls);

#ifdef __cplusplus
}
#endif
#endif /* PDCS_H */
