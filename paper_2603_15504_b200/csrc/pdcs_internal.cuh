// Internal engine structures shared by the libpdcs translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "pdcs_device.cuh"

namespace pdcs {

// Row schedule of one CSR matrix for the SpMV kernels: rows of up to
// `long_t` nnz are handled by VW lanes each (VW = 1: one thread, summed in
// index order exactly like scipy's csr_matvec); longer rows are split into
// chunks summed by whole CTAs, then finalised per row in chunk order.
struct SpmvPlan {
  int nrows = 0, ncols = 0, nnz = 0;
  const int* rowptr = nullptr;
  const int* colidx = nullptr;
  const double* val = nullptr;
  int vw = 1;
  int step_vw = 1;  // lanes per row of the fused step kernels (panel rows are shorter)
  double len_cv = 0.0;  // coefficient of variation of the short rows' lengths
  int long_t = 1 << 30;
  int n_long = 0, n_chunks = 0;
  int* d_long_rows = nullptr;     // [n_long]
  int* d_long_first = nullptr;    // [n_long + 1] first chunk of each long row
  int4* d_chunks = nullptr;       // [n_chunks] (row, begin, end, long-row index | LONG_DENSE)
  double* d_chunk_out = nullptr;  // [n_chunks]
  unsigned* d_long_cnt = nullptr;  // [n_long] chunks of the row finished (k_long_partial ticket)
  int grid = 1;                   // CTAs of the short-row kernel
  // row classes of a mixed-length matrix (class split): the rows of more than
  // CLS_SHORT entries (cls_vw lanes per row); the epilogue sums the others
  int* d_cls_long = nullptr;
  int n_cls_short = 0, n_cls_long = 0, cls_vw = 8;
  long long nnz_cls_long = 0;
  int cls_grid_l = 1;
  int pass_grid = 1;              // CTAs of the panel partial-sum passes (k_lane_pass)
  int* d_tiles = nullptr;         // [ntiles + 1] CSR-stream tile boundaries (rows)
  int ntiles = 0;
};

// Column-panelled copy of a CSR matrix for the fused step SpMVs: columns are
// cut into `np` equal ranges so the slice of the gathered vector a pass reads
// fits in L2; pass p sums row i's entries of panel p on top of the partial
// of passes 0..p-1 (index order is preserved, so a thread-per-row sum is
// still bit-identical to scipy's csr_matvec).  Long rows are left out (they
// go through the chunked path).  Offsets are flattened [panel][row]: panel
// p's row i spans po[p*nrows + i] .. po[p*nrows + i + 1].
struct PanelPlan {
  int np = 1;
  int width = 0;
  int* d_po = nullptr;      // [np*nrows + 1]
  int* d_pci = nullptr;     // [nnz_short] absolute column indices
  double* d_pva = nullptr;  // [nnz_short]
  int* d_pperm = nullptr;   // [nnz_short] position in the CSR
  int nnz_short = 0;
};

// Cone-block table of one space split into size classes.
struct BlockTable {
  PdcsBlock* d_all = nullptr;  // exp, thread, half-warp, warp, cta, giant classes in that order
  int n_exp = 0, n_thread = 0, n_half = 0, n_warp = 0, n_cta = 0, n_giant = 0;
  int g_exp = 0, g_thread = 0, g_half = 0, g_warp = 0, g_cta = 0, g_giant = 0;  // fixed grids (partial slots)
  double* d_gpart = nullptr;  // giant-block partial sums [n_giant][2][g_giant]
  double* d_gcoef = nullptr;  // giant-block SOC coefficients [n_giant][8]
  // y-step exp blocks in two launches (k_exp_y_fast / k_exp_y_slow): CTA c of
  // the fast kernel owns blocks [c*exp_per, (c+1)*exp_per) and queues the ones
  // needing the root search at d_queue[c*exp_per ...], d_qcount[c] of them
  bool exp_split = false;
  int exp_per = 0;
  int half_w = 16;    // lanes per block of the half-warp class kernel (PDCS_TUNE halfw / xhalfw = 4)
  int half_minb = 1;  // CTAs per SM the y-step half-warp block kernel is compiled for (PDCS_TUNE halfminb)
  int exp_minb = 4;  // CTAs per SM the exp kernels are compiled for (register budget; PDCS_TUNE expminb)
  int* d_queue = nullptr;   // [n_exp]
  int* d_qcount = nullptr;  // [g_exp]
  int total() const { return n_exp + n_thread + n_half + n_warp + n_cta + n_giant; }
  int grids() const {
    return g_exp * (exp_split ? 2 : 1) + g_thread + g_half + g_warp + g_cta + g_giant;
  }
};

constexpr int GIANT_MIN = 1 << 16;  // uniform dual SOC blocks above this use the whole grid
constexpr int GIANT_GRID = 2 * 148;

constexpr int TILE_ROWS = BS;    // rows per CSR-stream tile (one per thread in phase 2)
constexpr int TILE_NNZ = 2048;   // entries per tile; longer rows use the chunked path
constexpr int WARP_CLASS_MAX = 4096;  // dims above this get a whole CTA
constexpr int THREAD_CLASS_MAX = 4;   // dims up to this get one thread
constexpr int HALF_CLASS_MAX = 16;    // then up to this 16 lanes (two blocks per warp)
constexpr int CTA_BLOCK_THREADS = 512;

// Reduction groups of one line-search trial.
enum { GX_XX = 0, GX_DXDX, GX_CX, GX_N };
enum { GY_YY = 0, GY_DYDY, GY_INTER, GY_RP2, GY_YH, GY_N };
enum { GT_RD2 = 0, GT_LSUM, GT_USUM, GT_N };

struct Engine {
  PdcsEngineDesc d;  // caller pointers
  cudaStream_t stream = nullptr;
  int n = 0, m = 0, nbox = 0, nnz = 0, m_zero = 0, m_elem = 0;
  std::vector<int> pkind, pdim, dkind, ddim;
  int allow_nonuniform_dual_soc = 0;

  SpmvPlan G, GT;  // G^ (m x n) and G^T (n x m)
  PanelPlan PG, PGT;  // panelled copies used by the fused step kernels
  double* d_wpart_y = nullptr;  // partial sums of the G^ passes  [m]
  double* d_wpart_x = nullptr;  // partial sums of the G^T passes [n]
  BlockTable tabX, tabY;
  bool has_xblocks = false, has_yblocks = false;
  std::vector<PdcsBlock> xblocks;  // primal cone blocks (host copy)
  BlockTable tabXs;                // the blocks of this rank's x-slice (sharded)
  double* d_exp_rho = nullptr;     // Newton warm starts of the dual exp blocks [2 n_exp]
  bool xsplit = false;             // x-space split across the ranks (pdcs_engine_set_xsplit)
  // uniformity groups for preconditioning (blocks whose scale is made uniform)
  PdcsBlock* d_unif_x = nullptr;
  int n_unif_x = 0;
  PdcsBlock* d_unif_y = nullptr;
  int n_unif_y = 0;

  // device workspace owned by the library
  PdcsCtrl* d_ctrl = nullptr;
  double* d_red = nullptr;  // scalars handed from the line-search controller to the beta controller
  double* d_partX = nullptr;
  double* d_partY = nullptr;
  double* d_partT = nullptr;
  int capX = 0, capY = 0, capT = 0;
  int gridX = 1, gridXE = 1;  // x-space streaming grid
  int gridStepX = 1;          // k_step_x grid (one wave of resident CTAs)
  int gridStepX2 = 1;         // k_step_x2 grid (16-byte variant)
  float keep_xt = 1.0f, keep_yh = 1.0f;  // evict_last fractions (L2 set-aside / vector bytes)
  bool tile_y = false, tile_t = false;  // step SpMVs: tiled CSR-stream or lane-mapped
  int gp = 0;  // lane-step gathers: 0 plain, 1 with the L2::64B fill hint
  bool fuse_ctrl = true;  // fold the controllers into the last CTA of the step kernels
  bool pdl = true;        // programmatic dependent launches between the step kernels of a trial
  bool split = false;     // split step SpMVs: gather-only panel passes + streaming epilogues
  bool soc_tile = false;  // dual SOC blocks projected inside the tiled y-step (d_rowhead)
  bool vec = false;       // 16-byte streaming epilogues of the split step
  bool cls_y = false, cls_t = false;
  bool xexp_fused = false;  // primal exp coordinates' x-step inside the exp block kernel (k_exp_xstep)
  bool texp_fused = false;  // their G^T rows and lambda_2 projection in one kernel (k_exp_tstep)
  bool exp_fused = false;   // exp rows' y-step inside the exp block kernel (k_exp_ystep)
  bool yblk_fused = false;  // half-warp dual blocks projected in the class-split epilogue (k_y_epi_blk)
  int yblk_ga = 1;          // its CTAs for the elementwise rows (the rest take the blocks)  // class-split step SpMVs (mixed row lengths)
  bool persist = false;   // small instances: one cooperative launch runs all trials (k_persist)
  int pgrid = 0;          // its grid (one CTA per SM)
  double *d_pX = nullptr, *d_pY = nullptr, *d_pT = nullptr;  // its partial slots [NQ][pgrid]
  int* d_rowhead = nullptr;  // [m] first row of the cone block of each row, -1 outside
  bool ubox = false;      // every box coordinate has the bounds [ubox_l, ubox_u] (unscaled)
  double ubox_l = 0.0, ubox_u = 0.0;
  int precond_mode = 0;   // last pdcs_precondition mode (2 = as-is: bounds unscaled)
  bool hs = false;        // evict_first L2 policy on the panel passes' streams
  size_t l2_persist = 0;                 // persisting-L2 set-aside requested at create
  int gridY = 1;              // y-space streaming grid (elementwise kernels)
  double* d_partC = nullptr;  // check path partials [max(PDCS_NMET, 4 GAP_K)][capC]
  int capC = 0;
  double* d_out = nullptr;  // [64]
  int* d_err = nullptr;     // numerical error code of projections
  unsigned* d_ticket = nullptr;  // finished-CTA counters of the folded controllers [4]
  double* h_pinned = nullptr;  // pinned readback [128]: [0, 64) general, [64, 128) 2nd ctrl copy
  cudaEvent_t ev_ctrl[2] = {nullptr, nullptr};  // run_inner's in-flight ctrl read-backs

  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int graph_slots = 0;
  int64_t graph_nodes = 0;

  // sharded mode (row slice of G^ + NCCL communicator)
  void* comm = nullptr;       // ncclComm_t
  int rank = 0, nranks = 1;
  double* d_yred = nullptr;   // all-reduced trial scalars [16]: y sums, x sums, t sums
  double* d_gtp = nullptr;    // local G^T y_hat partial sums [n, padded]
  // x-space split: this rank steps x-slice [xs0, xs1) (all of x when not sharded)
  int xs0 = 0, xs1 = 0;
  int xcnt = 0;                // equal-slice length (0: slices cut at block boundaries)
  std::vector<int> xcut;       // [nranks + 1]
};

}  // namespace pdcs
