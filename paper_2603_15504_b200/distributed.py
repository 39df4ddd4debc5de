"""Sharded multi-GPU solve (with its recommended refinement).

Rows of G^ (the y-space) are split into contiguous ranges, one per rank, cut
only at cone-block boundaries (ZERO / NONNEG rows may be cut anywhere; SOC,
EXP and DUAL_EXP blocks are indivisible) and balanced by nonzeros plus a row
term.  The x-space is split too: rank r steps x-slice [cut_r, cut_r+1)
(equal slices when no primal cone block straddles them), keeping full-length
buffers.  Per PDHG trial the device graph (NCCL, in-graph):
  all-gathers x~ after the primal half-step (G_p x~ needs all of it),
  all-reduces the 5 y-space + 3 x-space line-search sums,
  reduce-scatters the G_p^T y_hat_p partial sums (each rank gets its slice),
  all-reduces the 3 x-space beta sums.
This moves the bytes of one all-reduce of G^T y per trial but splits the
x-space streaming work (k_step_x and the G^T epilogue) N ways.  At a batch
end the host flushes the pending Halpern step and all-gathers the x-space
state, after which every rank holds identical full copies; the check path
then runs the reference's host logic on reductions that `ShardedDevice`
combines across ranks with torch.distributed.

Preconditioning: each rank uploads only its row slice; Ruiz + Pock-Chambolle
runs on the slice with the column statistics (max-abs per Ruiz round, 1-norms
for Pock-Chambolle) all-reduced over the ranks inside libpdcs, so every rank
holds its slice of D1 and the global D2 (SURVEY.md 8(e) "At setup").
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .device import DeviceEngine
from .model import Cone, ConeSpec, ConicProblem, dual_layout


# ---------------------------------------------------------------------------
# partition
# ---------------------------------------------------------------------------


def allowed_cuts(problem: ConicProblem) -> np.ndarray:
    """Row indices at which the y-space may be cut: every row boundary inside
    the ZERO / NONNEG rows, then only cone-block boundaries."""
    _, m_elem = dual_layout(problem)
    cuts = list(range(0, m_elem + 1))
    pos = 0
    for spec in problem.dual_cones:
        pos += spec.dim
        if pos > m_elem:
            cuts.append(pos)
    return np.unique(np.asarray(cuts + [problem.m], dtype=np.int64))


def partition_rows(problem: ConicProblem, world: int, row_weight: float = 1.0):
    """Contiguous [r0, r1) per rank, balanced by nnz + row_weight * rows."""
    if world < 1:
        raise ValueError("world must be >= 1")
    m = problem.m
    if world == 1 or m == 0:
        return [(0, m)] + [(m, m)] * (world - 1)
    nnz_row = np.diff(problem.G._csr.indptr).astype(np.float64)
    cum = np.concatenate([[0.0], np.cumsum(nnz_row + row_weight)])
    cuts = allowed_cuts(problem)
    total = cum[-1]
    bounds = [0]
    for k in range(1, world):
        target = total * k / world
        i = int(np.searchsorted(cum[cuts], target))
        cand = [cuts[j] for j in (i - 1, i) if 0 <= j < len(cuts)]
        best = min(cand, key=lambda c: abs(cum[c] - target))
        best = max(best, bounds[-1])
        bounds.append(int(best))
    bounds.append(m)
    return [(bounds[i], bounds[i + 1]) for i in range(world)]


def allowed_xcuts(problem: ConicProblem) -> np.ndarray:
    """x-space indices at which the x-space may be cut: anywhere inside the
    box coordinates, then only primal cone-block boundaries."""
    cuts = list(range(0, problem.num_box + 1))
    pos = problem.num_box
    for spec in problem.primal_cones:
        pos += spec.dim
        cuts.append(pos)
    return np.unique(np.asarray(cuts + [problem.n], dtype=np.int64))


def partition_cols(problem: ConicProblem, world: int) -> list[int]:
    """x-slice cuts [0 = c_0 <= ... <= c_world = n]: the equal split
    c_r = min(r ceil(n / world), n) when it cuts no primal cone block (the
    engine then uses NCCL all-gather / reduce-scatter), else the allowed cut
    nearest to r n / world."""
    n = problem.n
    if world < 1:
        raise ValueError("world must be >= 1")
    cnt = -(-n // world) if n else 0
    equal = [min(r * cnt, n) for r in range(world + 1)]
    allowed = allowed_xcuts(problem)
    ok = set(allowed.tolist())
    if all(c in ok for c in equal):
        return equal
    cuts = [0]
    for r in range(1, world):
        target = n * r / world
        i = int(np.searchsorted(allowed, target))
        cand = [int(allowed[j]) for j in (i - 1, i) if 0 <= j < len(allowed)]
        cuts.append(max(min(cand, key=lambda c: abs(c - target)), cuts[-1]))
    cuts.append(n)
    return cuts


def slice_problem(work: ConicProblem, r0: int, r1: int) -> ConicProblem:
    """The rank's sub-instance: rows [r0, r1) of G and h with their cone
    blocks (ZERO / NONNEG blocks cut to the range), full x-space."""
    from .linalg import SparseMatrix

    g = work.G._csr[r0:r1]
    specs, pos = [], 0
    for spec in work.dual_cones:
        a, b = pos, pos + spec.dim
        pos = b
        lo, hi = max(a, r0), min(b, r1)
        if hi <= lo:
            continue
        if spec.kind in (Cone.ZERO, Cone.NONNEG):
            specs.append(ConeSpec(spec.kind, hi - lo))
        else:
            if lo != a or hi != b:
                raise ValueError(f"row range [{r0}, {r1}) splits a {spec.kind.value} block")
            specs.append(spec)
    return ConicProblem(c=work.c, G=SparseMatrix.from_csr_arrays(g.indptr, g.indices, g.data,
                                                                 (r1 - r0, work.n)),
                        h=work.h[r0:r1], l=work.l, u=work.u, num_box=work.num_box,
                        primal_cones=work.primal_cones, dual_cones=tuple(specs))


# ---------------------------------------------------------------------------
# reductions of the check path
# ---------------------------------------------------------------------------

# y-space entries of pdcs_metrics / pdcs_rays / pdcs_gap_probe (the rest are
# x-space quantities, identical on every rank)
MET_Y_SUM = (N.MET_RV2, N.MET_YH, N.MET_H1, N.MET_YY, N.MET_NONFINITE)
MET_Y_MAX = (N.MET_RVMAX, N.MET_HMAX, N.MET_GXMAX, N.MET_RPMAX)
RAY_Y_SUM = (2,)
RAY_Y_MAX = (5,)
GAP_Y_SUM = (1, 3)


def combine(values: np.ndarray, sum_idx, max_idx, allreduce) -> np.ndarray:
    """Combine one rank's reductions with the others': y-space sums add,
    y-space maxima take the max, x-space entries are already global."""
    out = np.array(values, dtype=np.float64)
    if sum_idx:
        out[list(sum_idx)] = allreduce(out[list(sum_idx)], "sum")
    if max_idx:
        out[list(max_idx)] = allreduce(out[list(max_idx)], "max")
    return out


def torch_allreduce(group=None):
    """allreduce(numpy array, "sum"|"max") over a torch.distributed group."""
    import torch
    import torch.distributed as dist

    def run(arr, op):
        backend = dist.get_backend(group)
        dev = "cuda" if backend == "nccl" else "cpu"
        t = torch.as_tensor(np.ascontiguousarray(arr, dtype=np.float64), device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX, group=group)
        return t.cpu().numpy()

    return run


def combine_stats(stats: dict, allreduce) -> dict:
    """A rank's pdcs_stats over its row slice -> the whole instance's: the
    y-space norms of h add, the matrix maxima (max |G^_ij|, max row 1-norm)
    take the max, the x-space norms of c are already global."""
    out = dict(stats)
    s = allreduce(np.array([stats["h1"], stats["h2"]]), "sum")
    mx = allreduce(np.array([stats["gmax"], stats["rowsum_max"]]), "max")
    out["h1"], out["h2"] = float(s[0]), float(s[1])
    out["gmax"], out["rowsum_max"] = float(mx[0]), float(mx[1])
    return out


class ShardedDevice:
    """A rank's DeviceEngine whose reductions and G^T products are combined
    across ranks, so the single-GPU `_Loop` host logic runs unchanged."""

    def __init__(self, dev: DeviceEngine, allreduce, vec_allreduce, m_total: int):
        self._dev = dev
        self._ar = allreduce
        self._vec_ar = vec_allreduce
        self.m_total = m_total

    def __getattr__(self, name):
        return getattr(self._dev, name)

    # x-space state the device loop leaves stale outside each rank's slice
    X_STATE = ("x", "xh", "xb", "gty", "gth")

    def flush(self):
        """Apply the pending Halpern step, then give every rank full copies of
        the x-space state (each rank only stepped its x-slice)."""
        import ctypes

        self._dev.flush()
        bufs = [getattr(self._dev, nm) for nm in self.X_STATE]
        arr = (ctypes.c_void_p * len(bufs))(*[b.data_ptr() for b in bufs])
        N.check(self._dev.lib.pdcs_allgather_x(self._dev.handle, arr, len(bufs)), "pdcs_allgather_x")

    def spmv(self, transpose: bool, src, dst):
        self._dev.spmv(transpose, src, dst)
        if transpose:
            self._dev.stream.synchronize()
            self._vec_ar(dst[: self._dev.n])

    def metrics(self, mode, x, y, gx, gty):
        return combine(self._dev.metrics(mode, x, y, gx, gty), MET_Y_SUM, MET_Y_MAX, self._ar)

    def rays(self, x, y, gx, gty, xnorm, ynorm):
        return combine(self._dev.rays(x, y, gx, gty, xnorm, ynorm), RAY_Y_SUM, RAY_Y_MAX, self._ar)

    def gap_probe(self, x, y, gx, gty, t, tau, sigma):
        r = combine(np.array(self._dev.gap_probe(x, y, gx, gty, t, tau, sigma)), GAP_Y_SUM, (), self._ar)
        return float(r[0]), float(r[1]), float(r[2]), float(r[3])

    def gap_probes(self, x, y, gx, gty, ts, tau, sigma):
        r = np.array(self._dev.gap_probes(x, y, gx, gty, ts, tau, sigma)).reshape(-1)
        ysum = [4 * i + q for i in range(len(ts)) for q in GAP_Y_SUM]
        r = combine(r, ysum, (), self._ar)
        return [tuple(float(v) for v in r[4 * i:4 * i + 4]) for i in range(len(ts))]

    def dist2(self, space, a, b=None):
        v = self._dev.dist2(space, a, b)
        return float(self._ar(np.array([v]), "sum")[0]) if space == 1 else v

    def dot_diff(self, space, a, b, c, d):
        v = self._dev.dot_diff(space, a, b, c, d)
        return float(self._ar(np.array([v]), "sum")[0]) if space == 1 else v


def _make_sharded_loop_class():
    from .engine import _Loop

    class ShardedLoop(_Loop):
        """`_Loop` on a row slice with in-graph NCCL all-reduces."""

        def __init__(self, original, options, group=None):
            import torch.distributed as dist

            self._group = group
            self._rank = dist.get_rank(group)
            self._world = dist.get_world_size(group)
            super().__init__(original, options)

        def _make_device(self, options):
            import ctypes

            import torch
            import torch.distributed as dist

            work = self.work
            enabled = 1 if (options.use_preconditioner and work.G.nnz > 0) else 0
            r0, r1 = partition_rows(work, self._world)[self._rank]
            self.row_range = (r0, r1)
            local = slice_problem(work, r0, r1)
            # only the rank's row slice is uploaded (and transposed, and panelled)
            dev = DeviceEngine(local, allow_nonuniform_dual_soc=options.allow_nonuniform_dual_soc,
                               x_pad=self._world)
            # NCCL communicator of libpdcs (its collectives live in the graph and
            # in the sharded preconditioning)
            buf = [None]
            if self._rank == 0:
                idb = ctypes.create_string_buffer(128)
                N.check(dev.lib.pdcs_comm_unique_id(idb), "pdcs_comm_unique_id")
                buf = [bytes(idb.raw)]
            dist.broadcast_object_list(buf, src=0, group=self._group)
            N.check(dev.lib.pdcs_engine_set_comm(dev.handle, buf[0], self._rank, self._world),
                    "pdcs_engine_set_comm")
            self.xcuts = partition_cols(work, self._world)
            cuts = (ctypes.c_int32 * len(self.xcuts))(*self.xcuts)
            N.check(dev.lib.pdcs_engine_set_xsplit(dev.handle, cuts, self._world), "pdcs_engine_set_xsplit")
            # Ruiz + Pock-Chambolle on the slice: row statistics local, column
            # statistics all-reduced inside libpdcs (max / sum over the ranks)
            dev.precondition(enabled, options.ruiz_iterations, options.use_pock_chambolle)
            ar = torch_allreduce(self._group)
            stats = combine_stats(dev.stats(), ar)

            def vec_ar(t):
                # the engine stream is the current stream, so NCCL orders the
                # all-reduce after the engine's kernels that wrote `t` and the
                # engine's next kernels (metrics, rays, gap probes) after it
                with torch.cuda.stream(dev.stream):
                    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self._group)

            self.local_problem = local
            return ShardedDevice(dev, ar, vec_ar, work.m), stats

        def _elapsed(self):
            # every rank must take the same time-limit decisions
            return float(torch_allreduce(self._group)(np.array([super()._elapsed()]), "max")[0])

        def _next_stop(self, state):
            # batch ends must coincide: the graphs' collectives pair up trial by trial
            return _agree_min(self._group, super()._next_stop(state))

        def _gather_y(self, arr):
            import torch.distributed as dist

            parts = [None] * self._world
            dist.all_gather_object(parts, np.asarray(arr), group=self._group)
            return np.concatenate(parts)

        def _materialize(self, state):
            s = super()._materialize(state)

            def full(z):
                return None if z is None else type(z)(z.x, self._gather_y(z.y))

            s.z, s.z_anchor = full(s.z), full(s.z_anchor)
            s.z_prev_anchor, s.z_bar = full(s.z_prev_anchor), full(s.z_bar)
            return s

        def _assemble_y(self, y_w, slack_w):
            return self._gather_y(y_w), self._gather_y(slack_w)

    return ShardedLoop


def _agree_min(group, k: int) -> int:
    """The smallest batch end over the ranks (one scalar all-reduce; round 1
    pickled an all_gather_object here at every batch boundary)."""
    return int(-torch_allreduce(group)(np.array([-float(k)]), "max")[0])


_SHARDED = None


def sharded_loop_class():
    global _SHARDED
    if _SHARDED is None:
        _SHARDED = _make_sharded_loop_class()
    return _SHARDED


def solve_sharded(problem: ConicProblem, options=None, group=None):
    """solve() with G's rows sharded over the ranks of a torch.distributed
    group (one GPU per rank, torch.cuda.set_device already called).  Every
    rank returns the full SolveResult."""
    from .engine import SolverOptions, _adopt

    if options is None:
        options = SolverOptions()
    options.validate()
    if not isinstance(problem, ConicProblem):
        problem = _adopt(problem)
    loop = sharded_loop_class()(problem, options, group)
    try:
        return loop.run()
    finally:
        loop.close()
