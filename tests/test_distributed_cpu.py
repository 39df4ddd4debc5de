"""Multi-rank (gloo, world_size 2-3) CPU tests of the row-sharded design:
the partitioner cuts only at cone-block boundaries and balances nonzeros,
and the sharded iteration with the all-reduce plan of the CUDA graph
reproduces the single-process oracle iterate for iterate."""

import functools
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from dist_emulation import sharded_run
from oracle import pdcs_oracle as O
from paper_2603_15504_b200 import instances
from paper_2603_15504_b200.distributed import (
    GAP_Y_SUM, MET_Y_MAX, MET_Y_SUM, allowed_cuts, allowed_xcuts, combine, partition_cols,
    partition_rows, slice_problem)
from paper_2603_15504_b200.model import Cone, rsoc_to_soc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _prim():
    from golden_io import load, problem

    return problem(load("solve_prim"))


PROBLEMS = {
    "prim": _prim,
    "lp": functools.partial(instances.lp_large, m=600, n=1200, nnz_per_row=5, eq_frac=0.3, seed=5),
    "socp": functools.partial(instances.group_robust_regression, ngroups=30, gsize=5, q=80,
                              nnz_per_row=10, seed=2),
    "exp": functools.partial(instances.entropy_max, nblk=60, p=10, nnz_per_col=2, seed=3),
    "rsoc": functools.partial(instances.markowitz_rsoc, N=80, k=4, seed=4),
}


@pytest.mark.parametrize("name", sorted(PROBLEMS))
@pytest.mark.parametrize("world", [2, 3, 5])
def test_partition_cuts_only_at_block_boundaries(name, world):
    work = rsoc_to_soc(PROBLEMS[name]())
    parts = partition_rows(work, world)
    assert parts[0][0] == 0 and parts[-1][1] == work.m
    assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
    cuts = set(allowed_cuts(work).tolist())
    for r0, r1 in parts:
        assert r0 in cuts and r1 in cuts
        sub = slice_problem(work, r0, r1)  # raises if a cone block were split
        assert sub.m == r1 - r0 and sub.n == work.n
    if name == "lp":  # elementwise rows: nnz balanced within a few rows
        nnz = [work.G._csr[r0:r1].nnz for r0, r1 in parts]
        assert max(nnz) - min(nnz) <= 20


@pytest.mark.parametrize("name", sorted(PROBLEMS))
@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_xsplit_cuts_only_at_primal_block_boundaries(name, world):
    work = rsoc_to_soc(PROBLEMS[name]())
    cuts = partition_cols(work, world)
    assert len(cuts) == world + 1 and cuts[0] == 0 and cuts[-1] == work.n
    assert all(a <= b for a, b in zip(cuts, cuts[1:]))
    assert set(cuts) <= set(allowed_xcuts(work).tolist())
    if not work.primal_cones:  # equal slices: the engine's all-gather / reduce-scatter path
        cnt = -(-work.n // world)
        assert cuts == [min(r * cnt, work.n) for r in range(world + 1)]


def test_slices_reassemble_the_matrix():
    work = rsoc_to_soc(PROBLEMS["socp"]())
    parts = partition_rows(work, 3)
    import scipy.sparse as sp

    G = sp.vstack([slice_problem(work, r0, r1).G._csr for r0, r1 in parts]).toarray()
    np.testing.assert_array_equal(G, work.G.toarray())
    kinds = [s.kind for r0, r1 in parts for s in slice_problem(work, r0, r1).dual_cones]
    assert kinds.count(Cone.SOC) == 30


def test_combine_plan():
    """y-space entries are summed / maxed across ranks, x-space ones kept."""
    from paper_2603_15504_b200 import _native as N

    ranks = [np.arange(N.NMET, dtype=float) + 100 * r for r in range(2)]

    def fake_allreduce(vals_by_rank):
        def run(arr, op):
            idx = run.idx[op]
            stack = np.array([v[idx] for v in vals_by_rank])
            return stack.sum(0) if op == "sum" else stack.max(0)
        return run

    ar = fake_allreduce(ranks)
    ar.idx = {"sum": list(MET_Y_SUM), "max": list(MET_Y_MAX)}
    out = combine(ranks[0], MET_Y_SUM, MET_Y_MAX, ar)
    for i in range(N.NMET):
        if i in MET_Y_SUM:
            assert out[i] == ranks[0][i] + ranks[1][i]
        elif i in MET_Y_MAX:
            assert out[i] == max(ranks[0][i], ranks[1][i])
        else:
            assert out[i] == ranks[0][i]
    assert GAP_Y_SUM == (1, 3)


@pytest.mark.parametrize("name,world", [("lp", 2), ("socp", 2), ("exp", 3), ("rsoc", 2), ("prim", 3)])
def test_sharded_iterations_match_single_process_oracle(tmp_path, name, world):
    iters = 40
    out = str(tmp_path / "sharded.npz")
    mp.start_processes(sharded_run, args=(world, PROBLEMS[name], iters, _free_port(), out),
                       nprocs=world, join=True, start_method="spawn")
    got = np.load(out)
    snap = {}

    class Done(Exception):
        pass

    def cb(st, loop):
        if st.k == iters:
            snap["x"], snap["y"], snap["k_bar"] = st.x.copy(), st.y.copy(), st.k_bar
            raise Done

    with pytest.raises(Done):
        O.solve(PROBLEMS[name](), O.options_from(None, use_adaptive_restart=False, max_iter=10**6,
                                                  rel_tol=1e-300, abs_tol=1e-300), callback=cb)
    assert int(got["k_bar"]) == snap["k_bar"]
    for key in ("x", "y"):
        scale = max(1.0, float(np.max(np.abs(snap[key]))))
        assert np.max(np.abs(got[key] - snap[key])) <= 1e-9 * scale, key


@pytest.mark.parametrize("name,world", [("lp", 2), ("socp", 3), ("exp", 2), ("rsoc", 2), ("prim", 2)])
def test_sharded_restarts_match_single_process_oracle(tmp_path, name, world):
    """Restarts on (checks every 10 k_bar): the products are refreshed and the
    restart candidate is chosen by the normalized duality gap with every dot
    product combined across the ranks, then the restart criteria and the
    primal-weight update run on the combined scalars -- the same iterates,
    k_bar and restart count as the single-process oracle."""
    iters, freq = 45, 10
    out = str(tmp_path / "sharded_rs.npz")
    mp.start_processes(sharded_run, args=(world, PROBLEMS[name], iters, _free_port(), out, freq),
                       nprocs=world, join=True, start_method="spawn")
    got = np.load(out)
    kb = int(got["k_bar"])
    assert kb % freq != 0  # the snapshot below is taken before any check at kb
    snap = {}

    def cb(st, loop):
        if st.k_bar == kb:
            snap["x"], snap["y"], snap["restarts"] = st.x.copy(), st.y.copy(), loop.restarts

    o = O.options_from(None, duality_gap_restart_freq=freq, max_iter=kb, rel_tol=1e-300, abs_tol=1e-300)
    O.solve(PROBLEMS[name](), o, callback=cb)
    assert "x" in snap, "the oracle never reached the emulation's k_bar"
    assert int(got["restarts"]) == snap["restarts"] >= 1, (int(got["restarts"]), snap["restarts"])
    for key in ("x", "y"):
        scale = max(1.0, float(np.max(np.abs(snap[key]))))
        assert np.max(np.abs(got[key] - snap[key])) <= 1e-9 * scale, key
