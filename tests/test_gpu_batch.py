"""Batched multi-instance solves: one CUDA graph per
replay advances every instance (libpdcs pdcs_batch_run), each instance keeps
the reference's host loop.  Results must be bit-identical to sequential
`solve` calls -- status, iterations, restarts, x, y."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert a.exit_status == b.exit_status, (a.exit_status, b.exit_status)
    assert a.iterations == b.iterations and a.restarts == b.restarts
    np.testing.assert_array_equal(a.x, b.x)
    np.testing.assert_array_equal(a.y, b.y)
    assert a.p_obj == b.p_obj


def test_batched_matches_sequential_mixed_shapes():
    """LPs, SOCPs, exp-cone and RSOC instances of different sizes in one batch
    (different iteration counts, so members finish at different times), plus
    an instance that stops at the entry scan (zero objective, feasible 0)."""
    from golden_io import load, problem

    import paper_2603_15504_b200 as P
    from paper_2603_15504_b200 import instances
    from paper_2603_15504_b200.batch import solve_many

    probs = [instances.lp_random(150, 300, 0.05, s) for s in range(5)]
    probs += [instances.group_robust_regression(ngroups=20, gsize=5, q=60, nnz_per_row=10, seed=2),
              instances.entropy_max(nblk=40, p=8, nnz_per_col=2, seed=3),
              instances.markowitz_rsoc(N=60, k=5, seed=4),
              problem(load("solve_tiny"))]
    zero = instances.lp_random(50, 80, 0.1, 9)
    probs.append(type(zero)(c=np.zeros(zero.n), G=zero.G, h=-np.abs(zero.h) - 1.0, l=zero.l, u=zero.u,
                            num_box=zero.num_box, dual_cones=zero.dual_cones))
    opts = P.SolverOptions(rel_tol=1e-5, abs_tol=1e-5, max_iter=60_000)
    seq = [P.solve(p, opts) for p in probs]
    bat = solve_many(probs, opts)
    for a, b in zip(seq, bat):
        _same(a, b)
    assert seq[-1].iterations == 0  # the entry-scan member


def test_batched_many_c1_class_and_large_uploads():
    """64 C1-class instances, some larger than the 1 MB pinned-staging
    threshold, so concurrent setups stream through their per-thread staging
    buffers (shared staging raced)."""
    import paper_2603_15504_b200 as P
    from paper_2603_15504_b200 import instances
    from paper_2603_15504_b200.batch import solve_many

    probs = [instances.lp_random(400, 800, 0.02, s) for s in range(60)]
    probs += [instances.lp_large(m=60_000, n=120_000, nnz_per_row=5, eq_frac=0.3, seed=s) for s in range(4)]
    opts = P.SolverOptions(rel_tol=1e-4, abs_tol=1e-4, max_iter=4000)
    bat = solve_many(probs, opts)
    for i in (0, 17, 59, 60, 63):
        _same(P.solve(probs[i], opts), bat[i])


def test_threaded_solve_many_large_instances():
    """The thread-pool path with instances above the staging threshold."""
    import paper_2603_15504_b200 as P
    from paper_2603_15504_b200 import instances
    from paper_2603_15504_b200.batch import solve_many

    probs = [instances.lp_large(m=60_000, n=120_000, nnz_per_row=5, eq_frac=0.3, seed=s) for s in range(6)]
    opts = P.SolverOptions(rel_tol=1e-12, abs_tol=1e-12, max_iter=300)
    par = solve_many(probs, opts, batched=False, max_workers=6)
    for i in (0, 5):
        _same(P.solve(probs[i], opts), par[i])
