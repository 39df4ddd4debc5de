"""Synthetic instances of the five benchmark shapes.

All generators are seeded and return a `ConicProblem`; sizes are parameters
so tests can build small versions of the same structure.  The full-size
configurations are:

  C1 lp_random(2000, 4000, 0.01)          LP, NONNEG rows, box [-2, 2]
  C2 group_robust_regression(10_000)      SOCP, 10k SOC(11) blocks, free vars
  C3 entropy_max(1_000_000)               1M exponential-cone blocks
  C4 markowitz_rsoc(500_000, 40)          one rotated SOC of dim 500,042
  C5 lp_large(10_000_000, 20_000_000)     50M-nnz LP, ZERO + NONNEG rows
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .linalg import SparseMatrix
from .model import Cone, ConeSpec, ConicProblem


def _canon(rows_or_indptr, cols, vals, shape, csr_direct=False):
    if csr_direct:
        g = sp.csr_matrix((vals, cols, rows_or_indptr), shape=shape)
    else:
        g = sp.coo_matrix((vals, (rows_or_indptr, cols)), shape=shape).tocsr()
    g.sum_duplicates()
    g.sort_indices()
    return SparseMatrix.from_csr_arrays(g.indptr, g.indices, g.data, shape)


def lp_random(m=2000, n=4000, density=0.01, seed=0) -> ConicProblem:
    """G1/C1: random sparse LP, feasible by construction (make_box_lp pattern)."""
    rng = np.random.default_rng(seed)
    G = sp.random(m, n, density, format="csr", random_state=rng, data_rvs=rng.standard_normal)
    x0 = rng.uniform(-1.0, 1.0, n)
    h = G @ x0 - rng.uniform(0.1, 1.0, m)
    c = rng.standard_normal(n)
    return ConicProblem(c=c, G=SparseMatrix(G), h=h, l=-2.0 * np.ones(n), u=2.0 * np.ones(n),
                        num_box=n, dual_cones=(ConeSpec(Cone.NONNEG, m),))


def group_robust_regression(ngroups=10_000, gsize=10, q=45_000, nnz_per_row=48, lam=0.1,
                            seed=2) -> ConicProblem:
    """G2/C2: sum_g ||A_g x - b_g|| + lam ||x||_1 as an SOCP.

    Variables [x (q), s (q), t (ngroups)], all free.  Rows: NONNEG(2q) for
    s >= |x| ([-I I 0; I I 0], h = 0), then per group SOC(gsize+1) with rows
    [t_g; A_g x] and h = [0; b_g]."""
    rng = np.random.default_rng(seed)
    na = ngroups * gsize
    A = sp.random(na, q, min(1.0, nnz_per_row / q), format="csr", random_state=rng,
                  data_rvs=rng.standard_normal)
    x_true = rng.standard_normal(q) * (rng.random(q) < 0.1)
    b = A @ x_true + 0.1 * rng.standard_normal(na)
    n = 2 * q + ngroups
    eye = np.arange(q)
    rows = [eye, eye, q + eye, q + eye]
    cols = [eye, q + eye, eye, q + eye]
    vals = [-np.ones(q), np.ones(q), np.ones(q), np.ones(q)]
    # SOC block g occupies rows 2q + g*(gsize+1) .. ; first row is t_g
    base = 2 * q + np.arange(ngroups) * (gsize + 1)
    rows.append(base)
    cols.append(2 * q + np.arange(ngroups))
    vals.append(np.ones(ngroups))
    ac = A.tocoo()
    arow = ac.row // gsize
    rows.append(base[arow] + 1 + ac.row % gsize)
    cols.append(ac.col)
    vals.append(ac.data)
    m = 2 * q + ngroups * (gsize + 1)
    G = _canon(np.concatenate(rows), np.concatenate(cols), np.concatenate(vals), (m, n))
    h = np.zeros(m)
    bidx = np.arange(na)
    h[base[bidx // gsize] + 1 + bidx % gsize] = b
    c = np.concatenate([np.zeros(q), lam * np.ones(q), np.ones(ngroups)])
    dual = (ConeSpec(Cone.NONNEG, 2 * q),) + tuple(ConeSpec(Cone.SOC, gsize + 1) for _ in range(ngroups))
    return ConicProblem(c=c, G=G, h=h, l=-np.inf * np.ones(n), u=np.inf * np.ones(n), num_box=n,
                        dual_cones=dual)


def entropy_max(nblk=1_000_000, p=1_000, nnz_per_col=4, seed=3) -> ConicProblem:
    """G3/C3: max sum_i -x_i log x_i  s.t.  A x = b, via (t_i, x_i, 1) in K_exp.

    Variables [x (nblk), t (nblk)] free.  Rows: ZERO(p) [A 0] with h = b, then
    per block an EXP block with rows (t_i, x_i, 0) and h = (0, 0, -1)."""
    rng = np.random.default_rng(seed)
    arows = rng.integers(0, p, size=(nblk, nnz_per_col))
    avals = rng.uniform(0.5, 1.5, size=(nblk, nnz_per_col))
    acols = np.repeat(np.arange(nblk), nnz_per_col)
    x0 = rng.uniform(0.1, 1.0, nblk)
    A = sp.coo_matrix((avals.ravel(), (arows.ravel(), acols)), shape=(p, nblk)).tocsr()
    A.sum_duplicates()
    b = A @ x0
    n, m = 2 * nblk, p + 3 * nblk
    ac = A.tocoo()
    blk = p + 3 * np.arange(nblk)
    rows = np.concatenate([ac.row, blk, blk + 1])
    cols = np.concatenate([ac.col, nblk + np.arange(nblk), np.arange(nblk)])
    vals = np.concatenate([ac.data, np.ones(nblk), np.ones(nblk)])
    G = _canon(rows, cols, vals, (m, n))
    h = np.zeros(m)
    h[:p] = b
    h[blk + 2] = -1.0
    c = np.concatenate([np.zeros(nblk), -np.ones(nblk)])
    dual = (ConeSpec(Cone.ZERO, p),) + tuple(ConeSpec(Cone.EXP, 3) for _ in range(nblk))
    return ConicProblem(c=c, G=G, h=h, l=-np.inf * np.ones(n), u=np.inf * np.ones(n), num_box=n,
                        dual_cones=dual)


def markowitz_rsoc(N=500_000, k=40, gamma=1.0, seed=4) -> ConicProblem:
    """G4/C4: min -mu'x + gamma s  s.t.  1'x = 1, F'x = f, 2 s (1/2) >= ||f||^2 + ||D^1/2 x||^2.

    Variables [x in [0,1]^N, f free (k), s free].  Rows: ZERO(1+k) then one
    RSOC(2+k+N) with rows (s, 0, f, diag(sqrt d) x) and h = (0, -1/2, 0, 0)."""
    rng = np.random.default_rng(seed)
    F = rng.standard_normal((N, k)) / np.sqrt(k)
    d = rng.uniform(0.01, 0.1, N)
    mu = rng.normal(0.05, 0.02, N)
    n = N + k + 1
    m = 1 + k + 2 + k + N
    xs = np.arange(N)
    rows = [np.zeros(N, dtype=np.int64)]
    cols = [xs]
    vals = [np.ones(N)]
    # F' x - f = 0  (rows 1..k)
    rows.append(np.repeat(np.arange(1, k + 1), N))
    cols.append(np.tile(xs, k))
    vals.append(F.T.ravel())
    rows.append(np.arange(1, k + 1))
    cols.append(N + np.arange(k))
    vals.append(-np.ones(k))
    r0 = 1 + k  # RSOC block start: p = s, q = constant row, w = (f, D^1/2 x)
    rows.append(np.array([r0]))
    cols.append(np.array([N + k]))
    vals.append(np.ones(1))
    rows.append(r0 + 2 + np.arange(k))
    cols.append(N + np.arange(k))
    vals.append(np.ones(k))
    rows.append(r0 + 2 + k + xs)
    cols.append(xs)
    vals.append(np.sqrt(d))
    G = _canon(np.concatenate(rows), np.concatenate(cols), np.concatenate(vals), (m, n))
    h = np.zeros(m)
    h[0] = 1.0
    h[r0 + 1] = -0.5
    c = np.concatenate([-mu, np.zeros(k), [gamma]])
    l = np.concatenate([np.zeros(N), -np.inf * np.ones(k + 1)])
    u = np.concatenate([np.ones(N), np.inf * np.ones(k + 1)])
    dual = (ConeSpec(Cone.ZERO, 1 + k), ConeSpec(Cone.RSOC, 2 + k + N))
    return ConicProblem(c=c, G=G, h=h, l=l, u=u, num_box=n, dual_cones=dual)


def lp_large(m=10_000_000, n=20_000_000, nnz_per_row=5, eq_frac=0.3, seed=5) -> ConicProblem:
    """G5/C5: exactly nnz_per_row uniformly random columns per row (duplicates
    summed), N(0,1) values; the first eq_frac rows ZERO with h = G x0, the
    rest NONNEG with h = G x0 - U(0.1, 1); c ~ N(0,1); box [-2, 2]."""
    rng = np.random.default_rng(seed)
    cols = rng.integers(0, n, size=m * nnz_per_row, dtype=np.int64).astype(np.int32)
    vals = rng.standard_normal(m * nnz_per_row)
    indptr = np.arange(0, m * nnz_per_row + 1, nnz_per_row, dtype=np.int64)
    G = sp.csr_matrix((vals, cols, indptr), shape=(m, n))
    G.sum_duplicates()  # sorts each row and merges repeated columns
    x0 = rng.uniform(-1.0, 1.0, n)
    gx0 = G @ x0
    m_eq = int(eq_frac * m)
    h = gx0.copy()
    h[m_eq:] -= rng.uniform(0.1, 1.0, m - m_eq)
    c = rng.standard_normal(n)
    dual = (ConeSpec(Cone.ZERO, m_eq), ConeSpec(Cone.NONNEG, m - m_eq))
    Gm = SparseMatrix.from_csr_arrays(G.indptr, G.indices, G.data, (m, n))
    return ConicProblem(c=c, G=Gm, h=h, l=-2.0 * np.ones(n), u=2.0 * np.ones(n), num_box=n,
                        dual_cones=dual)


def lp_planted(m=10_000_000, n=20_000_000, nnz_per_row=5, eq_frac=0.3, seed=5) -> ConicProblem:
    """The C5 pattern (exactly nnz_per_row uniformly random columns per row,
    N(0,1) values, first eq_frac rows ZERO, the rest NONNEG, box [-2, 2]) with
    a planted strictly complementary optimum (x*, y*, lambda*):
    x* is at -2 / +2 / interior U(-1.5, 1.5) with probabilities 3/8, 3/8, 1/4;
    y* is N(0,1) on ZERO rows, U(0.1, 1) on half the NONNEG rows (active,
    zero slack) and 0 on the rest (slack U(0.1, 1));
    h = G x* - slack, c = G^T y* + lambda* with lambda* = +-U(0.1, 1) at the
    lower / upper bounds and 0 inside.  The instance is feasible and bounded
    with a known optimal value c'x*, so time-to-tolerance is well defined."""
    rng = np.random.default_rng(seed)
    cols = rng.integers(0, n, size=m * nnz_per_row, dtype=np.int64).astype(np.int32)
    vals = rng.standard_normal(m * nnz_per_row)
    indptr = np.arange(0, m * nnz_per_row + 1, nnz_per_row, dtype=np.int64)
    G = sp.csr_matrix((vals, cols, indptr), shape=(m, n))
    G.sum_duplicates()
    state = rng.choice(3, size=n, p=[0.375, 0.375, 0.25])
    xs = np.where(state == 0, -2.0, np.where(state == 1, 2.0, rng.uniform(-1.5, 1.5, n)))
    lam = np.where(state == 0, rng.uniform(0.1, 1.0, n), np.where(state == 1, -rng.uniform(0.1, 1.0, n), 0.0))
    m_eq = int(eq_frac * m)
    active = rng.random(m - m_eq) < 0.5
    ys = np.concatenate([rng.standard_normal(m_eq), np.where(active, rng.uniform(0.1, 1.0, m - m_eq), 0.0)])
    slack = np.concatenate([np.zeros(m_eq), np.where(active, 0.0, rng.uniform(0.1, 1.0, m - m_eq))])
    h = G @ xs - slack
    c = G.T @ ys + lam
    dual = (ConeSpec(Cone.ZERO, m_eq), ConeSpec(Cone.NONNEG, m - m_eq))
    Gm = SparseMatrix.from_csr_arrays(G.indptr, G.indices, G.data, (m, n))
    return ConicProblem(c=c, G=Gm, h=h, l=-2.0 * np.ones(n), u=2.0 * np.ones(n), num_box=n,
                        dual_cones=dual)


def entropy_max_primal(nblk=1_000_000, p=1_000, nnz_per_col=4, seed=3) -> ConicProblem:
    """C3's entropy maximisation with the exponential cones on the PRIMAL side
    (primal cone blocks at scale): variables per block
    (t_i, x_i, s_i) in K_exp (s >= x e^{t/x}); ZERO rows A x = b and s_i = 1;
    minimise -sum t_i, i.e. maximise sum -x_i log x_i.  num_box = 0."""
    rng = np.random.default_rng(seed)
    arows = rng.integers(0, p, size=(nblk, nnz_per_col))
    avals = rng.uniform(0.5, 1.5, size=(nblk, nnz_per_col))
    acols = np.repeat(np.arange(nblk), nnz_per_col)
    x0 = rng.uniform(0.1, 1.0, nblk)
    A = sp.coo_matrix((avals.ravel(), (arows.ravel(), acols)), shape=(p, nblk)).tocsr()
    A.sum_duplicates()
    b = A @ x0
    n, m = 3 * nblk, p + nblk
    ac = A.tocoo()
    rows = np.concatenate([ac.row, p + np.arange(nblk)])
    cols = np.concatenate([3 * ac.col + 1, 3 * np.arange(nblk) + 2])
    vals = np.concatenate([ac.data, np.ones(nblk)])
    G = _canon(rows, cols, vals, (m, n))
    h = np.concatenate([b, np.ones(nblk)])
    c = np.zeros(n)
    c[0::3] = -1.0
    return ConicProblem(c=c, G=G, h=h, l=np.zeros(0), u=np.zeros(0), num_box=0,
                        primal_cones=tuple(ConeSpec(Cone.EXP, 3) for _ in range(nblk)),
                        dual_cones=(ConeSpec(Cone.ZERO, m),))


def group_regression_primal(ngroups=10_000, gsize=10, q=45_000, nnz_per_row=48, seed=2) -> ConicProblem:
    """C2's group robust regression with the second-order cones on the PRIMAL
    side: variables [x (q, free box), then per group (t_g, r_g) in SOC(gsize+1)];
    ZERO rows A_g x + r_g = b_g; minimise sum t_g.  After Ruiz scaling the
    primal SOC blocks are non-uniformly scaled, so every projection is the
    rescaled-SOC root search (cones.py:353-429) -- at scale."""
    rng = np.random.default_rng(seed)
    na = ngroups * gsize
    A = sp.random(na, q, min(1.0, nnz_per_row / q), format="csr", random_state=rng,
                  data_rvs=rng.standard_normal)
    x_true = rng.standard_normal(q) * (rng.random(q) < 0.1)
    bvec = A @ x_true + 0.1 * rng.standard_normal(na)
    blk = gsize + 1
    n = q + ngroups * blk
    ac = A.tocoo()
    gi, ri = ac.row // gsize, ac.row % gsize
    # residual variable of row a: r_{g, i} at x-space index q + g*blk + 1 + i
    rvar = q + np.arange(na) // gsize * blk + 1 + np.arange(na) % gsize
    rows = np.concatenate([ac.row, np.arange(na)])
    cols = np.concatenate([ac.col, rvar])
    vals = np.concatenate([ac.data, np.ones(na)])
    del gi, ri
    G = _canon(rows, cols, vals, (na, n))
    c = np.zeros(n)
    c[q + np.arange(ngroups) * blk] = 1.0
    return ConicProblem(c=c, G=G, h=bvec, l=-np.inf * np.ones(q), u=np.inf * np.ones(q), num_box=q,
                        primal_cones=tuple(ConeSpec(Cone.SOC, blk) for _ in range(ngroups)),
                        dual_cones=(ConeSpec(Cone.ZERO, na),))


CONFIGS = {
    "C1": lambda: lp_random(2000, 4000, 0.01, 0),
    "C2": lambda: group_robust_regression(),
    "C3": lambda: entropy_max(),
    "C4": lambda: markowitz_rsoc(),
    "C5": lambda: lp_large(),
}


def algorithmic_bytes(problem: ConicProblem) -> int:
    """B_alg per PDHG iteration:
    24 nnz + 4(m+1) + 4(n+1) + 8 (13 n + 2 n_b + 13 m), n_b = box coordinates
    with at least one finite bound."""
    n, m, nnz = problem.n, problem.m, problem.G.nnz
    nb = int(np.sum(np.isfinite(problem.l) | np.isfinite(problem.u)))
    return 24 * nnz + 4 * (m + 1) + 4 * (n + 1) + 8 * (13 * n + 2 * nb + 13 * m)
