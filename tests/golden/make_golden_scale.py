"""Benchmark-scale golden fixtures from the REFERENCE (conic_pdhg 0.1.0).

Run in the build container, where /root/reference exists (CPU only, ~30 min
on 8 cores; every solve pins BLAS to one thread):

    python tests/golden/make_golden_scale.py [case ...]

Cases (SURVEY.md 8(c) parity contract, VERDICT r1 "next round" item 1):

  c1_1e6, c1_1e4   full C1 (lp_random 2000 x 4000, 1%) to 1e-6 / 1e-4
  c2d_1e4          C2 at 1/10 (1,000 SOC(11) groups, q = 4,500) to 1e-4
  c4d_1e4          C4 at 1/10 (Markowitz RSOC, N = 50,000, k = 40) to 1e-4
  c3p_1e5, c2p_1e5 small primal-cone instances (exp / rescaled SOC) to 1e-5
  c3p_traj, c2p_traj  primal-cone instances at scale (100k primal exp blocks,
                   2,000 primal SOC(11) blocks): the reference's early iterates
  c3h_traj         C3 shape with 100k exponential-cone blocks: the reference's
                   early iterates (k = 5, 10, 20), every 5th coordinate
  c3_traj, c5_traj full-size C3 (1M exp blocks) / C5 (50M nnz): the
                   reference's iterates at k = 1, 2 (resp. 1..3), subsampled

For the whole solves the reference is also re-solved with 3 noise seeds: each
SpMV output is multiplied by (1 + 2.2e-16 N(0,1)) -- the survey's model of
GPU summation reordering -- and the [min, max] of the
iteration counts is stored as the reference's own round-off band.

Instances are not stored: the seeded generators in
paper_2603_15504_b200/instances.py rebuild them bit for bit (the fixture
keeps a checksum of G, c, h to prove it).  Solutions x, y are stored whole
for the solves, subsampled for the trajectories.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

from paper_2603_15504_b200 import instances  # noqa: E402

TIGHT6 = dict(rel_tol=1e-6, abs_tol=1e-6, time_limit=1e6)
TIGHT4 = dict(rel_tol=1e-4, abs_tol=1e-4, time_limit=1e6)

CASES = {
    "c1_1e6": (lambda: instances.lp_random(2000, 4000, 0.01, 0), TIGHT6, "solve"),
    "c1_1e4": (lambda: instances.lp_random(2000, 4000, 0.01, 0), TIGHT4, "solve"),
    "c2d_1e4": (lambda: instances.group_robust_regression(ngroups=1000, gsize=10, q=4500,
                                                         nnz_per_row=48, seed=2), TIGHT4, "solve"),
    "c4d_1e4": (lambda: instances.markowitz_rsoc(N=50_000, k=40, seed=4), TIGHT4, "solve"),
    # primal cone blocks: exp cones and non-uniformly
    # rescaled SOC blocks on the primal side, solved and traced
    "c3p_1e5": (lambda: instances.entropy_max_primal(nblk=60, p=8, nnz_per_col=2, seed=3),
                dict(rel_tol=1e-5, abs_tol=1e-5, time_limit=1e6), "solve"),
    "c2p_1e5": (lambda: instances.group_regression_primal(ngroups=20, gsize=5, q=60, nnz_per_row=10, seed=2),
                dict(rel_tol=1e-5, abs_tol=1e-5, time_limit=1e6), "solve"),
    "c3p_traj": (lambda: instances.entropy_max_primal(nblk=100_000, p=100, nnz_per_col=4, seed=3),
                 dict(max_iter=20, rel_tol=1e-14, abs_tol=1e-14, time_limit=1e6), "traj"),
    "c2p_traj": (lambda: instances.group_regression_primal(ngroups=2_000, gsize=10, q=9_000, nnz_per_row=48,
                                                           seed=2),
                 dict(max_iter=20, rel_tol=1e-14, abs_tol=1e-14, time_limit=1e6), "traj"),
    "c3h_traj": (lambda: instances.entropy_max(nblk=100_000, p=100, nnz_per_col=4, seed=3),
                 dict(max_iter=20, rel_tol=1e-14, abs_tol=1e-14, time_limit=1e6), "traj"),
    "c3_traj": (lambda: instances.entropy_max(), dict(max_iter=2, rel_tol=1e-14, abs_tol=1e-14,
                                                     time_limit=1e6), "traj"),
    "c5_traj": (lambda: instances.lp_large(), dict(max_iter=3, rel_tol=1e-14, abs_tol=1e-14,
                                                  time_limit=1e6), "traj"),
}
TRACE = {"c3h_traj": ((5, 10, 20), 5), "c3_traj": ((1, 2), 50), "c5_traj": ((1, 2, 3), 200),
         "c3p_traj": ((5, 10, 20), 5), "c2p_traj": ((5, 10, 20), 1)}
NOISE_SEEDS = (1, 2, 3)


def checksum(p) -> str:
    g = p.G.to_scipy()
    h = hashlib.sha256()
    for a in (g.indptr, g.indices, g.data, p.c, p.h, p.l, p.u):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def ref_solve(p, opts, noise_seed=None, trace_at=(), stride=1):
    import conic_pdhg as ref
    import conic_pdhg.engine as reng
    from conic_pdhg import linalg as rlin
    from make_golden import to_ref

    snaps = {}
    o = reng.SolverOptions(**opts)
    if trace_at:
        def cb(s):
            if s.k_bar in trace_at:
                snaps[s.k_bar] = (s.z.x[::stride].copy(), s.z.y[::stride].copy())

        o.iteration_callback = cb
    saved = (rlin.SparseMatrix.matvec, rlin.SparseMatrix.rmatvec)
    if noise_seed is not None:
        rng = np.random.default_rng(noise_seed)

        def noisy(f):
            def g(self, v):
                w = f(self, v)
                return w * (1.0 + 2.2e-16 * rng.standard_normal(w.shape))
            return g

        rlin.SparseMatrix.matvec = noisy(saved[0])
        rlin.SparseMatrix.rmatvec = noisy(saved[1])
    try:
        r = ref.solve(to_ref(p), o)
    finally:
        rlin.SparseMatrix.matvec, rlin.SparseMatrix.rmatvec = saved
    return r, snaps


def run_case(name: str) -> None:
    import time

    make, opts, kind = CASES[name]
    p = make()
    out = dict(opts_json=json.dumps(opts), checksum=checksum(p), numpy=np.__version__)
    import scipy

    out["scipy"] = scipy.__version__
    t0 = time.monotonic()
    if kind == "traj":
        kb, stride = TRACE[name]
        r, snaps = ref_solve(p, opts, trace_at=kb, stride=stride)
        out["stride"] = stride
        for k, (x, y) in snaps.items():
            out[f"trace_x_{k}"] = x
            out[f"trace_y_{k}"] = y
        out["iterations"] = r.iterations
    else:
        r, _ = ref_solve(p, opts)
        out.update(code=r.exit_code, status=r.exit_status, iterations=r.iterations, p_obj=r.p_obj,
                   d_obj=r.d_obj, restarts=r.restarts, x=r.x, y=r.y, wall_s=r.exit.wall_time_s)
        its, pobjs = [], []
        for s in NOISE_SEEDS:
            rn, _ = ref_solve(p, opts, noise_seed=s)
            its.append(rn.iterations)
            pobjs.append(rn.p_obj)
            assert rn.exit_status == r.exit_status, (name, s, rn.exit_status)
        out["noise_iterations"] = np.array(its)
        out["noise_p_obj"] = np.array(pobjs)
    np.savez_compressed(os.path.join(HERE, f"scale_{name}.npz"), **out)
    print(f"{name}: {out.get('status', 'traj')} iters={out['iterations']} "
          f"noise={list(out.get('noise_iterations', []))} {time.monotonic() - t0:.0f}s", flush=True)


def main():
    names = sys.argv[1:] or list(CASES)
    for n in names:
        run_case(n)


if __name__ == "__main__":
    main()
