"""Benchmark-scale parity: the CUDA path against the REFERENCE's own outputs
at (or near) the BASELINE configurations (fixtures from
tests/golden/make_golden_scale.py, which imported /root/reference).

Whole solves (SURVEY.md 8(c) contract, no slack factors):
  * same exit status;
  * iterations inside the reference's own round-off band -- [min, max] over
    the nominal solve and 3 re-solves with 1-ulp SpMV noise -- widened by one
    check interval (2000);
  * objective: |p_gpu - p_ref| <= tol (1 + |p_ref|);
  * KKT triplet (rel_p_inf, rel_d_inf, rel_gap_term), recomputed by the
    oracle on both solutions: |e_gpu - e_ref| <= max(1e-6, tol).
Trajectories: the reference's early iterates (subsampled coordinates) on C3
with 100k exponential-cone blocks (the warm-started exp-cone Newton at scale),
on full C3 (1M blocks) and on full C5 (50M nnz), and on primal-cone instances
at scale: 100k primal exponential-cone blocks and 2,000 primal SOC(11)
blocks, whose non-uniform scaling makes every projection the rescaled-SOC
root search (Brent's method on the device).
"""

import json
import os

import numpy as np
import pytest

from oracle import pdcs_oracle as O

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    path = os.path.join(GOLDEN, f"scale_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"fixture {path} not generated")
    with np.load(path, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def _instance(name):
    import sys

    sys.path.insert(0, GOLDEN)
    from make_golden_scale import CASES, checksum  # generators only; no reference import

    p = CASES[name][0]()
    return p, checksum(p)


def _kkt(p, x, y):
    op = O.as_oproblem(p)
    work = O.rsoc_presolve(op)
    if work is not op:
        x, y, _ = O.rsoc_unrotate(op, x, y, np.zeros(op.m))
    rep = O.metrics(work, x, y)
    return np.array([rep["rel_p_inf"], rep["rel_d_inf"], rep["rel_gap_term"]])


@pytest.mark.parametrize("name", ["c1_1e6", "c1_1e4", "c2d_1e4", "c4d_1e4", "c3p_1e5", "c2p_1e5"])
def test_solve_matches_reference_at_scale(name):
    import paper_2603_15504_b200 as P

    d = _load(name)
    p, cs = _instance(name)
    assert cs == str(d["checksum"]), "generator does not rebuild the reference's instance"
    opts = json.loads(str(d["opts_json"]))
    r = P.solve(p, P.SolverOptions(**opts))
    assert r.exit_status == str(d["status"]), (name, r.exit_status, r.iterations)
    its = [int(d["iterations"])] + [int(v) for v in d["noise_iterations"]]
    lo, hi = min(its) - 2000, max(its) + 2000
    assert lo <= r.iterations <= hi, (name, r.iterations, its)
    tol = opts["rel_tol"]
    p_ref = float(d["p_obj"])
    assert abs(r.p_obj - p_ref) <= tol * (1.0 + abs(p_ref)), (name, r.p_obj, p_ref)
    e_gpu, e_ref = _kkt(p, r.x, r.y), _kkt(p, d["x"], d["y"])
    assert np.all(np.abs(e_gpu - e_ref) <= max(1e-6, tol)), (name, e_gpu, e_ref)
    assert np.all(e_gpu <= tol), (name, e_gpu)


@pytest.mark.parametrize("name,lim", [("c3h_traj", 1e-10), ("c3_traj", 1e-11), ("c5_traj", 1e-11),
                                      ("c3p_traj", 1e-10), ("c2p_traj", 1e-10)])
def test_trajectory_matches_reference_at_scale(name, lim):
    import paper_2603_15504_b200 as P

    d = _load(name)
    p, cs = _instance(name)
    assert cs == str(d["checksum"])
    opts = json.loads(str(d["opts_json"]))
    stride = int(d["stride"])
    kbars = sorted(int(k.split("_")[-1]) for k in d if k.startswith("trace_x_"))
    got = {}

    def cb(s):
        if s.k_bar in kbars:
            got[s.k_bar] = (s.z.x[::stride].copy(), s.z.y[::stride].copy())

    P.solve(p, P.SolverOptions(**opts, iteration_callback=cb))
    assert sorted(got) == kbars, (sorted(got), kbars)
    for k in kbars:
        for a, b in zip(got[k], (d[f"trace_x_{k}"], d[f"trace_y_{k}"])):
            scale = max(1.0, float(np.max(np.abs(b))))
            err = float(np.max(np.abs(a - b)))
            assert err <= lim * scale, (name, k, err)
