"""Generate golden fixtures from the REFERENCE implementation (conic_pdhg 0.1.0).

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

It imports the reference from /root/reference/pkg/src, builds small seeded
instances of every benchmark shape plus the reference tests' hand instances,
and stores inputs and reference outputs as .npz files next to this script.
The GPU box has no /root/reference; tests there compare against these files
and against oracle/pdcs_oracle.py (which is itself pinned to these files).
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import conic_pdhg as ref  # noqa: E402
import conic_pdhg.cones as rcones  # noqa: E402
import conic_pdhg.engine as reng  # noqa: E402
import conic_pdhg.restart as rrestart  # noqa: E402
import conic_pdhg.scaling as rscaling  # noqa: E402
import conic_pdhg.termination as rterm  # noqa: E402
from conic_pdhg.linalg import SparseMatrix as RSparse  # noqa: E402
from conic_pdhg.model import Cone as RCone, ConeSpec as RSpec, ConicProblem as RProblem  # noqa: E402

from paper_2603_15504_b200 import instances  # noqa: E402  (pure host generators)

OPT_KEYS = ("rel_tol", "abs_tol", "max_iter", "duality_gap_restart_freq", "use_preconditioner",
            "method", "use_adaptive_restart", "use_adaptive_step_size_weight", "use_kkt_restart",
            "kkt_restart_freq", "fixed_reflection_beta", "initial_step_norm")


def to_ref(p) -> RProblem:
    def specs(seq):
        return tuple(RSpec(RCone(s.kind.value), s.dim) for s in seq)

    return RProblem(c=p.c, G=RSparse(p.G.to_scipy()), h=p.h, l=p.l, u=p.u, num_box=p.num_box,
                    primal_cones=specs(p.primal_cones), dual_cones=specs(p.dual_cones))


def dense_problem(c, G, h, l, u, nbox, dual, primal=()):
    from paper_2603_15504_b200.linalg import SparseMatrix
    from paper_2603_15504_b200.model import Cone, ConeSpec, ConicProblem

    return ConicProblem(c=np.asarray(c, float), G=SparseMatrix(np.asarray(G, float)),
                        h=np.asarray(h, float), l=np.asarray(l, float), u=np.asarray(u, float),
                        num_box=nbox, primal_cones=tuple(ConeSpec(Cone(k), d) for k, d in primal),
                        dual_cones=tuple(ConeSpec(Cone(k), d) for k, d in dual))


def problem_arrays(p) -> dict:
    g = p.G.to_scipy()
    return dict(c=p.c, h=p.h, l=p.l, u=p.u, num_box=p.num_box, shape=np.array(g.shape),
                indptr=g.indptr, indices=g.indices, data=g.data,
                pkinds=json.dumps([s.kind.value for s in p.primal_cones]),
                pdims=np.array([s.dim for s in p.primal_cones], dtype=np.int64),
                dkinds=json.dumps([s.kind.value for s in p.dual_cones]),
                ddims=np.array([s.dim for s in p.dual_cones], dtype=np.int64))


def solve_case(name, p, opts: dict, trace_at=(10, 20, 50)):
    o = reng.SolverOptions(**opts)
    snaps = {}

    def cb(s):
        if s.k_bar in trace_at:
            snaps[s.k_bar] = (s.z.x.copy(), s.z.y.copy())

    o.iteration_callback = cb
    r = ref.solve(to_ref(p), o)
    out = problem_arrays(p)
    out.update(opts_json=json.dumps(opts), code=r.exit_code, status=r.exit_status,
               iterations=r.iterations, p_obj=r.p_obj, d_obj=r.d_obj, restarts=r.restarts,
               x=r.x, y=r.y, lam=r.lam, slack=r.slack)
    for kb, (x, y) in snaps.items():
        out[f"trace_x_{kb}"] = x
        out[f"trace_y_{kb}"] = y
    np.savez_compressed(os.path.join(HERE, f"solve_{name}.npz"), **out)
    print(f"{name}: {r.exit_status} iters={r.iterations} restarts={r.restarts} pobj={r.p_obj:.10e}")


def hand_instances():
    tiny = dense_problem([-1.0, -1.0], [[1.0, 1.0]], [0.5], [0.0, 0.0], [1.0, 1.0], 2, [("nonneg", 1)])
    G = np.zeros((3, 2)); G[1, 0] = 1.0; G[2, 1] = 1.0
    ball = dense_problem([1.0, 0.0], G, [-1.0, 0.0, 0.0], [-5.0, -5.0], [5.0, 5.0], 2, [("soc", 3)])
    G = np.zeros((3, 1)); G[2, 0] = 1.0
    expc = dense_problem([1.0], G, [-1.0, -1.0, 0.0], [-math.inf], [math.inf], 1, [("exp", 3)])
    dexp = dense_problem([1.0], G, [1.0, -1.0, 0.0], [-math.inf], [math.inf], 1, [("dual_exp", 3)])
    G = np.zeros((3, 2)); G[0, 0] = 1.0; G[1, 1] = 1.0
    rsoc = dense_problem([1.0, 1.0], G, [0.0, 0.0, -1.0], [-10.0, -10.0], [10.0, 10.0], 2, [("rsoc", 3)])
    # primal cones: x = (b, s0, s1, s2, e0, e1, e2) with s in SOC, e in EXP
    rng = np.random.default_rng(77)
    Gp = rng.standard_normal((4, 7))
    xfeas = np.array([0.2, 2.0, 0.5, -0.7, -1.0, 1.0, 2.0])
    hp = Gp @ xfeas - rng.uniform(0.1, 0.5, 4)
    prim = dense_problem([1.0, 1.0, 0.3, -0.2, 0.1, 0.2, 1.0], Gp, hp, [-3.0], [3.0], 1, [("nonneg", 4)],
                         primal=[("soc", 3), ("exp", 3)])
    infeas = dense_problem([1.0, 1.0], [[1.0, 1.0]], [3.0], [0.0, 0.0], [1.0, 1.0], 2, [("nonneg", 1)])
    unbnd = dense_problem([-1.0, 0.0], [[1.0, -1.0]], [0.0], [-math.inf, 0.0], [math.inf, 1.0], 2,
                          [("nonneg", 1)])
    return dict(tiny=tiny, ball=ball, expc=expc, dexp=dexp, rsoc=rsoc, prim=prim, infeas=infeas,
                unbnd=unbnd)


def small_benchmarks():
    return dict(
        c1s=instances.lp_random(200, 400, 0.05, 0),
        c2s=instances.group_robust_regression(ngroups=20, gsize=5, q=60, nnz_per_row=10, seed=2),
        c3s=instances.entropy_max(nblk=40, p=8, nnz_per_col=2, seed=3),
        c4s=instances.markowitz_rsoc(N=60, k=5, seed=4),
        c5s=instances.lp_large(m=300, n=600, nnz_per_row=5, eq_frac=0.3, seed=5),
    )


def projection_vectors():
    rng = np.random.default_rng(1)
    out = {}
    pts = rng.uniform(-5.0, 5.0, (300, 3))
    out["exp_in"] = pts
    out["exp_out"] = np.array([rcones.project_exp(v) for v in pts])
    out["dexp_out"] = np.array([rcones.project_dual_exp(v) for v in pts])
    # stiff exponential-cone points (large / tiny magnitudes)
    stiff = np.concatenate([rng.standard_normal((100, 3)) * 1e3, rng.standard_normal((100, 3)) * 1e-3,
                            rng.standard_normal((100, 3)) * np.array([30.0, 0.1, 1.0])])
    out["exp_stiff_in"] = stiff
    out["exp_stiff_out"] = np.array([rcones.project_exp(v) for v in stiff])
    socs = [rng.standard_normal(int(rng.integers(2, 40))) * 3.0 for _ in range(200)]
    out["soc_len"] = np.array([len(v) for v in socs])
    out["soc_in"] = np.concatenate(socs)
    out["soc_out"] = np.concatenate([rcones.project_soc(v) for v in socs])
    rs_in, rs_sc, rs_out = [], [], []
    for _ in range(200):
        d = int(rng.integers(2, 30))
        v = rng.standard_normal(d) * 3.0
        s = rng.uniform(0.1, 10.0, d)
        rs_in.append(v)
        rs_sc.append(s)
        rs_out.append(rcones.project_rescaled_soc(v, s))
    out["rsoc_len"] = np.array([len(v) for v in rs_in])
    out["rsoc_in"] = np.concatenate(rs_in)
    out["rsoc_scale"] = np.concatenate(rs_sc)
    out["rsoc_out"] = np.concatenate(rs_out)
    np.savez_compressed(os.path.join(HERE, "projections.npz"), **out)


def component_vectors(bench):
    """Scaling vectors, compute_errors, line search and gap values."""
    out = {}
    for name, p in bench.items():
        from conic_pdhg.model import rsoc_to_soc

        work = rsoc_to_soc(to_ref(p))
        s = rscaling.build_scaling(work)
        out[f"{name}_d1"] = s.d1
        out[f"{name}_d2"] = s.d2
        sc = rscaling.rescale_problem(work, s)
        rng = np.random.default_rng(5)
        x = rng.standard_normal(sc.n)
        y = rng.standard_normal(sc.m)
        rep = rterm.compute_errors(sc, x, y)
        out[f"{name}_err_x"] = x
        out[f"{name}_err_y"] = y
        out[f"{name}_err"] = np.array([getattr(rep, f) for f in rterm.ErrorReport.__dataclass_fields__])
        # one line search from a random point and a gap value at it
        omega, eta = 1.3, 0.9 / sc.G.max_abs()
        z = reng.IterateZ(x * 0.1, np.abs(y) * 0.1)
        st = reng.adaptive_step_pdhg(sc, z, omega, eta, 7)
        out[f"{name}_ls"] = np.array([st.eta_used, st.eta_next, st.k_bar, st.trials])
        out[f"{name}_ls_x"] = st.z_hat.x
        out[f"{name}_ls_y"] = st.z_hat.y
        ctx = ref.WeightedNormContext(omega, eta)
        gx, gty = sc.G.matvec(z.x), sc.G.rmatvec(z.y)
        q = rrestart.GapQuery(x=z.x, y=z.y, b1=gty - sc.c, b2=sc.h - gx, r=0.5, ctx=ctx,
                              proj_x=lambda v: rcones.project_primal_set(v, sc),
                              proj_y=lambda v: rcones.project_dual_set(v, sc))
        try:
            out[f"{name}_gap"] = np.array([rrestart.normalized_gap(q)])
        except rrestart.GapEvaluationError:
            out[f"{name}_gap"] = np.array([np.nan])
    np.savez_compressed(os.path.join(HERE, "components.npz"), **out)


def main():
    projection_vectors()
    hand = hand_instances()
    bench = small_benchmarks()
    tight = dict(rel_tol=1e-6, abs_tol=1e-6)
    solve_case("tiny", hand["tiny"], tight)
    solve_case("ball", hand["ball"], tight)
    solve_case("expc", hand["expc"], tight)
    solve_case("dexp", hand["dexp"], tight)
    solve_case("rsoc", hand["rsoc"], tight)
    solve_case("prim", hand["prim"], dict(rel_tol=1e-5, abs_tol=1e-5, max_iter=200_000))
    solve_case("infeas", hand["infeas"], dict(max_iter=100_000))
    solve_case("unbnd", hand["unbnd"], dict(max_iter=100_000))
    solve_case("maxit", hand["tiny"], dict(max_iter=5, rel_tol=1e-12, abs_tol=1e-12))
    solve_case("plain", hand["tiny"], dict(use_preconditioner=False, use_adaptive_restart=False,
                                           use_adaptive_step_size_weight=False,
                                           fixed_reflection_beta=0.0, max_iter=200,
                                           rel_tol=1e-14, abs_tol=1e-14))
    solve_case("c1s", bench["c1s"], tight)
    solve_case("c1s_avg", bench["c1s"], dict(rel_tol=1e-4, abs_tol=1e-4, method="average"))
    solve_case("c1s_kkt", bench["c1s"], dict(rel_tol=1e-4, abs_tol=1e-4, use_duality_gap_restart=False,
                                             use_kkt_restart=True))
    solve_case("c2s", bench["c2s"], dict(rel_tol=1e-5, abs_tol=1e-5, max_iter=200_000))
    solve_case("c3s", bench["c3s"], dict(rel_tol=1e-5, abs_tol=1e-5, max_iter=200_000))
    solve_case("c4s", bench["c4s"], dict(rel_tol=1e-5, abs_tol=1e-5, max_iter=200_000))
    solve_case("c5s", bench["c5s"], dict(rel_tol=1e-5, abs_tol=1e-5, max_iter=200_000))
    component_vectors(bench)


if __name__ == "__main__":
    main()
