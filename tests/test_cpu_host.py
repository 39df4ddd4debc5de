"""CPU-only checks: the C-ABI library loads and exports every symbol that
include/pdcs.h declares, the ctypes structures match the header layout, and
the host-side logic (API surface, file format, generators, B_alg) works
without a GPU."""

import ctypes
import math
import os
import re
import subprocess

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "pdcs.h")


def _declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pdcs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2603_15504_b200 import _native

    lib = _native.load_library()
    declared = _declared_functions()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_native.EXPORTED)
    assert lib.pdcs_abi_version() == 1


def test_ctypes_layout_matches_header(tmp_path):
    from paper_2603_15504_b200 import _native as N

    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include "pdcs.h"\n#include <stddef.h>\n'
                   'int main(){printf("%zu %zu %zu %zu %zu\\n", sizeof(PdcsCtrl), sizeof(PdcsEngineDesc),'
                   ' sizeof(PdcsBlock), offsetof(PdcsCtrl, eta_hat), offsetof(PdcsEngineDesc, d_ty2));}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(REPO, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(N.PdcsCtrl), ctypes.sizeof(N.PdcsEngineDesc), ctypes.sizeof(N.PdcsBlock),
            N.PdcsCtrl.eta_hat.offset, N.PdcsEngineDesc.d_ty2.offset]
    assert got == want


def test_public_surface_matches_reference_names():
    import paper_2603_15504_b200 as P

    want = ["Cone", "ConeSpec", "ConicProblem", "DualRecovery", "ErrorReport", "ExitInfo", "EXIT_STATUS",
            "IterateZ", "LambdaSet", "NumericalError", "SolveResult", "SolverOptions", "SolverState",
            "SparseMatrix", "WeightedNormContext", "parse_problem", "serialize_problem", "solve",
            "write_result"]
    assert P.__all__ == want
    for name in want:
        assert hasattr(P, name)


def test_device_path_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2603_15504_b200 as P
    from paper_2603_15504_b200._native import NativeUnavailable

    p = P.ConicProblem(c=np.array([1.0]), G=P.SparseMatrix(np.zeros((0, 1))), h=np.zeros(0),
                       l=np.array([0.0]), u=np.array([1.0]), num_box=1)
    with pytest.raises(NativeUnavailable):
        P.solve(p)


def test_options_validation():
    import paper_2603_15504_b200 as P

    for bad in (dict(method="nope"), dict(rel_tol=0.0), dict(initial_step_norm="spectral"),
                dict(time_limit=0.0), dict(fixed_reflection_beta=2.0), dict(max_iter=0)):
        with pytest.raises(ValueError):
            P.SolverOptions(**bad).validate()


def test_model_validation_and_layout():
    from paper_2603_15504_b200.model import Cone, ConeSpec, ConicProblem, dual_layout
    from paper_2603_15504_b200.linalg import SparseMatrix

    with pytest.raises(ValueError):
        ConeSpec(Cone.EXP, 2)
    with pytest.raises(ValueError):
        ConeSpec(Cone.FREE, 2)
    G = SparseMatrix(np.ones((6, 2)))
    p = ConicProblem(c=np.zeros(2), G=G, h=np.zeros(6), l=-np.ones(2), u=np.ones(2), num_box=2,
                     dual_cones=(ConeSpec(Cone.ZERO, 1), ConeSpec(Cone.NONNEG, 2), ConeSpec(Cone.SOC, 3)))
    assert dual_layout(p) == (1, 3)
    with pytest.raises(ValueError):
        ConicProblem(c=np.zeros(2), G=G, h=np.zeros(6), l=-np.ones(2), u=np.ones(2), num_box=2,
                     dual_cones=(ConeSpec(Cone.SOC, 3), ConeSpec(Cone.NONNEG, 3)))


def test_rsoc_presolve_matches_oracle():
    from golden_io import load, problem
    from oracle import pdcs_oracle as O
    from paper_2603_15504_b200.model import rsoc_to_soc

    p = problem(load("solve_c4s"))
    w = rsoc_to_soc(p)
    ow = O.rsoc_presolve(O.as_oproblem(p))
    np.testing.assert_array_equal(w.h, ow.h)
    np.testing.assert_array_equal(w.G.toarray(), ow.G.toarray())
    assert [s.kind.value for s in w.dual_cones] == [k for k, _, _ in ow.dcones]


def test_fileio_roundtrip(tmp_path):
    from paper_2603_15504_b200 import fileio, instances

    p = instances.lp_random(30, 50, 0.2, 1)
    path = str(tmp_path / "p.json")
    fileio.serialize_problem(p, path)
    q = fileio.parse_problem(path)
    np.testing.assert_array_equal(p.c, q.c)
    np.testing.assert_array_equal(p.G.toarray(), q.G.toarray())
    assert [s.kind for s in p.dual_cones] == [s.kind for s in q.dual_cones]
    with pytest.raises(fileio.ProblemFormatError):
        fileio.document_to_problem({"format_version": 2})


def test_generators_have_the_surveyed_structure():
    from paper_2603_15504_b200 import instances

    p2 = instances.group_robust_regression(ngroups=20, gsize=10, q=90, nnz_per_row=12)
    assert p2.m == 2 * 90 + 20 * 11 and p2.n == 2 * 90 + 20
    p3 = instances.entropy_max(nblk=50, p=10)
    assert p3.m == 10 + 150 and p3.n == 100
    p4 = instances.markowitz_rsoc(N=100, k=4)
    assert p4.m == 1 + 4 + 2 + 4 + 100 and p4.n == 105
    assert p4.G.nnz == 100 + 100 * 4 + 4 + 1 + 4 + 100
    p5 = instances.lp_large(m=1000, n=2000)
    assert p5.G.nnz <= 5000 and np.all(np.diff(p5.G._csr.indptr) <= 5)


def test_algorithmic_bytes_formula():
    from paper_2603_15504_b200 import instances

    p = instances.lp_large(m=1000, n=2000)
    nnz = p.G.nnz
    assert instances.algorithmic_bytes(p) == 24 * nnz + 4 * 1001 + 4 * 2001 + 8 * (13 * 2000 + 2 * 2000 + 13 * 1000)


def test_normalized_gap_closed_form_host_query():
    """Criterion 7 of the reference acceptance suite on the API's host query."""
    from paper_2603_15504_b200.linalg import WeightedNormContext
    from paper_2603_15504_b200.restart import GapQuery, normalized_gap

    rng = np.random.default_rng(7)
    for _ in range(50):
        n, m = int(rng.integers(1, 8)), int(rng.integers(1, 8))
        ctx = WeightedNormContext(float(rng.uniform(0.2, 5.0)), float(rng.uniform(0.2, 5.0)))
        q = GapQuery(x=rng.standard_normal(n), y=rng.standard_normal(m), b1=rng.standard_normal(n),
                     b2=rng.standard_normal(m), r=float(rng.uniform(0.1, 10.0)), ctx=ctx,
                     proj_x=lambda v: v, proj_y=lambda v: v)
        closed = math.sqrt(ctx.tau * float(q.b1 @ q.b1) + ctx.sigma * float(q.b2 @ q.b2))
        assert abs(normalized_gap(q) - closed) <= 1e-6 * max(1.0, closed)


def test_restart_rules_and_constants():
    from paper_2603_15504_b200 import restart as R

    c = R.RestartConstants()
    assert (c.beta_sufficient, c.beta_necessary, c.beta_artificial, c.theta) == (0.4, 0.8, 0.223, 0.5)
    assert R.should_restart(0.39, 10.0, 1.0, 1, 100)
    assert R.should_restart(0.7, 0.6, 1.0, 1, 100)
    assert not R.should_restart(0.7, 0.8, 1.0, 1, 100)
    assert R.should_restart(0.9, 0.8, 1.0, 23, 100)
    assert R.update_primal_weight(1.0, 4.0, 1.0, 7.0) == pytest.approx(2.0)
    assert R.update_primal_weight(1e-12, 4.0, 3.0, 7.0) == 3.0
    assert R.update_primal_weight(1.0, 1e12, 1e4, 7.0) == 7.0
