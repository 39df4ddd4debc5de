"""Pin the CPU oracle (oracle/pdcs_oracle.py) to the reference's own outputs.

The golden fixtures were produced by running the reference conic_pdhg on the
same inputs (tests/golden/make_golden.py).  The oracle restates the reference
algorithm operation for operation, so agreement is expected to the last bit
or within a few ulps; iteration counts and statuses must match exactly.
"""

import math

import numpy as np
import pytest

from golden_io import SOLVE_CASES, load, options, problem
from oracle import pdcs_oracle as O


@pytest.fixture(scope="module")
def proj():
    return load("projections")


def _split(flat, lens):
    out, s = [], 0
    for n in lens:
        out.append(flat[s:s + n])
        s += n
    return out


def test_exp_projection_matches_reference(proj):
    got = np.array([O.proj_exp(v) for v in proj["exp_in"]])
    np.testing.assert_allclose(got, proj["exp_out"], rtol=0, atol=1e-13)
    got = np.array([O.proj_dual_exp(v) for v in proj["exp_in"]])
    np.testing.assert_allclose(got, proj["dexp_out"], rtol=0, atol=1e-13)
    got = np.array([O.proj_exp(v) for v in proj["exp_stiff_in"]])
    np.testing.assert_allclose(got, proj["exp_stiff_out"], rtol=1e-13, atol=1e-13)


def test_soc_projections_match_reference(proj):
    for v, w in zip(_split(proj["soc_in"], proj["soc_len"]), _split(proj["soc_out"], proj["soc_len"])):
        np.testing.assert_array_equal(O.proj_soc(v), w)
    ins = _split(proj["rsoc_in"], proj["rsoc_len"])
    scs = _split(proj["rsoc_scale"], proj["rsoc_len"])
    outs = _split(proj["rsoc_out"], proj["rsoc_len"])
    for v, s, w in zip(ins, scs, outs):
        np.testing.assert_array_equal(O.proj_scaled_soc(v, s), w)


@pytest.mark.parametrize("case", SOLVE_CASES)
def test_oracle_solve_matches_reference(case):
    d = load("solve_" + case)
    p = problem(d)
    opts = options(d)
    snaps = {}

    def cb(st, loop):
        if ("trace_x_%d" % st.k_bar) in d:
            snaps[st.k_bar] = (st.x.copy(), st.y.copy())

    r = O.solve(p, O.options_from(None, **opts), callback=cb)
    assert r["status"] == str(d["status"])
    assert r["iterations"] == int(d["iterations"])
    assert r["restarts"] == int(d["restarts"])
    if math.isfinite(float(d["p_obj"])) and abs(float(d["p_obj"])) < 1e10:
        assert r["p_obj"] == pytest.approx(float(d["p_obj"]), rel=1e-9, abs=1e-9)
    scale = max(1.0, float(np.max(np.abs(d["x"]))) if d["x"].size else 1.0)
    np.testing.assert_allclose(r["x"], d["x"], rtol=0, atol=1e-8 * scale)
    for kb, (x, y) in snaps.items():
        np.testing.assert_allclose(x, d["trace_x_%d" % kb], rtol=0, atol=1e-12)
        np.testing.assert_allclose(y, d["trace_y_%d" % kb], rtol=0, atol=1e-12)


@pytest.mark.parametrize("name", ["c1s", "c2s", "c3s", "c4s", "c5s"])
def test_oracle_components_match_reference(name):
    comp = load("components")
    p = O.as_oproblem(problem(load("solve_" + name)))
    work = O.rsoc_presolve(p)
    d1, d2 = O.build_scaling(work)
    np.testing.assert_allclose(d1, comp[name + "_d1"], rtol=1e-14)
    np.testing.assert_allclose(d2, comp[name + "_d2"], rtol=1e-14)
    S = O.rescale(work, comp[name + "_d1"], comp[name + "_d2"])
    rep = O.metrics(S, comp[name + "_err_x"], comp[name + "_err_y"])
    keys = ["abs_p", "abs_d", "abs_gap", "rel_p1", "rel_d1", "rel_gap1", "abs_p_inf", "abs_d_inf",
            "abs_gap_term", "rel_p_inf", "rel_d_inf", "rel_gap_term", "primal_obj", "dual_obj"]
    np.testing.assert_allclose([rep[k] for k in keys], comp[name + "_err"], rtol=1e-12, atol=1e-12)
    x, y = comp[name + "_err_x"] * 0.1, np.abs(comp[name + "_err_y"]) * 0.1
    omega, eta = 1.3, 0.9 / float(np.max(np.abs(S.G.data)))
    xh, yh, eu, en, kb, trials, _ = O.line_search(S, x, y, omega, eta, 7, S.rmv(y), S.mv(x))
    np.testing.assert_allclose([eu, en, kb, trials], comp[name + "_ls"], rtol=1e-12)
    np.testing.assert_allclose(xh, comp[name + "_ls_x"], atol=1e-12)
    np.testing.assert_allclose(yh, comp[name + "_ls_y"], atol=1e-12)
    gx, gty = S.mv(x), S.rmv(y)
    try:
        g = O.normalized_gap(x, y, gty - S.c, S.h - gx, 0.5, eta / omega, eta * omega,
                             lambda v: O.proj_X(S, v), lambda v: O.proj_Y(S, v))
    except O.OracleGapError:
        g = float("nan")
    ref = float(comp[name + "_gap"][0])
    if math.isnan(ref):
        assert math.isnan(g)
    else:
        assert g == pytest.approx(ref, rel=1e-10, abs=1e-12)
