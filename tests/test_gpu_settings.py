"""ProjectionSettings honoured on the device (reference cones.py:24-32):
root_tol / max_root_iters reach the exp-cone Newton + bisection
(cones.py:225-265) and the rescaled-SOC brentq (cones.py:414-425) of the
standalone projection API, checked against the oracle run with the same
settings."""

import numpy as np
import pytest

from oracle import pdcs_oracle as O

pytestmark = pytest.mark.gpu


def _stiff_points(n=400, seed=11):
    rng = np.random.default_rng(seed)
    return np.concatenate([rng.standard_normal((n // 2, 3)) * 3.0,
                           rng.standard_normal((n // 2, 3)) * np.array([30.0, 0.1, 1.0])])


@pytest.mark.parametrize("tol,iters", [(1e-12, 100), (1e-6, 100), (1e-12, 22), (1e-3, 30), (1e-12, 5)])
def test_exp_projection_follows_settings(tol, iters):
    from paper_2603_15504_b200 import cones

    st = cones.ProjectionSettings(root_tol=tol, max_root_iters=iters)
    for v in _stiff_points():
        got = cones.project_exp(v, st)
        ref = O.proj_exp(v, tol, iters)
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12 * max(1.0, np.abs(v).max()))
        gd = cones.project_dual_exp(v, st)
        rd = O.proj_dual_exp(v, tol, iters)
        np.testing.assert_allclose(gd, rd, rtol=1e-12, atol=1e-12 * max(1.0, np.abs(v).max()))


def test_loose_settings_change_the_exp_result():
    """A root search capped at 2 Newton steps (max_root_iters=2: no
    bisection left) gives a coarser root than the default on some points: the
    device must follow the cap, not silently use the defaults."""
    from paper_2603_15504_b200 import cones

    differ = 0
    for v in _stiff_points():
        a = cones.project_exp(v)
        b = cones.project_exp(v, cones.ProjectionSettings(max_root_iters=2))
        differ += int(np.max(np.abs(a - b)) > 1e-10)
    assert differ > 0


def test_rescaled_soc_iteration_cap_raises_like_brentq():
    from paper_2603_15504_b200 import cones
    from paper_2603_15504_b200.linalg import NumericalError

    rng = np.random.default_rng(3)
    hits = 0
    for _ in range(50):
        d = int(rng.integers(3, 20))
        v = rng.standard_normal(d) * 3.0
        sc = rng.uniform(0.1, 10.0, d)
        try:
            ref = O.proj_scaled_soc(v, sc, iters=3)
        except O.OracleNumericalError:
            ref = None
        if ref is None:
            with pytest.raises(NumericalError):
                cones.project_rescaled_soc(v, sc, cones.ProjectionSettings(max_root_iters=3))
            hits += 1
        else:
            got = cones.project_rescaled_soc(v, sc, cones.ProjectionSettings(max_root_iters=3))
            np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-13)
    assert hits > 0
