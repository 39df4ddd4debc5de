"""The batched normalized-gap search (restart._normalized_gap_batched: several
probes per device pass) must return exactly what the reference's sequential
exponential search + bisection returns (restart.py:80-132 of the reference;
oracle.pdcs_oracle.normalized_gap)."""

import math

import numpy as np
import pytest

from oracle import pdcs_oracle as O
from paper_2603_15504_b200 import restart as R


class SeqQuery:
    """probe(t) only: drives the sequential search."""

    def __init__(self, f, r):
        self.f, self.r, self.calls = f, r, []

    def probe(self, t):
        self.calls.append(t)
        return self.f(t)


class BatchQuery(SeqQuery):
    def __init__(self, f, r):
        super().__init__(f, r)
        self.passes = 0

    def probe_many(self, ts):
        self.passes += 1
        return [self.probe(t) for t in ts]


def saturating(scale, cap, slope):
    """dist grows like scale*sqrt(t) up to cap (a bounded feasible set); the
    gap value is a smooth increasing function of t."""
    def f(t):
        d = min(scale * math.sqrt(t), cap)
        return d, slope * (1.0 - math.exp(-t)) + 1e-3 * d
    return f


CASES = [
    (saturating(1.0, 1e9, 2.0), 3.0),      # brackets after a few doublings
    (saturating(1.0, 1e9, 2.0), 0.5),      # brackets at the first probe
    (saturating(1e-6, 1e9, 1.0), 10.0),    # many doublings (beyond one batch)
    (saturating(1.0, 2.0, 1.0), 5.0),      # saturates below r: two-stall exit
    (saturating(3.0, 1e9, -1.0), 7.25),
]


@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("t0", [1.0, 0.37, 1e-3])
def test_batched_search_matches_sequential(case, t0):
    f, r = CASES[case]
    seq, bat = SeqQuery(f, r), BatchQuery(f, r)
    v_seq = R._normalized_gap_sequential(seq, t0, 1e-8)
    v_bat = R.normalized_gap(bat, t0)
    assert v_bat == v_seq  # bit-identical: same probes along the same path
    assert set(seq.calls) <= set(bat.calls)
    assert bat.passes < len(seq.calls)


def test_batched_search_matches_oracle():
    """Against the oracle's restatement of the reference search on real
    vectors (box primal set, nonnegative dual set)."""
    rng = np.random.default_rng(0)
    for trial in range(10):
        n, m = 50, 30
        x, y = rng.standard_normal(n), np.abs(rng.standard_normal(m))
        b1, b2 = rng.standard_normal(n), rng.standard_normal(m)
        tau, sigma = rng.uniform(0.1, 2), rng.uniform(0.1, 2)
        r = rng.uniform(0.1, 3.0)
        px = lambda v: np.clip(v, -2.0, 2.0)  # noqa: E731
        py = lambda v: np.maximum(v, 0.0)  # noqa: E731

        def f(t):
            zx, zy = px(x + (t * tau) * b1), py(y + (t * sigma) * b2)
            dx, dy = x - zx, y - zy
            d = float(np.sqrt(np.dot(dx, dx) / tau + np.dot(dy, dy) / sigma))
            return d, (float(np.dot(b1, zx - x)) + float(np.dot(b2, zy - y))) / r

        try:
            v_or = O.normalized_gap(x, y, b1, b2, r, tau, sigma, px, py)
        except O.OracleGapError:
            with pytest.raises(R.GapEvaluationError):
                R.normalized_gap(BatchQuery(f, r))
            continue
        assert R.normalized_gap(BatchQuery(f, r)) == v_or, trial


def test_constant_distance_stalls():
    f = lambda t: (0.25, 0.0)  # noqa: E731 -- never exceeds r: two-stall exit
    assert R.normalized_gap(BatchQuery(f, 1.0)) == R._normalized_gap_sequential(SeqQuery(f, 1.0), 1.0, 1e-8)


def test_tiny_radius():
    assert R.normalized_gap(BatchQuery(lambda t: (1.0, 1.0), 0.0)) == 0.0
