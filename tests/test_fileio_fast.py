"""The native problem-file reader (csrc/pdcs_io.cpp)
against the json-module path on the same files: identical ConicProblem
arrays, identical warnings and errors (documents outside the fast grammar
fall back to json)."""

import json
import math
import warnings

import numpy as np
import pytest

from paper_2603_15504_b200 import fileio, instances
from paper_2603_15504_b200.fileio import ProblemFormatError


def _same_problem(a, b):
    for k in ("c", "h", "l", "u"):
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k))
    ga, gb = a.G.to_scipy(), b.G.to_scipy()
    np.testing.assert_array_equal(ga.indptr, gb.indptr)
    np.testing.assert_array_equal(ga.indices, gb.indices)
    np.testing.assert_array_equal(ga.data, gb.data)
    assert a.num_box == b.num_box
    assert [(s.kind, s.dim) for s in a.dual_cones] == [(s.kind, s.dim) for s in b.dual_cones]


def _both(path):
    fast = fileio.parse_problem(str(path))
    slow = fileio.parse_problem(str(path), fast=False)
    _same_problem(fast, slow)
    return fast


@pytest.mark.parametrize("make", [
    lambda: instances.lp_random(200, 400, 0.05, 3),
    lambda: instances.group_robust_regression(ngroups=20, gsize=5, q=60, nnz_per_row=10, seed=2),
    lambda: instances.entropy_max(nblk=40, p=8, nnz_per_col=2, seed=3),
])
def test_fast_reader_matches_json(tmp_path, make):
    p = make()
    if p.num_box != p.n:
        pytest.skip("file format is box-only")
    path = tmp_path / "p.json"
    fileio.serialize_problem(p, str(path))
    _both(path)


def test_fast_reader_inf_bounds_rsoc_unknown_keys_and_large_arrays(tmp_path):
    rng = np.random.default_rng(4)
    n, m, nnz = 3000, 2500, 40_000
    doc = {"format_version": 1, "n": n, "m": m, "nb": n,
           "c": rng.standard_normal(n).tolist(), "h": (rng.standard_normal(m) * 1e-7).tolist(),
           "bl": ["-inf" if i % 3 == 0 else -1.5 for i in range(n)],
           "bu": ["inf" if i % 5 == 0 else 2.0 for i in range(n)],
           "G": {"rows": rng.integers(0, m, nnz).tolist(), "cols": rng.integers(0, n, nnz).tolist(),
                 "vals": (rng.standard_normal(nnz) * 10.0 ** rng.integers(-30, 30, nnz)).tolist()},
           "mGzero": 100, "mGnonnegative": 2000, "socG": [5, 10], "expG": 10, "dual_expG": 5,
           "rsocG": [340], "comment": {"nested": [1, 2, {"x": "y"}]}, "zz_extra": "text"}
    path = tmp_path / "big.json"
    path.write_text(json.dumps(doc, indent=1))
    with warnings.catch_warnings(record=True) as w1:
        warnings.simplefilter("always")
        fast = fileio.parse_problem(str(path))
    with warnings.catch_warnings(record=True) as w2:
        warnings.simplefilter("always")
        slow = fileio.parse_problem(str(path), fast=False)
    _same_problem(fast, slow)
    assert [str(x.message) for x in w1] == [str(x.message) for x in w2] != []
    assert math.isinf(fast.l[0]) and fast.l[0] < 0 and math.isinf(fast.u[0])


@pytest.mark.parametrize("text", [
    '{"format_version": 1, "n": 1, "m": 1, "nb": 1, "c": [NaN], "h": [0.0], "bl": [0], "bu": [1],'
    ' "G": {"rows": [0], "cols": [0], "vals": [1.0]}, "mGnonnegative": 1}',
    '{"format_version": 1, "n": 1, "m": 1, "nb": 1, "c": [1.0], "h": [0.0], "bl": ["-infinity"],'
    ' "bu": [1], "G": {"rows": [0], "cols": [0], "vals": [1.0]}, "mGnonnegative": 1}',
    '{"format_version": 1, "n": 1, "m": 1, "nb": 1, "c": [1.0], "h": [0.0], "bl": [1e400], "bu": [1],'
    ' "G": {"rows": [0], "cols": [0], "vals": [1.0]}, "mGnonnegative": 1}',
    '{"format_version": 2, "n": 1, "m": 1, "nb": 1, "c": [1.0], "h": [0.0], "bl": [0], "bu": [1],'
    ' "G": {"rows": [0], "cols": [0], "vals": [1.0]}, "mGnonnegative": 1}',
    '{"format_version": 1, "n": 1, "m": 1, "nb": 1, "c": [1.0], "h": [0.0], "bl": [0], "bu": [1],'
    ' "G": {"rows": [3], "cols": [0], "vals": [1.0]}, "mGnonnegative": 1}',
    '{"format_version": 1, "n": 1, "m": 2, "nb": 1, "c": [1.0], "h": [0.0, 1], "bl": [0], "bu": [1],'
    ' "G": {"rows": [0], "cols": [0], "vals": [1.0]}, "mGnonnegative": 1}',
    '{"format_version": 1, "n": 1, "m": 1, "nb": 1, "c": [1.0,], "h": [0.0]}',
    '{"format_version": 1, "n": 1, "m": 1, "nb": 1, "c": [1.0], "h": [0.0], "bl": [0], "bu": [1],'
    ' "G": {"rows": [0.5], "cols": [0], "vals": [1.0]}, "mGnonnegative": 1}',
    'not json',
])
def test_fast_reader_errors_match_json(tmp_path, text):
    path = tmp_path / "bad.json"
    path.write_text(text)

    def outcome(fast):
        try:
            return "ok", fileio.parse_problem(str(path), fast=fast)
        except (ProblemFormatError, ValueError) as exc:
            return type(exc).__name__, str(exc)

    a, b = outcome(True), outcome(False)
    assert a[0] == b[0], (a, b)
    if a[0] == "ok":
        _same_problem(a[1], b[1])
    else:
        assert a[1] == b[1]
