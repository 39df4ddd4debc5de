"""conic-pdhg command line (paper_2603_15504_b200.cli) against the reference
CLI contract (cli.py:26-110): flags, exit codes 0 / 1 / 64, result file."""

import json

import numpy as np
import pytest

from golden_io import load, problem


def _write_problem(tmp_path, name="tiny"):
    from paper_2603_15504_b200 import fileio

    p = problem(load("solve_" + name))
    path = tmp_path / f"{name}.json"
    fileio.serialize_problem(p, str(path))
    return p, path


def _main(argv):
    from paper_2603_15504_b200.cli import main

    return main(argv)


def test_missing_input_flag_is_usage_error(capsys):
    assert _main([]) == 64
    assert "error" in capsys.readouterr().err


def test_missing_file_is_usage_error(tmp_path):
    assert _main(["--input", str(tmp_path / "nope.json")]) == 64


def test_malformed_file_is_usage_error(tmp_path):
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"format_version": 2}))
    assert _main(["--input", str(bad)]) == 64
    bad.write_text("{not json")
    assert _main(["--input", str(bad)]) == 64


def test_invalid_options_are_usage_errors(tmp_path):
    _, path = _write_problem(tmp_path)
    assert _main(["--input", str(path), "--rel-tol", "-1"]) == 64
    assert _main(["--input", str(path), "--max-iter", "0"]) == 64
    assert _main(["--input", str(path), "--method", "nope"]) == 64
    assert _main(["--input", str(path), "--verbose", "7"]) == 64


def test_threads_env_is_validated(tmp_path, monkeypatch):
    _, path = _write_problem(tmp_path)
    # reference cli.py:66-78, 86: SystemExit(message) outside the usage-error path
    # (T/test_cli.py test_threads_env_validation expects pytest.raises(SystemExit))
    monkeypatch.setenv("CONIC_PDHG_THREADS", "zero")
    with pytest.raises(SystemExit, match="must be an integer"):
        _main(["--input", str(path)])
    monkeypatch.setenv("CONIC_PDHG_THREADS", "0")
    with pytest.raises(SystemExit, match="at least 1"):
        _main(["--input", str(path)])


def test_help_exits_zero():
    assert _main(["--help"]) == 0


def test_options_mapping():
    from paper_2603_15504_b200.cli import build_parser, options_from_args

    a = build_parser().parse_args(["--input", "x", "--rel-tol", "1e-4", "--no-preconditioner",
                                   "--kkt-restart", "--gap-restart-freq", "64", "--method", "average"])
    o = options_from_args(a)
    assert o.rel_tol == 1e-4 and not o.use_preconditioner and o.use_kkt_restart
    assert o.duality_gap_restart_freq == 64 and o.method == "average"


@pytest.mark.gpu
def test_cli_solves_and_writes_result(tmp_path):
    from paper_2603_15504_b200.fileio import load_result

    d = load("solve_tiny")
    _, path = _write_problem(tmp_path)
    out = tmp_path / "res.json"
    opts = json.loads(str(d["opts_json"]))
    argv = ["--input", str(path), "--output", str(out), "--rel-tol", str(opts.get("rel_tol", 1e-6)),
            "--abs-tol", str(opts.get("abs_tol", 1e-6))]
    assert _main(argv) == 0
    res = load_result(str(out))
    assert res["exit_status"] == str(d["status"])
    assert np.isclose(res["pObj"], float(d["p_obj"]), rtol=1e-5, atol=1e-6)


@pytest.mark.gpu
def test_cli_limit_exits_one(tmp_path):
    _, path = _write_problem(tmp_path, "c1s")
    assert _main(["--input", str(path), "--max-iter", "10"]) == 1
