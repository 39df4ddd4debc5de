"""One small solve per golden case, for compute-sanitizer runs
(tests/test_gpu_sanitizer.py):  python tools/sanitize_case.py c1s [max_iter]"""

import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def main(case: str, max_iter: int) -> None:
    from golden_io import load, options, problem
    from paper_2603_15504_b200 import SolverOptions, solve

    d = load("solve_" + case)
    opts = dict(options(d))
    opts["max_iter"] = min(int(opts.get("max_iter", 10**6)), max_iter)
    # a short check cadence so the check path (metrics, rays, gap probes,
    # restarts) runs inside the sanitized window too
    opts["duality_gap_restart_freq"] = 64
    r = solve(problem(d), SolverOptions(**opts))
    print(f"{case}: {r.exit_status} iterations={r.iterations}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 400)
