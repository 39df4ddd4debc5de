"""Iterations to tolerance of the C5 family at reduced sizes (on a GPU box).

    python tools/convergence_probe.py 100000 200000 [max_iter] [seed] [generator]

Prints the solver's check lines (verbose=1) and the exit record.
"""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2603_15504_b200 import SolverOptions, instances, solve

    m, n = int(sys.argv[1]), int(sys.argv[2])
    max_iter = int(sys.argv[3]) if len(sys.argv) > 3 else 200_000
    seed = int(sys.argv[4]) if len(sys.argv) > 4 else 5
    gen = sys.argv[5] if len(sys.argv) > 5 else "lp_large"
    p = getattr(instances, gen)(m, n, seed=seed)
    t0 = time.perf_counter()
    r = solve(p, SolverOptions(rel_tol=1e-6, abs_tol=1e-6, max_iter=max_iter, time_limit=600,
                               verbose=1, print_freq=10_000))
    print(f"m={m} n={n}: {r.exit_status} iters={r.iterations} wall={time.perf_counter() - t0:.2f}s "
          f"restarts={r.restarts}")


if __name__ == "__main__":
    main()
