"""Where does one check (termination scan + restart check) spend its time?

    python tools/profile_check.py C5        (on a GPU box)

Builds the bench loop for a config, advances to one iteration before the
first check, then runs the batch that ends at the check under cProfile and
prints the top entries by cumulative time.
"""

import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(cfg):
    import bench
    from paper_2603_15504_b200 import SolverOptions, instances
    from paper_2603_15504_b200.engine import _Loop

    _, make = bench.WORKLOADS[cfg]
    problem = make(instances)
    loop = _Loop(problem, SolverOptions(rel_tol=1e-12, abs_tol=1e-12, max_iter=10**9, time_limit=1e9))
    state, ex = loop._start()
    ex = loop._advance(state, ex, until=loop.check_freq - 1)
    loop.dev.stream.synchronize()
    t0 = time.monotonic()
    pr = cProfile.Profile()
    pr.enable()
    ex = loop._advance(state, ex, until=loop.check_freq + 1)
    loop.dev.stream.synchronize()
    pr.disable()
    print(f"{cfg}: batch through the check at k_bar={loop.check_freq}: {time.monotonic() - t0:.4f} s")
    pstats.Stats(pr).sort_stats("cumulative").print_stats(35)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C5")
