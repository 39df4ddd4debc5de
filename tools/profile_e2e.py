"""Host-side profile of the public solve() on a config (the e2e leg of bench.py).

    python tools/profile_e2e.py C5 [iterations]     (on a GPU box)
"""

import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(cfg, iters, cold=False):
    import torch

    import bench
    from paper_2603_15504_b200 import SolverOptions, instances, solve

    _, make = bench.WORKLOADS[cfg]
    problem = make(instances)
    opts = SolverOptions(rel_tol=1e-12, abs_tol=1e-12, max_iter=iters, time_limit=1e9)
    solve(problem, SolverOptions(rel_tol=1e-12, abs_tol=1e-12, max_iter=2, time_limit=1e9))  # warm
    torch.cuda.synchronize()
    if cold:  # as bench.py's e2e leg: the caching allocator emptied first
        torch.cuda.empty_cache()
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    r = solve(problem, opts)
    pr.disable()
    print(f"{cfg}: {r.iterations} iterations, wall {time.perf_counter() - t0:.3f} s")
    pstats.Stats(pr).sort_stats("cumulative").print_stats(40)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C5", int(sys.argv[2]) if len(sys.argv) > 2 else 2000,
         len(sys.argv) > 3 and sys.argv[3] == "cold")
