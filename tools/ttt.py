"""Time-to-tolerance runs through the public solve(): status,
iterations, wall time (setup included, like the reference's wall_time_s) and
the loop-only time, one JSON line per run.

    python tools/ttt.py C5 1e-4 [time_limit_s]
    python tools/ttt.py C5planted 1e-6 [time_limit_s]   (lp_planted: a known optimum)
"""

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(cfg, tol, limit):
    from paper_2603_15504_b200 import SolverOptions, instances, solve

    make = {"C1": lambda: instances.lp_random(2000, 4000, 0.01, 0), "C2": instances.group_robust_regression,
            "C3": instances.entropy_max, "C4": instances.markowitz_rsoc, "C5": instances.lp_large,
            "C5planted": instances.lp_planted}[cfg]
    t0 = time.perf_counter()
    p = make()
    gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    r = solve(p, SolverOptions(rel_tol=tol, abs_tol=tol, time_limit=limit))
    wall = time.perf_counter() - t0
    line = {"config": cfg, "tol": tol, "status": r.exit_status, "iterations": r.iterations,
            "restarts": r.restarts, "wall_s": wall, "solve_time_s": r.solve_time_s, "p_obj": r.p_obj,
            "d_obj": r.d_obj, "time_limit_s": limit, "instance_gen_s": gen}
    if cfg == "C5planted":
        import numpy as np

        # lp_planted's optimum value c'x* (the generator plants x*; recomputed here)
        line["note"] = "lp_planted: C5 pattern with a planted strictly complementary optimum"
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), float(sys.argv[3]) if len(sys.argv) > 3 else 3600.0)
