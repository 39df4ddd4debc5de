"""Run-to-run spread of the C5 end-to-end solve (bench.py's e2e leg), with the
engine's setup phases (PDCS_TIMING=1) on stderr.   python tools/e2e_var.py [reps]"""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(reps):
    import torch

    import bench
    from paper_2603_15504_b200 import SolverOptions, instances, solve

    import collections
    import functools

    from paper_2603_15504_b200 import device, engine

    acc = collections.defaultdict(float)

    def timed(owner, name, label):
        f = getattr(owner, name)

        @functools.wraps(f)
        def w(*a, **k):
            t = time.perf_counter()
            try:
                return f(*a, **k)
            finally:
                acc[label] += time.perf_counter() - t
        setattr(owner, name, w)

    timed(device, "h2d", "h2d")
    timed(device, "d2h", "d2h")
    timed(device, "_slab", "slab zeros")
    timed(device.DeviceEngine, "__init__", "engine init (slabs+h2d+create)")
    timed(device.DeviceEngine, "precondition", "precondition")
    timed(device.DeviceEngine, "run_inner", "run_inner")
    timed(engine._Loop, "__init__", "loop init")
    timed(engine._Loop, "run", "loop run")
    timed(engine._Loop, "close", "close")
    _, make = bench.WORKLOADS["C5"]
    p = make(instances)
    opts = SolverOptions(rel_tol=1e-12, abs_tol=1e-12, max_iter=20, time_limit=1e9)
    for i in range(reps):
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        t0 = time.perf_counter()
        r = solve(p, opts)
        print(f"rep {i}: {r.iterations} it, wall {time.perf_counter() - t0:.3f} s  "
              + "  ".join(f"{k} {v * 1e3:.1f}" for k, v in acc.items()), flush=True)
        acc.clear()
        print(f"rep {i} done", file=sys.stderr, flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
