"""Engine setup cost of a public solve() on C5 (GPU box).

    python tools/time_setup.py

Times DeviceEngine construction (slab allocation, H2D staging, libpdcs engine
create: transpose, SpMV plans, panels) and device preconditioning inside a
2-iteration solve, after a warm-up solve.
"""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2603_15504_b200.device as dev
    from paper_2603_15504_b200 import SolverOptions, instances, solve

    p = instances.lp_large()
    opts = SolverOptions(max_iter=2, rel_tol=1e-12, abs_tol=1e-12)
    solve(p, opts)  # warm-up (CUDA context, libpdcs load, pinned staging buffers)
    torch.cuda.synchronize()
    times = {}

    def timed(name, fn):
        def wrapper(self, *a, **k):
            t0 = time.perf_counter()
            out = fn(self, *a, **k)
            times[name] = time.perf_counter() - t0
            return out
        return wrapper

    dev.DeviceEngine.__init__ = timed("engine_init", dev.DeviceEngine.__init__)
    dev.DeviceEngine.precondition = timed("precondition", dev.DeviceEngine.precondition)
    t0 = time.perf_counter()
    solve(p, opts)
    print("solve of 2 iterations: %.3f s" % (time.perf_counter() - t0),
          {k: round(v, 3) for k, v in times.items()})


if __name__ == "__main__":
    main()
