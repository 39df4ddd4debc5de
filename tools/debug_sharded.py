"""Compare the sharded engine (world 1) with the single-GPU engine iteration by iteration."""
import os, socket, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch, torch.distributed as dist
from golden_io import load, problem
import paper_2603_15504_b200 as P
from paper_2603_15504_b200.distributed import solve_sharded

s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1, device_id=torch.device("cuda", 0))
p = problem(load("solve_" + (sys.argv[1] if len(sys.argv) > 1 else "c1s")))
tr = {"one": [], "sh": []}
def grab(w):
    def cb(s):
        tr[w].append((s.k_bar, s.eta, s.eta_hat, s.omega, s.beta, s.k, float(np.linalg.norm(s.z.x)), float(np.linalg.norm(s.z.y))))
    return cb
N = int(sys.argv[2]) if len(sys.argv) > 2 else 60
P.solve(p, P.SolverOptions(max_iter=N, rel_tol=1e-14, abs_tol=1e-14, iteration_callback=grab("one")))
solve_sharded(p, P.SolverOptions(max_iter=N, rel_tol=1e-14, abs_tol=1e-14, iteration_callback=grab("sh")))
for a, b in zip(tr["one"], tr["sh"]):
    flag = "" if np.allclose(a, b, rtol=1e-12, atol=1e-14) else "  <-- differs"
    print(a, "\n", b, flag)
r1 = P.solve(p, P.SolverOptions(rel_tol=1e-6, abs_tol=1e-6))
r2 = solve_sharded(p, P.SolverOptions(rel_tol=1e-6, abs_tol=1e-6))
print("single", r1.exit_status, r1.iterations, r1.p_obj, "sharded", r2.exit_status, r2.iterations, r2.p_obj)
dist.destroy_process_group()
