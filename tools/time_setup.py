import sys, time
sys.path.insert(0, '.')
import torch
from paper_2603_15504_b200 import instances, SolverOptions, solve
from paper_2603_15504_b200 import device as D
import ctypes as C
p = instances.lp_large()
solve(p, SolverOptions(max_iter=2, rel_tol=1e-12, abs_tol=1e-12))  # warm
torch.cuda.synchronize()
orig = D.N.lib().pdcs_engine_create
t = {}
lib = D.N.lib()
class Wrap:
    pass
import paper_2603_15504_b200.device as dev
old_init = dev.DeviceEngine.__init__
def timed_init(self, *a, **k):
    t0 = time.perf_counter(); old_init(self, *a, **k); t['init'] = time.perf_counter() - t0
dev.DeviceEngine.__init__ = timed_init
old_pre = dev.DeviceEngine.precondition
def timed_pre(self, *a, **k):
    t0 = time.perf_counter(); old_pre(self, *a, **k); t['pre'] = time.perf_counter() - t0
dev.DeviceEngine.precondition = timed_pre
t0 = time.perf_counter()
r = solve(p, SolverOptions(max_iter=2, rel_tol=1e-12, abs_tol=1e-12))
print('solve 2 its total %.3f s' % (time.perf_counter() - t0), {k: round(v, 3) for k, v in t.items()})
