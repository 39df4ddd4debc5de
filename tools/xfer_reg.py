"""cudaHostRegister of an existing numpy array + direct DMA vs the staged copy
path of device.h2d (600 MB, like C5's value array + column indices)."""
import ctypes
import time

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_15504_b200 import device  # noqa: E402

n = 75_000_000
a = np.random.default_rng(0).random(n)
d = torch.empty(n, dtype=torch.float64, device="cuda")
s = torch.cuda.Stream()
rt = torch.cuda.cudart()
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    device.h2d(d, a, s)
    t1 = time.perf_counter() - t
    t = time.perf_counter()
    ptr = a.ctypes.data
    r = rt.cudaHostRegister(ptr, a.nbytes, 0)
    t_reg = time.perf_counter() - t
    src = torch.from_numpy(a)
    with torch.cuda.stream(s):
        d.copy_(src, non_blocking=True)
    s.synchronize()
    t_dma = time.perf_counter() - t - t_reg
    t = time.perf_counter()
    rt.cudaHostUnregister(ptr)
    t_unreg = time.perf_counter() - t
    print(f"staged h2d {t1*1e3:.1f} ms | register {t_reg*1e3:.1f} + dma {t_dma*1e3:.1f} + unregister {t_unreg*1e3:.1f} ms (rc {r})")
