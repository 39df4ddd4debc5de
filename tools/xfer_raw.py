"""Raw pinned host->device / device->host copy bandwidth on the GPU box."""
import time

import torch

n = 512 << 20
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, f in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
    f(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(f"{name} pinned 512 MB: {n / dt / 1e9:.1f} GB/s")
import numpy as np
a = np.ones(n // 8); b = np.empty_like(a); b[:] = a
t = time.perf_counter(); b[:] = a; dt = time.perf_counter() - t
print(f"host memcpy 512 MB one thread: {n / dt / 1e9:.1f} GB/s")
