"""Host-side copy speeds on the GPU box: fresh np.empty pages (first-touch
faults) vs a transparent-huge-page mapping, for the download path."""
import mmap
import time

import numpy as np

n = 20_000_000
src = np.random.default_rng(0).random(n)
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
for rep in range(3):
    t = time.perf_counter(); out = np.empty(n); out[:] = src; a = time.perf_counter() - t
    t = time.perf_counter(); out[:] = src; b = time.perf_counter() - t
    t = time.perf_counter()
    m = mmap.mmap(-1, n * 8, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    m.madvise(mmap.MADV_HUGEPAGE)
    o2 = np.frombuffer(m, dtype=np.float64); o2[:] = src
    c = time.perf_counter() - t
    print(f"fresh np.empty + copy {a*1e3:.1f} ms, warm copy {b*1e3:.1f} ms, THP mmap + copy {c*1e3:.1f} ms (160 MB)")
