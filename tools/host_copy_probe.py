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

for rep in range(3):
    t = time.perf_counter()
    m = mmap.mmap(-1, n * 8, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS | mmap.MAP_POPULATE)
    o3 = np.frombuffer(m, dtype=np.float64)
    a = time.perf_counter() - t
    o3[:] = src
    b = time.perf_counter() - t
    print(f"MAP_POPULATE mmap {a*1e3:.1f} ms, + copy {b*1e3:.1f} ms (160 MB)")
from concurrent.futures import ThreadPoolExecutor
pool = ThreadPoolExecutor(4)
for rep in range(3):
    t = time.perf_counter()
    out = np.empty(n)
    k = 4
    cuts = [n * i // k for i in range(k + 1)]
    list(pool.map(lambda i: out.__setitem__(slice(cuts[i], cuts[i + 1]), src[cuts[i]:cuts[i + 1]]), range(k)))
    print(f"fresh np.empty + 4-thread copy {(time.perf_counter() - t)*1e3:.1f} ms (160 MB)")
