"""Host<->device transfer and allocation options for the e2e path (GPU box).

    python tools/xfer_probe.py
"""

import time

import numpy as np
import torch


def t(f, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def main():
    n = 50_000_000
    a = np.random.default_rng(0).standard_normal(n)
    gb = a.nbytes / 1e9
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    print(f"array {gb:.2f} GB")
    print("H2D pageable copy_        %.1f GB/s" % (gb / t(lambda: d.copy_(torch.from_numpy(a)))))

    def pinned_stage():
        p = torch.from_numpy(a).pin_memory()
        d.copy_(p, non_blocking=True)
    print("H2D pin_memory + copy     %.1f GB/s" % (gb / t(pinned_stage)))

    cudart = torch.cuda.cudart()

    def registered():
        ptr = a.ctypes.data
        cudart.cudaHostRegister(ptr, a.nbytes, 0)
        d.copy_(torch.from_numpy(a), non_blocking=True)
        torch.cuda.synchronize()
        cudart.cudaHostUnregister(ptr)
    print("H2D cudaHostRegister      %.1f GB/s" % (gb / t(registered)))

    # chunked staging through a reused pinned buffer (two buffers, overlapped)
    stage = [torch.empty(1 << 24, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    s = torch.cuda.Stream()

    def chunked():
        src = torch.from_numpy(a)
        ev = [None, None]
        for i, off in enumerate(range(0, n, 1 << 24)):
            b = i & 1
            if ev[b] is not None:
                ev[b].synchronize()
            k = min(1 << 24, n - off)
            stage[b][:k].copy_(src[off:off + k])
            with torch.cuda.stream(s):
                d[off:off + k].copy_(stage[b][:k], non_blocking=True)
                ev[b] = torch.cuda.Event()
                ev[b].record(s)
        s.synchronize()
    print("H2D chunked pinned stage  %.1f GB/s" % (gb / t(chunked)))

    print("D2H .cpu()                %.1f GB/s" % (gb / t(lambda: d.cpu())))
    print("D2H .cpu().numpy().copy() %.1f GB/s" % (gb / t(lambda: d.cpu().numpy().copy())))
    hp = torch.empty(n, dtype=torch.float64, pin_memory=True)
    print("D2H into pinned           %.1f GB/s" % (gb / t(lambda: hp.copy_(d))))
    print("D2H into pinned + np copy %.1f GB/s" % (gb / t(lambda: hp.copy_(d).numpy().copy())))

    del d
    torch.cuda.empty_cache()
    sizes = [160 << 20] * 17 + [80 << 20] * 16

    def alloc_many():
        xs = [torch.zeros(sz // 8, dtype=torch.float64, device="cuda") for sz in sizes]
        torch.cuda.synchronize()
        del xs
        torch.cuda.empty_cache()
    print("alloc 33 vectors (4.0 GB) zeros: %.3f s" % t(alloc_many, 2))

    def alloc_slab():
        slab = torch.zeros(sum(sizes) // 8, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        del slab
        torch.cuda.empty_cache()
    print("alloc one 4.0 GB slab zeros:     %.3f s" % t(alloc_slab, 2))

    def alloc_empty_slab():
        slab = torch.empty(sum(sizes) // 8, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        del slab
        torch.cuda.empty_cache()
    print("alloc one 4.0 GB slab empty:     %.3f s" % t(alloc_empty_slab, 2))


if __name__ == "__main__":
    main()
