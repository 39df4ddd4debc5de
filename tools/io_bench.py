"""Problem-file read time: native reader vs the json module.

    python tools/io_bench.py [m] [n]     (default the C5 shape at 1/10: m=1M, n=2M, 5M nnz)
"""

import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(m, n):
    from paper_2603_15504_b200 import fileio, instances

    p = instances.lp_large(m=m, n=n, nnz_per_row=5, eq_frac=0.3, seed=5)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "p.json")
        t0 = time.perf_counter()
        fileio.serialize_problem(p, path)
        tw = time.perf_counter() - t0
        size = os.path.getsize(path)
        t0 = time.perf_counter()
        a = fileio.parse_problem(path)
        tf = time.perf_counter() - t0
        t0 = time.perf_counter()
        b = fileio.parse_problem(path, fast=False)
        tj = time.perf_counter() - t0
        assert (a.G.to_scipy() != b.G.to_scipy()).nnz == 0
    print(f"m={m} n={n} nnz={p.G.nnz} file {size / 1e6:.0f} MB: write {tw:.1f} s, "
          f"native read {tf:.2f} s ({size / tf / 1e9:.2f} GB/s, {os.cpu_count()} threads), "
          f"json read {tj:.1f} s -> {tj / tf:.1f}x")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000, int(sys.argv[2]) if len(sys.argv) > 2 else 2_000_000)
