"""Per-kernel table of an ncu launch list (the format of profiles/r01_kernels_C1-C5.txt).

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none \
        --launch-skip S --launch-count K --csv --log-file gpurun_out/k_C1.csv \
        python bench.py --config C1 --steps 400 --warmup 5 --no-cpu-baseline --no-e2e
    python tools/kernel_table.py gpurun_out/k_C1.csv C1

prints "## C1" and one line per kernel: launches, mean us, mean MB of DRAM
traffic, GB/s and mean active-warp occupancy.
"""

import csv
import sys
from collections import defaultdict

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
        "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "%": 1.0}


def main(path, config):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    iid, ik, im, iu, iv = (h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"),
                           h.index("Metric Unit"), h.index("Metric Value"))
    per = defaultdict(dict)  # launch id -> {name, metrics}
    for r in rows[1:]:
        try:
            v = float(r[iv].replace(",", "")) * UNIT.get(r[iu], 1.0)
        except ValueError:
            continue
        d = per[r[iid]]
        d["name"] = r[ik].split("(")[0].replace("void ", "").replace("pdcs::", "")
        d[r[im]] = v
    agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    order = []
    for d in per.values():
        a = agg[d["name"]]
        if a[0] == 0:
            order.append(d["name"])
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        a[3] += d.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0.0)
    print(f"## {config}")
    print(f"{'kernel':<40}{'n':>3}{'us/launch':>11}{'MB/launch':>11}{'GB/s':>10}{'occ%':>7}")
    for k in order:
        n, t, b, o = agg[k]
        print(f"{k[:39]:<40}{n:>3}{t / n * 1e6:>11.1f}{b / n / 1e6:>11.2f}"
              f"{(b / t / 1e9 if t else 0):>10.0f}{o / n:>7.0f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
