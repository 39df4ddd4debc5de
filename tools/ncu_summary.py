"""Summarise an `ncu --set full` capture of bench.py into profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep C5 r01

writes profiles/<round>_<config>_ncu_full.txt (per kernel: duration, DRAM
bytes, throughput, hit rates, occupancy) and profiles/traffic_<config>.json
(DRAM bytes read + write per launch of each bench stage, the `traffic` field
of bench.py's roofline).
"""

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

STAGE_OF = {  # final kernel name prefix -> bench stage (pdcs_profile_slot names)
    "k_step_x": "step_x",
    "k_step_y": "step_y_spmv",
    "k_step_t": "step_t_spmv",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size"]


def main(rep, config, rnd):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {k: hdr.index(k) for k in KEYS + ["Kernel Name"] if k in hdr}
    lines = [f"# ncu --set full --clock-control none: {rep} ({config})\n"]
    # a stage's traffic per launch: the final kernel of a step SpMV plus the
    # partial-sum passes (k_lane_pass / k_tile_pass) launched just before it
    per_stage = defaultdict(list)
    pending = []
    for r in rows[2:]:
        name = r[idx["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
        lines.append(f"{name}\n")
        for k in KEYS:
            if k in idx:
                lines.append(f"  {k} = {r[idx[k]]} {units[idx[k]]}\n")
        rd = float(r[idx["dram__bytes_read.sum"]]) * UNIT.get(units[idx["dram__bytes_read.sum"]], 1)
        wr = float(r[idx["dram__bytes_write.sum"]]) * UNIT.get(units[idx["dram__bytes_write.sum"]], 1)
        lines.append(f"  dram read+write = {(rd + wr) / 1e9:.3f} GB\n")
        if short in ("k_lane_pass", "k_tile_pass"):
            pending.append(rd + wr)
            continue
        for prefix, stage in STAGE_OF.items():
            if short.startswith(prefix):
                extra = sum(pending) if stage != "step_x" else 0.0
                per_stage[stage].append(rd + wr + extra)
                pending = []
                break
    stages = {stage: sum(v) / len(v) for stage, v in per_stage.items()}
    os.makedirs("profiles", exist_ok=True)
    with open(f"profiles/{rnd}_{config}_ncu_full.txt", "w") as f:
        f.writelines(lines)
    with open(f"profiles/traffic_{config}.json", "w") as f:
        json.dump({"source": os.path.basename(rep), "stages": dict(stages),
                   "note": "DRAM bytes (read + write) per launch from one ncu --set full capture"},
                  f, indent=1)
    print("".join(lines))
    print(dict(stages))


if __name__ == "__main__":
    main(*sys.argv[1:4])
