#!/usr/bin/env python
"""Summarise the full-size C2 ncu capture (scripts/gpu_ncu_c2.sh ->
gpurun_out/raw_c2.csv) into profiles/r01_ncu_full_c2_2048cubed.json (one
record per captured launch) and profiles/ncu_traffic.json (DRAM bytes per
launch of tv_tvc k = 0, 1, 2: the `traffic` field of bench.py's roofline).

    python scripts/ncu_c2_summary.py [gpurun_out/raw_c2.csv]
"""

from __future__ import annotations

import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_sectors_srcunit_tex_op_read.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main(path: str = os.path.join(ROOT, "gpurun_out", "raw_c2.csv")) -> int:
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    recs = []
    for r in rows[2:]:
        rec = {"kernel": r[idx["Kernel Name"]].split("(")[0]}
        for k in KEYS:
            if k in idx:
                rec[k] = f"{r[idx[k]]} {units[idx[k]]}".strip()
        total = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            total += float(r[idx[k]].replace(",", "")) * SCALE.get(units[idx[k]], 1.0)
        rec["dram_bytes_total"] = total
        recs.append(rec)
    with open(os.path.join(ROOT, "profiles", "r01_ncu_full_c2_2048cubed.json"), "w") as fh:
        json.dump(recs, fh, indent=1)
    # the three sweep launches, in launch order k = 0, 1, 2
    traffic = {"c2": {f"k{k}": int(recs[k]["dram_bytes_total"]) for k in range(min(3, len(recs)))},
               "_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch of tv_tvc k=0,1,2 on the "
                        "full C2 2048^3 fp64 tensor, one ncu --set full capture "
                        "(profiles/r01_ncu_full_c2_2048cubed.json)"}
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as fh:
        json.dump(traffic, fh, indent=1)
    print(json.dumps(traffic))
    return 0


if __name__ == "__main__":
    sys.exit(main(*sys.argv[1:]))
