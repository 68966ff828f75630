#!/usr/bin/env python
"""Summarise the round-2 ncu files (scripts/gpu_ncu_r02.sh -> gpurun_out/ncu_r02/)
into profiles/r02_ncu/: the launch list of the default bench command (kernel
shares of the run), DRAM bytes per launch of the TVC kernels against their
algorithmic bytes, and the --set full capture of the C2 kernels.

    python scripts/ncu_r02_summary.py
"""

from __future__ import annotations

import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "ncu_r02")
DST = os.path.join(ROOT, "profiles", "r02_ncu")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1.0, "%": 1.0, "": 1.0, "register/thread": 1.0, "block": 1.0}


def read_long(path: str) -> list[dict]:
    """ncu --csv --log-file (one row per metric) -> one dict per launch."""
    lines = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    out: dict = collections.OrderedDict()
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        rec = out.setdefault(d["ID"], {"id": int(d["ID"]), "kernel": d["Kernel Name"], "grid": d["Grid Size"],
                                        "block": d["Block Size"]})
        try:
            val = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
        except ValueError:
            val = d["Metric Value"]
        rec[d["Metric Name"]] = val
    return list(out.values())


def short(name: str) -> str:
    name = name.split("(")[0]
    return name.replace("void ", "").replace("tv::", "")


def main() -> int:
    os.makedirs(DST, exist_ok=True)
    summary = {}
    # 1. launch list: time share per kernel (serialised, cold cache)
    launches = read_long(os.path.join(SRC, "launches_default.csv"))
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in launches:
        tot[short(r["kernel"])] += r.get("gpu__time_duration.sum", 0.0)
        cnt[short(r["kernel"])] += 1
    all_t = sum(tot.values())
    # the share among the contraction work: without the bench's own spin
    # kernels (the ~0.5 s hold before each timed loop, the nvbench-style
    # blocking kernel before each per-mode timing) and the one-off tensor fill
    setup = ("spin_kernel", "k_fill", "k_read_stream")
    work_t = sum(t for k, t in tot.items() if not any(x in k for x in setup))
    summary["launch_list_default"] = {
        "command": "python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline (C2 sweep + C4 dHOPM3 leg)",
        "launches": len(launches),
        "note": "share = of all GPU time under ncu (serialised); share_of_work excludes the bench's spin "
                "kernels (hold / blocking kernel, outside every timed event pair), the one-off fill and the "
                "read-stream probe",
        "kernels": [{"kernel": k, "launches": cnt[k], "ms": round(t * 1e3, 3), "share": round(t / all_t, 4),
                     **({} if any(x in k for x in setup) else {"share_of_work": round(t / work_t, 4)})}
                    for k, t in tot.most_common()]}
    # 2. DRAM bytes per TVC launch vs the algorithmic bytes of the view
    dram = read_long(os.path.join(SRC, "dram_default.csv"))
    recs = []
    for r in dram:
        b = r.get("dram__bytes_read.sum", 0.0) + r.get("dram__bytes_write.sum", 0.0)
        t = r.get("gpu__time_duration.sum", 0.0)
        recs.append({"kernel": short(r["kernel"]), "grid": r["grid"], "ms": round(t * 1e3, 4),
                     "dram_gb": round(b / 1e9, 4), "dram_gbs": round(b / t / 1e9, 1) if t else None,
                     "dram_pct_peak": r.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                     "regs": r.get("launch__registers_per_thread")})
    # the C2 launches: 68.75 GB of algorithmic bytes each (2048^3 fp64 + x + out)
    alg_c2 = (2048 ** 3 + 2048 + 2048 ** 2) * 8
    c2 = [x for x in recs if abs(x["dram_gb"] * 1e9 - alg_c2) / alg_c2 < 0.01]
    summary["dram_per_launch"] = {
        "command": "same, -k regex:'k_cols|k_rows', single-pass metrics",
        "c2_launches": len(c2), "c2_alg_bytes": alg_c2,
        "c2_dram_over_alg": [round(x["dram_gb"] * 1e9 / alg_c2, 5) for x in c2],
        "c2_dram_pct_peak": [x["dram_pct_peak"] for x in c2],
        "launches": recs}
    # 3. the full capture of the C2 kernels
    raw = os.path.join(SRC, "raw_c2.csv")
    if os.path.exists(raw):
        rows = list(csv.reader(open(raw)))
        hdr, units = rows[0], rows[1]
        keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
                "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
                "lts__t_sector_hit_rate.pct"]
        full = []
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            full.append({"kernel": short(d["Kernel Name"]),
                         **{k: f"{d.get(k, '')} {units[hdr.index(k)] if k in hdr else ''}".strip() for k in keys}})
        summary["full_c2"] = full
    # 4. C1: the PDL-chained sweep's kernels (serialised under ncu)
    c1 = read_long(os.path.join(SRC, "launches_c1.csv"))
    alg_c1 = (256 ** 3 + 256 + 256 ** 2) * 8
    tvc = [r for r in c1 if "k_cols" in r["kernel"] or "k_rows" in r["kernel"]]
    summary["c1_tvc_launches"] = {
        "alg_bytes": alg_c1,
        "launches": [{"kernel": short(r["kernel"]), "grid": r["grid"],
                      "us": round(r.get("gpu__time_duration.sum", 0) * 1e6, 2),
                      "dram_over_alg": round((r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0))
                                             / alg_c1, 4)} for r in tvc[-9:]]}
    with open(os.path.join(DST, "summary.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps({k: (v if k != "dram_per_launch" else {kk: vv for kk, vv in v.items() if kk != "launches"})
                      for k, v in summary.items() if k != "full_c2"}, indent=1)[:4000])
    for f in summary.get("full_c2", []):
        print(f)
    return 0


if __name__ == "__main__":
    sys.exit(main())
