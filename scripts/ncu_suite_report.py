#!/usr/bin/env python
"""Summarise gpurun_out/ncu_suite/*.csv (scripts/gpu_ncu_suite.sh) into a
markdown table: duration, algorithmic bytes and GB/s, DRAM bytes and their
ratio to the algorithmic bytes, DRAM throughput, global-load sector
efficiency (bytes the kernel needs / bytes in the 32-byte sectors it fetched
through L1), occupancy and issue activity."""

from __future__ import annotations

import csv
import glob
import json
import math
import os
import sys

SB = {"f64": 8, "f32": 4, "f32f64": 4, "f16f32": 2, "bf16f32": 2}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9}


def num(v: str) -> float:
    return float(v.replace(",", "")) if v not in ("", "n/a") else float("nan")


def main(out_dir: str = "gpurun_out/ncu_suite") -> None:
    peaks = json.load(open("MEASURED_PEAKS.json"))
    peak = peaks.get("hbm_gbs", 6650.0)
    lines = ["| case | kernel | ms | alg GB | alg GB/s | % of copy peak | DRAM GB | DRAM/alg | DRAM % peak (ncu) | sector eff | warps active % | issue % | regs |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for f in sorted(glob.glob(os.path.join(out_dir, "*.csv"))):
        rows = list(csv.reader(open(f)))
        if len(rows) < 3:
            continue
        hdr, units = rows[0], rows[1]
        idx = {h: i for i, h in enumerate(hdr)}
        for r in rows[2:]:
            case = r[0]
            get = lambda k: num(r[idx[k]]) * UNIT.get(units[idx[k]], 1.0)  # noqa: E731
            t = get("gpu__time_duration.sum")
            dram = get("dram__bytes_read.sum") + get("dram__bytes_write.sum")
            kern = r[idx["Kernel Name"]].split("(")[0].replace("void ", "")
            alg = None
            log = os.path.join(out_dir, f"one_{case}.log")
            if os.path.exists(log):
                shape_s, mode, k, _reg = open(log).read().split()[:4]
                shape = [int(v) for v in shape_s.split(",")]
                k = int(k)
                n = math.prod(shape)
                alg = (n + shape[k] + n // shape[k]) * SB[mode]
            sectors = num(r[idx["l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"]])
            ldgsts = get("sm__sass_l1tex_m_xbar2l1tex_read_bytes_mem_global_op_ldgsts_cache_bypass.sum")
            fetched = sectors * 32 if sectors > 0 else ldgsts
            eff = (alg / fetched) if (alg and fetched and fetched > 0) else float("nan")
            cells = [case, f"`{kern}`", f"{t * 1e3:.3f}",
                     f"{alg / 1e9:.2f}" if alg else "-",
                     f"{alg / t / 1e9:.0f}" if alg else "-",
                     f"{alg / t / 1e9 / peak * 100:.0f}%" if alg else "-",
                     f"{dram / 1e9:.2f}", f"{dram / alg:.3f}" if alg else "-",
                     f"{num(r[idx['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']]):.1f}",
                     "TMA" if "k_staged" in kern else (f"{eff:.2f}" if eff == eff else "-"),
                     f"{num(r[idx['sm__warps_active.avg.pct_of_peak_sustained_active']]):.0f}",
                     f"{num(r[idx['smsp__issue_active.avg.pct_of_peak_sustained_active']]):.0f}",
                     r[idx["launch__registers_per_thread"]]]
            lines.append("| " + " | ".join(cells) + " |")
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:])
