#!/bin/bash
# launch list (per-kernel durations, DRAM bytes) of scripts/tall_probe.py
mkdir -p gpurun_out/tall
python scripts/tall_probe.py > gpurun_out/tall/probe.jsonl 2>&1; echo probe_rc=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size \
  --clock-control none -c 2000 --csv --log-file gpurun_out/tall/launches.csv python scripts/tall_probe.py > gpurun_out/tall/ncu.log 2>&1; echo ncu_rc=$?
cat gpurun_out/tall/probe.jsonl
