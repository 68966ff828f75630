#!/bin/bash
# C3 (96^5 fp32) sweep kernels at N = 1: single-pass DRAM metrics for every mode,
# then one --set full capture of the COLS launches (k = 0, 1)
mkdir -p gpurun_out/ncu_c3
CMD="python bench.py --workload c3 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/ncu_c3/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size \
      --clock-control none -k regex:"k_cols|k_staged|k_flat|k_rows" -c 10 --csv --log-file gpurun_out/ncu_c3/metrics.csv $CMD \
      > gpurun_out/ncu_c3/metrics.log 2>&1
echo metrics_rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_cols" -c 2 -o /tmp/prof_c3 $CMD \
    > gpurun_out/ncu_c3/full.log 2>&1
echo full_rc=$?
ncu -i /tmp/prof_c3.ncu-rep --page raw --csv > gpurun_out/ncu_c3/raw.csv 2>/dev/null
ncu -i /tmp/prof_c3.ncu-rep --page details --csv > gpurun_out/ncu_c3/details.csv 2>/dev/null
ncu -i /tmp/prof_c3.ncu-rep --page source --csv > gpurun_out/ncu_c3/source.csv 2>/dev/null
ls -la gpurun_out/ncu_c3
