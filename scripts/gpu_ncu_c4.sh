#!/bin/bash
# DRAM bytes of the C4 dHOPM3 full-slab passes (single-pass metrics, no replay)
mkdir -p gpurun_out/ncu_r02
CMD="python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/ncu_r02/c4_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size \
      --clock-control none -k regex:"k_cols" -c 8 --csv --log-file gpurun_out/ncu_r02/dram_c4.csv $CMD > gpurun_out/ncu_r02/dram_c4.log 2>&1
echo rc=$?
