#!/bin/bash
# End-of-round ncu evidence for the default bench command with the final code
# (parts 1, 2 and 4 of gpu_ncu_r02.sh; the C2 kernels' --set full capture is
# unchanged since their code is): launch list, DRAM bytes per TVC launch, C1.
mkdir -p gpurun_out/ncu_r02
CMD="python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/ncu_r02/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv \
      --log-file gpurun_out/ncu_r02/launches_default.csv $CMD > gpurun_out/ncu_r02/launches.log 2>&1
echo launches_rc=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__registers_per_thread \
    --clock-control none -k regex:"k_cols|k_rows" -c 40 --csv --log-file gpurun_out/ncu_r02/dram_default.csv \
    $CMD > gpurun_out/ncu_r02/dram.log 2>&1
echo dram_rc=$?
C1="python bench.py --workload c1 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$C1 > gpurun_out/ncu_r02/plain_c1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
      --log-file gpurun_out/ncu_r02/launches_c1.csv $C1 > gpurun_out/ncu_r02/launches_c1.log 2>&1
echo c1_rc=$?
