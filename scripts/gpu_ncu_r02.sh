#!/bin/bash
# Round-2 ncu evidence for the default bench command (C2 sweep + C4 dHOPM3 leg):
#  1. the launch list (gpu__time_duration, cold-cache serialised launches)
#  2. DRAM bytes + duration of every k_cols / k_rows launch (single-pass metrics,
#     no replay of the 174 GB C4 tensor)
#  3. one --set full capture of the C2 kernels (k = 0, 1, 2)
#  4. the C1 sweep (PDL-chained, serialised under ncu) launch list
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
C2="python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --hopm-workload none"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_cols|k_rows" -c 3 -o /tmp/prof_c2 $C2 \
    > gpurun_out/ncu_r02/full_c2.log 2>&1
echo full_rc=$?
ncu -i /tmp/prof_c2.ncu-rep --page raw --csv > gpurun_out/ncu_r02/raw_c2.csv 2>/dev/null
ncu -i /tmp/prof_c2.ncu-rep --page details --csv > gpurun_out/ncu_r02/details_c2.csv 2>/dev/null
C1="python bench.py --workload c1 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$C1 > gpurun_out/ncu_r02/plain_c1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
      --log-file gpurun_out/ncu_r02/launches_c1.csv $C1 > gpurun_out/ncu_r02/launches_c1.log 2>&1
echo c1_rc=$?
ls -la gpurun_out/ncu_r02
