#!/bin/bash
mkdir -p gpurun_out/ncu_r02k
CMD="python scripts/ncu_r02_kernels.py"
$CMD > gpurun_out/ncu_r02k/plain.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_rows|k_flat_u|k_repack|k_fold" -c 8 \
      -o /tmp/prof_r02k $CMD > gpurun_out/ncu_r02k/full.log 2>&1
echo rc=$?
ncu -i /tmp/prof_r02k.ncu-rep --page raw --csv > gpurun_out/ncu_r02k/raw.csv 2>/dev/null
ncu -i /tmp/prof_r02k.ncu-rep --page details --csv > gpurun_out/ncu_r02k/details.csv 2>/dev/null
