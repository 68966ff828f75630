#!/bin/bash
mkdir -p gpurun_out/ncu_tall
python scripts/one_view.py 8,1000000,12 1 bf16f32 && \
ncu --set full --clock-control none --import-source on -k regex:k_staged_tall -s 2 -c 1 -o gpurun_out/ncu_tall/st_bf16 -f \
  python scripts/one_view.py 8,1000000,12 1 bf16f32 > gpurun_out/ncu_tall/log.txt 2>&1; echo rc=$?
ncu -i gpurun_out/ncu_tall/st_bf16.ncu-rep --page raw --csv > gpurun_out/ncu_tall/raw.csv 2>&1
ncu -i gpurun_out/ncu_tall/st_bf16.ncu-rep --page source --csv > gpurun_out/ncu_tall/source.csv 2>&1
ls -la gpurun_out/ncu_tall
