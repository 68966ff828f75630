#!/bin/bash
# ncu --set full of the round-2 kernels: double-buffered COLS_U (paper d = 2 k = 0)
# and STAGED_TALL ([8, 1e6, 12] bf16, [3000001, 7] fp64)
mkdir -p gpurun_out/ncu_new
cap() {  # name regex args...
  local name=$1 rx=$2; shift 2
  python scripts/one_view.py "$@" > /dev/null 2>&1 || { echo "$name: run failed"; return; }
  ncu --set full --clock-control none --import-source on -k regex:$rx -s 2 -c 1 -o gpurun_out/ncu_new/$name -f \
    python scripts/one_view.py "$@" > gpurun_out/ncu_new/$name.log 2>&1
  ncu -i gpurun_out/ncu_new/$name.ncu-rep --page raw --csv > gpurun_out/ncu_new/$name.raw.csv 2>&1
  echo "$name rc=$?"
}
cap colsu_d2 k_cols 30623,30623 0 f64
cap tall_bf16 k_staged_tall 8,1000000,12 1 bf16f32
cap tall_f64 k_staged_tall 3000001,7 0 f64
rm -f gpurun_out/ncu_new/*.ncu-rep
