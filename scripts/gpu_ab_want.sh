#!/bin/bash
# A/B: COLS row-phase target (CTAs per SM) over the Table-1 + BASELINE modes
mkdir -p gpurun_out
for w in 4 2 1; do
  TENVEC_B200_COL_WANT=$w timeout 400 python scripts/tvc_modes_bench.py --set all > gpurun_out/want_$w.jsonl 2>&1; echo want$w rc=$?
done
