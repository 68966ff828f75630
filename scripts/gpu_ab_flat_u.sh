#!/bin/bash
# tall narrow views: FLAT_U (flat 16-byte runs) vs SLABS / SLABS_U, bf16 and f16 included
mkdir -p gpurun_out/flatu
for fu in 1 0; do
  TENVEC_B200_FLAT_U=$fu timeout 300 python scripts/tall_probe.py > gpurun_out/flatu/tall_fu$fu.jsonl 2>&1
done
