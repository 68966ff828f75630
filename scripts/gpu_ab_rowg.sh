mkdir -p gpurun_out
for g in 0 8 16 32; do
  TENVEC_B200_ROW_G=$g timeout 300 python scripts/tvc_modes_bench.py --set baseline > gpurun_out/rowg_$g.jsonl 2>&1; echo g$g rc=$?
done
