mkdir -p gpurun_out
for jr in 0 1 2 4 8; do
  TENVEC_B200_COL_JR=$jr timeout 300 python scripts/tvc_modes_bench.py --set baseline > gpurun_out/jr_$jr.jsonl 2>&1; echo jr$jr rc=$?
done
