mkdir -p gpurun_out
timeout 600 python scripts/tvc_modes_bench.py --set table1 > gpurun_out/lg2_default.jsonl 2>&1; echo default rc=$?
TENVEC_B200_FORCE=11 timeout 600 python scripts/tvc_modes_bench.py --set table1 > gpurun_out/lg2_f11.jsonl 2>&1; echo f11 rc=$?
