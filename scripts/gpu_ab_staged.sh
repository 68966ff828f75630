mkdir -p gpurun_out
timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/st_default.jsonl 2>&1; echo default_rc=$?
TENVEC_B200_FORCE=8 timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/st_f8_16k.jsonl 2>&1; echo f8_16k rc=$?
TENVEC_B200_FORCE=8 TENVEC_B200_STAGE_BYTES=32768 timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/st_f8_32k.jsonl 2>&1; echo f8_32k rc=$?
TENVEC_B200_FORCE=8 TENVEC_B200_STAGE_BYTES=65536 timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/st_f8_64k.jsonl 2>&1; echo f8_64k rc=$?
TENVEC_B200_STAGE_ROW=8192 timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/st_row8k.jsonl 2>&1; echo row8k rc=$?
TENVEC_B200_STAGE_ROW=16384 TENVEC_B200_STAGE_BYTES=32768 timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/st_row16k_32k.jsonl 2>&1; echo row16k rc=$?
