mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/st2_default.jsonl 2>&1; echo default_rc=$?
TENVEC_B200_FORCE=8 timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/st2_f8.jsonl 2>&1; echo f8 rc=$?
TENVEC_B200_STAGE_BYTES=24576 timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/st2_24k.jsonl 2>&1; echo 24k rc=$?
TENVEC_B200_STAGE_BYTES=40960 timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/st2_40k.jsonl 2>&1; echo 40k rc=$?
