mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/lg_default.jsonl 2>&1; echo default rc=$?
TENVEC_B200_FORCE=11 timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/lg_f11.jsonl 2>&1; echo f11 rc=$?
