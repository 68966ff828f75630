mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tvc.py -x -q -p no:cacheprovider > gpurun_out/pytest_tvc.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pytest_tvc.log
timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/xs_default.jsonl 2>&1; echo modes rc=$?
