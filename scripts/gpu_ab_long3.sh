mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tvc.py -x -q -p no:cacheprovider -k staged_long > gpurun_out/pytest_long.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pytest_long.log
TENVEC_B200_FORCE=11 timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/lg3_f11.jsonl 2>&1; echo f11 rc=$?
