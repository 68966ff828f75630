mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tvc.py -x -q -p no:cacheprovider -k "cols_sh or cols_u" > gpurun_out/pytest_sh.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pytest_sh.log
TENVEC_B200_FORCE=12 timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/sh_f12.jsonl 2>&1; echo f12 rc=$?
