mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -15 gpurun_out/pytest_gpu.log
timeout 900 python scripts/tvc_modes_bench.py --set all > gpurun_out/modes_all.jsonl 2> gpurun_out/modes_all.err; echo modes_rc=$?
TENVEC_B200_STAGED=0 timeout 900 python scripts/tvc_modes_bench.py --set baseline > gpurun_out/modes_nostaged.jsonl 2> gpurun_out/modes_nostaged.err; echo modes2_rc=$?
