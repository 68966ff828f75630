mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/modes_${1:-tma}.jsonl 2> gpurun_out/modes_${1:-tma}.err; echo modes_rc=$?
grep '"staged"' gpurun_out/modes_${1:-tma}.jsonl | cut -c1-200
