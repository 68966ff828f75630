mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python scripts/tvc_modes_bench.py --set ${1:-baseline} > gpurun_out/modes_quick.jsonl 2> gpurun_out/modes_quick.err; echo modes_rc=$?
timeout 600 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo bench_rc=$?
