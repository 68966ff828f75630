mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pytest_gpu.log
timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/st5_default.jsonl 2>&1; echo default rc=$?
TENVEC_B200_STAGE_BYTES=40960 timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/st5_40k.jsonl 2>&1; echo 40k rc=$?
timeout 600 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo bench_rc=$?
