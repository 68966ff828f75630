mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python scripts/tvc_modes_bench.py --set all > gpurun_out/modes_all.jsonl 2> gpurun_out/modes_all.err; echo modes_rc=$?
for w in c2 c3 c1; do timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w rc=$?; done
