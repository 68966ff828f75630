mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_gpu.log
timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/jr_final.jsonl 2>&1; echo modes rc=$?
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/jr_c2.json 2> gpurun_out/jr_c2.err; echo c2 rc=$?
timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 > gpurun_out/jr_c4.json 2> gpurun_out/jr_c4.err; echo c4 rc=$?
