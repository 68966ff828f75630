mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python scripts/tvc_modes_bench.py --set all > gpurun_out/modes_all.jsonl 2> gpurun_out/modes_all.err; echo modes_rc=$?
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 5 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo ref_rc=$?
for w in c3 c4 c5; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w rc=$?; done
