mkdir -p gpurun_out
timeout 600 python bench.py --workload c1 --steps 20 --warmup 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo c1_rc=$?
timeout 600 python bench.py --workload c1 --steps 20 --warmup 3 --graph 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c1_eager.json 2> gpurun_out/bench_c1_eager.err; echo c1e_rc=$?
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "graph or sweep" > gpurun_out/pytest_graph.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_graph.log
