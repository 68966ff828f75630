mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/ab_default.jsonl 2>&1; echo default_rc=$?
for f in 1 2 3 4 5 6 7 8; do
  TENVEC_B200_FORCE=$f timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/ab_force$f.jsonl 2>&1; echo force$f rc=$?
done
