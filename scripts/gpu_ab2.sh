mkdir -p gpurun_out; rm -f gpurun_out/ab_*.jsonl
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/ab_default.jsonl 2>&1; echo default_rc=$?
for f in $FORCES; do
  TENVEC_B200_FORCE=$f timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/ab_force$f.jsonl 2>&1; echo force$f rc=$?
done
