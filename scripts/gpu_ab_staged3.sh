mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "regime or staged or tvc" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
for cfg in 2:32768 2:40960 2:49152 3:24576 3:32768 4:16384 4:24576; do
  n=${cfg%%:*}; b=${cfg##*:}
  TENVEC_B200_STAGES=$n TENVEC_B200_STAGE_BYTES=$b timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/st3_${n}x${b}.jsonl 2>&1; echo $cfg rc=$?
done
