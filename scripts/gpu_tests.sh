#!/bin/bash
# GPU test suite on the box: loopback transports first, the guard-page
# bounds checks, then the rest.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_loopback.py -x -q --durations=5 > gpurun_out/loopback.log 2>&1
python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_loopback.py --durations=10 > gpurun_out/gpu_all.log 2>&1
tail -25 gpurun_out/loopback.log; tail -20 gpurun_out/gpu_all.log
