#!/bin/bash
# tall views after a change: the probe, then the split-K / tvc parity tests
mkdir -p gpurun_out/tall
timeout 300 python scripts/tall_probe.py > gpurun_out/tall/after.jsonl 2>&1; echo probe_rc=$?
cat gpurun_out/tall/after.jsonl
timeout 900 python -m pytest tests/test_gpu_tvc.py tests/test_gpu_tvc_norm.py -q -p no:cacheprovider 2>&1 | tail -2
