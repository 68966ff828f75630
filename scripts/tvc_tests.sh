#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_tvc.py tests/test_gpu_guards.py tests/test_acceptance_b200.py tests/test_gpu_tvc_norm.py -q -p no:cacheprovider 2>&1 | tail -4
