export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 600 python -m pytest tests/test_gpu_multi.py tests/test_gpu_loopback.py -q -p no:cacheprovider 2>&1 | tail -3
