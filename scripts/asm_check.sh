mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 600 python -m pytest tests/test_gpu_loopback.py tests/test_acceptance_b200.py -q -p no:cacheprovider -k "loopback or a10 or a01" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_hopm.py -q -p no:cacheprovider -k "assembl or repack or undistrib" 2>&1 | tail -2
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 2 --workload c3 --steps 10 --warmup 3 --e2e-steps 0 > gpurun_out/c3_asm_n2.json 2>gpurun_out/c3_asm_n2.err
python -c "import json;d=json.loads(open('gpurun_out/c3_asm_n2.json').read().strip().splitlines()[-1]);print(d['value'],d.get('with_assembly'),d.get('parity'))"
