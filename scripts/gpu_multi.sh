#!/bin/bash
# N-GPU round: NCCL transport tests, then the bench legs at N (C2 + its C4
# dHOPM3 leg, C3, C5) and the reference arm.  Usage: gpurun --gpus N -- bash scripts/gpu_multi.sh N
mkdir -p gpurun_out
N=${1:-2}
nvidia-smi -L; free -g | head -2
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/pytest_multi_$N.log 2>&1; echo pytest_multi_rc=$?; tail -5 gpurun_out/pytest_multi_$N.log
run() {  # name port args...
  local name=$1 port=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus $N "$@" > gpurun_out/bench_${name}_n$N.json 2> gpurun_out/bench_${name}_n$N.err
  echo ${name}_rc=$?
}
run c2 29511 --steps 10 --warmup 3 --e2e-steps 1
run c3 29513 --workload c3 --steps 10 --warmup 3 --e2e-steps 0
run c5 29515 --workload c5 --steps 5 --warmup 3
run ref 29514 --impl reference --steps 3
