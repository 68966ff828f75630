#!/bin/bash
# C2 at N GPUs: step-time outliers with and without the nvidia-smi sampler (A/B only)
mkdir -p gpurun_out/clk
N=${1:-4}
export CUDA_DEVICE_MAX_CONNECTIONS=32
for i in 1; do
for nc in 0 1; do
  if [ $nc = 1 ]; then export TENVEC_BENCH_NO_CLOCKS=1; else unset TENVEC_BENCH_NO_CLOCKS; fi
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2970$nc \
    bench.py --gpus $N --steps 20 --warmup 3 --e2e-steps 0 --hopm-workload none > gpurun_out/clk/c2_nc${nc}_$i.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/clk/c2_nc${nc}_$i.json').read().strip().splitlines()[-1])
print('noclk=$nc run $i', d['value'], d['ms_per_step'], max(d['step_ms_rank0']), sorted(d['step_ms_rank0'])[-3:])"
done
done
