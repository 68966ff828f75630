#!/bin/bash
# A/B of the split-mode reduction transport in a dTVC sweep at N GPUs
mkdir -p gpurun_out/tr
N=${1:-4}
export CUDA_DEVICE_MAX_CONNECTIONS=32
for wl in c3 c2; do
  for algo in fused ce exact; do
    TENVEC_B200_ALLREDUCE=$algo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port 29640 bench.py --gpus $N --workload $wl --steps 20 --warmup 3 \
      --e2e-steps 0 --hopm-workload none > gpurun_out/tr/${wl}_${algo}_n$N.json 2> gpurun_out/tr/${wl}_${algo}_n$N.err
    python -c "import json; d=json.loads(open('gpurun_out/tr/${wl}_${algo}_n$N.json').read().strip().splitlines()[-1]); print('$wl $algo', d['value'], d['ms_per_step'], d['parity']['status'])" || tail -3 gpurun_out/tr/${wl}_${algo}_n$N.err
  done
done
