#!/bin/bash
# A/B of the split-mode reduction's overlap in a dTVC sweep at N GPUs:
# 0 serial, 1 fold + gather on the side stream, 2 the contraction too
mkdir -p gpurun_out/ovl
N=${1:-4}
export CUDA_DEVICE_MAX_CONNECTIONS=32
for wl in c3 c2; do
  for ov in 0 1 2; do
    TENVEC_B200_SWEEP_OVERLAP=$ov timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port $((29600 + ov)) bench.py --gpus $N --workload $wl --steps 20 --warmup 3 \
      --e2e-steps 0 --hopm-workload none > gpurun_out/ovl/${wl}_ov${ov}.json 2> gpurun_out/ovl/${wl}_ov${ov}.err
    python -c "import json; d=json.loads(open('gpurun_out/ovl/${wl}_ov${ov}.json').read().strip().splitlines()[-1]); print('$wl ov$ov', d['value'], d['ms_per_step'], d['parity']['status'])"
  done
done
