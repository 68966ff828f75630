# assembly checks + dTVC with assembly at N GPUs (usage: bash scripts/asm_check.sh N)
mkdir -p gpurun_out
N=${1:-2}
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 600 python -m pytest tests/test_gpu_multi.py tests/test_gpu_loopback.py -q -p no:cacheprovider 2>&1 | tail -3
for wl in c3 c2; do
  for mcast in 1 0; do
    TENVEC_B200_MULTICAST=$mcast timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 2963$mcast bench.py --gpus $N --workload $wl --steps 10 --warmup 3 --e2e-steps 0 --hopm-workload none \
      > gpurun_out/${wl}_asm_n${N}_mc$mcast.json 2>gpurun_out/${wl}_asm_n${N}_mc$mcast.err
    python -c "import json;d=json.loads(open('gpurun_out/${wl}_asm_n${N}_mc$mcast.json').read().strip().splitlines()[-1]);print('$wl mc=$mcast',d['value'],d.get('with_assembly'),d.get('parity',{}).get('status'))"
  done
done
