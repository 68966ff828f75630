# C3 (and C2) dTVC with assembly at N=4 after the push-based interleave
mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
for wl in c3 c2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2962${#wl} bench.py --gpus 4 --workload $wl --steps 10 --warmup 3 --e2e-steps 0 --hopm-workload none > gpurun_out/${wl}_asm_n4.json 2>gpurun_out/${wl}_asm_n4.err
python -c "import json;d=json.loads(open('gpurun_out/${wl}_asm_n4.json').read().strip().splitlines()[-1]);print('$wl',d['value'],d.get('with_assembly'),d.get('parity',{}).get('status'),d.get('clocks'))"
done
