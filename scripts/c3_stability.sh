# C3 at N GPUs, three back-to-back runs: plain value, clocks, with-assembly
mkdir -p gpurun_out
N=${1:-4}
export CUDA_DEVICE_MAX_CONNECTIONS=32
for i in 1 2 3; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 2964$i bench.py --gpus $N --workload c3 --steps 10 --warmup 3 --e2e-steps 0 --hopm-workload none \
    > gpurun_out/c3_stab_n${N}_$i.json 2>gpurun_out/c3_stab_n${N}_$i.err
  python -c "import json;d=json.loads(open('gpurun_out/c3_stab_n${N}_$i.json').read().strip().splitlines()[-1]);print($i,d['value'],d['ms_per_step'],d.get('clocks'),{k:(v['ms_per_step'],v.get('path')) for k,v in (d.get('with_assembly') or {}).items()})"
done
