# multi-GPU validation + every bench line at N GPUs (current code)
mkdir -p gpurun_out/multi
N=${1:-2}
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/multi/pytest_$N.log 2>&1; echo pytest_multi_rc=$?; tail -1 gpurun_out/multi/pytest_$N.log
port=2960
for w in c2 c3 c4 c5; do
  port=$((port+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --workload $w --steps 10 --warmup 3 --e2e-steps 1 > gpurun_out/multi/${w}_n$N.json 2> gpurun_out/multi/${w}_n$N.err; echo ${w}_rc=$?
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2969 bench.py --gpus $N --impl reference --steps 3 > gpurun_out/multi/ref_n$N.json 2> gpurun_out/multi/ref_n$N.err; echo ref_rc=$?
