mkdir -p gpurun_out
N=${1:-2}
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/pytest_multi_$N.log 2>&1; echo pytest_multi_rc=$?; tail -3 gpurun_out/pytest_multi_$N.log
for w in c4 c5; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N --workload $w --steps 5 --warmup 3 > gpurun_out/bench_${w}_n$N.json 2> gpurun_out/bench_${w}_n$N.err; echo bench_${w}_rc=$?
done
