# multi-GPU: the fused TVC + peer-memory reduction vs the NCCL exact path
mkdir -p gpurun_out
N=${1:-2}
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/pytest_multi_$N.log 2>&1; echo pytest_multi_rc=$?; tail -5 gpurun_out/pytest_multi_$N.log
for algo in exact fused; do
  for wl in c2 c3; do
    TENVEC_B200_ALLREDUCE=$algo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --workload $wl --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/fab_${wl}_${algo}_n$N.json 2> gpurun_out/fab_${wl}_${algo}_n$N.err; echo ${wl}_${algo}_rc=$?
  done
done
