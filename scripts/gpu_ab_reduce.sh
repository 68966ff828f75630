mkdir -p gpurun_out
N=${1:-4}
P=29800
run() { P=$((P+1)); timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N "$@"; }
for algo in exact p2p; do
  for ov in 0 1; do
    TENVEC_B200_ALLREDUCE=$algo TENVEC_B200_SWEEP_OVERLAP=$ov run --workload c3 --steps 10 --warmup 3 --e2e-steps 0 > gpurun_out/ab_c3_${algo}_ov$ov.json 2>&1; echo c3 $algo ov$ov rc=$?
    TENVEC_B200_ALLREDUCE=$algo TENVEC_B200_SWEEP_OVERLAP=$ov run --workload c2 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab_c2_${algo}_ov$ov.json 2>&1; echo c2 $algo ov$ov rc=$?
  done
done
