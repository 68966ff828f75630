mkdir -p gpurun_out
N=${1:-4}
for cfg in "0 1" "1 1" "1 0" "0 0"; do
  set -- $cfg
  TENVEC_B200_SWEEP_OVERLAP=$1 TENVEC_B200_SIDE_PRIORITY=$2 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2977 bench.py --gpus $N --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/prio_ov$1_p$2.json 2> gpurun_out/prio_ov$1_p$2.err; echo ov$1 p$2 rc=$?
  TENVEC_B200_SWEEP_OVERLAP=$1 TENVEC_B200_SIDE_PRIORITY=$2 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2978 bench.py --gpus $N --workload c3 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/prio3_ov$1_p$2.json 2> gpurun_out/prio3_ov$1_p$2.err; echo c3 ov$1 p$2 rc=$?
done
