mkdir -p gpurun_out
N=${1:-4}
for ov in 0 1; do
  TENVEC_B200_SWEEP_OVERLAP=$ov timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2971 bench.py --gpus $N --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ovl${ov}_c2_n$N.json 2> gpurun_out/ovl${ov}_c2_n$N.err; echo ov$ov rc=$?
done
