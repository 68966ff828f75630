mkdir -p gpurun_out
N=${1:-4}
for r in 1 2; do
for L in 1 2 4; do
  TENVEC_B200_OWNER_LANES=$L timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2995 bench.py --gpus $N --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/lanes${L}_$r.json 2>/dev/null; echo L$L rc=$?
done
done
