mkdir -p gpurun_out
N=${1:-4}
nvidia-smi -L | head -8; free -g | head -2
timeout 600 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/pytest_multi_$N.log 2>&1; echo pytest_multi_rc=$?; tail -3 gpurun_out/pytest_multi_$N.log
P=29600
run() { P=$((P+1)); timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N "$@"; }
run --steps 10 --warmup 3 --e2e-steps 1 > gpurun_out/bench_c2_n$N.json 2> gpurun_out/bench_c2_n$N.err; echo c2 rc=$?
TENVEC_B200_SWEEP_OVERLAP=1 run --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_c2_n${N}_ov1.json 2>&1; echo c2ov1 rc=$?
run --workload c3 --steps 10 --warmup 3 --e2e-steps 0 > gpurun_out/bench_c3_n$N.json 2> gpurun_out/bench_c3_n$N.err; echo c3 rc=$?
TENVEC_B200_SWEEP_OVERLAP=0 run --workload c3 --steps 10 --warmup 3 --e2e-steps 0 > gpurun_out/bench_c3_n${N}_ov0.json 2>&1; echo c3ov0 rc=$?
run --workload c4 --steps 5 --warmup 3 > gpurun_out/bench_c4_n$N.json 2> gpurun_out/bench_c4_n$N.err; echo c4 rc=$?
run --workload c5 --steps 5 --warmup 3 > gpurun_out/bench_c5_n$N.json 2> gpurun_out/bench_c5_n$N.err; echo c5 rc=$?
