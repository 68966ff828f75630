mkdir -p gpurun_out
N=${1:-2}
nvidia-smi -L; free -g | head -2
timeout 600 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/pytest_multi_$N.log 2>&1; echo pytest_multi_rc=$?; tail -5 gpurun_out/pytest_multi_$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 10 --warmup 3 --e2e-steps 1 > gpurun_out/bench_c2_n$N.json 2> gpurun_out/bench_c2_n$N.err; echo bench_c2_rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --workload c4 --steps 5 --warmup 3 > gpurun_out/bench_c4_n$N.json 2> gpurun_out/bench_c4_n$N.err; echo bench_c4_rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --workload c3 --steps 10 --warmup 3 --e2e-steps 0 > gpurun_out/bench_c3_n$N.json 2> gpurun_out/bench_c3_n$N.err; echo bench_c3_rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus $N --impl reference --steps 3 > gpurun_out/bench_ref_n$N.json 2> gpurun_out/bench_ref_n$N.err; echo ref_rc=$?
