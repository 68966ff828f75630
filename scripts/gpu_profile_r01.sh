CMD="python bench.py --shape 1024,1024,1024 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/plain_c2s.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2s.csv $CMD > gpurun_out/ncu_launch_c2s.log 2>&1
echo launches_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_cols|k_rows" -c 3 -o gpurun_out/prof_c2s $CMD > gpurun_out/ncu_full_c2s.log 2>&1
echo full_rc=$?
for w in c3 c1; do timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w rc=$?; done
for w in c5 c4; do timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w rc=$?; done
timeout 600 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_c2_read.json 2>&1; echo c2 rc=$?
