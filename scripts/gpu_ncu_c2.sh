mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/plain_c2.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu_launch_c2.log 2>&1
echo launches_rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_cols|k_rows" -c 3 -o /tmp/prof_c2 $CMD > gpurun_out/ncu_full_c2.log 2>&1
echo full_rc=$?
ncu -i /tmp/prof_c2.ncu-rep --page raw --csv > gpurun_out/raw_c2.csv 2>/dev/null
ncu -i /tmp/prof_c2.ncu-rep --page details --csv > gpurun_out/details_c2.csv 2>/dev/null
ncu -i /tmp/prof_c2.ncu-rep --page source --csv > gpurun_out/source_c2.csv 2>/dev/null
ls -la /tmp/prof_c2.ncu-rep
