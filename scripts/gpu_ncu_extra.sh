# one ncu --set full capture per kernel regime on representative views (final code)
mkdir -p gpurun_out/ncu_suite
KEYS='Kernel Name|gpu__time_duration.sum|dram__bytes_read.sum|dram__bytes_write.sum|gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed|l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum|l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum|derived__memory_l2_theoretical_sectors_global_excessive|sm__warps_active.avg.pct_of_peak_sustained_active|launch__registers_per_thread|smsp__issue_active.avg.pct_of_peak_sustained_active|launch__grid_size|sm__sass_l1tex_m_xbar2l1tex_read_bytes_mem_global_op_ldgsts_cache_bypass.sum'
run() {  # name shape mode k [forced regime] [extra tvc_one args]
  name=$1; shape=$2; mode=$3; k=$4; force=${5:--1}; extra=$6
  env TENVEC_B200_FORCE=$force python scripts/tvc_one.py --shape $shape --mode $mode --k $k $extra > gpurun_out/ncu_suite/one_$name.log 2>&1 && \
  env TENVEC_B200_FORCE=$force ncu --set full --clock-control none -k regex:"k_(rows|cols|slabs|staged|flat|naive)" -s 1 -c 1 -o /tmp/p_$name python scripts/tvc_one.py --shape $shape --mode $mode --k $k $extra > gpurun_out/ncu_suite/ncu_$name.log 2>&1
  echo $name rc=$?
  ncu -i /tmp/p_$name.ncu-rep --page raw --csv > /tmp/raw_$name.csv 2>/dev/null
  python - "$name" "$KEYS" <<'PY'
import csv, sys
name, keys = sys.argv[1], sys.argv[2].split('|')
rows = list(csv.reader(open(f'/tmp/raw_{name}.csv')))
hdr, units = rows[0], rows[1]
idx = {h: i for i, h in enumerate(hdr)}
with open(f'gpurun_out/ncu_suite/{name}.csv', 'w') as fh:
    w = csv.writer(fh)
    w.writerow(['case'] + keys)
    w.writerow([''] + [units[idx[k]] if k in idx else '' for k in keys])
    for r in rows[2:]:
        w.writerow([name] + [r[idx[k]] if k in idx else '' for k in keys])
PY
}
run staged_long_f64_d7k4 19,19,19,19,19,19,19 f64 4
run staged_long_f64_d8k4 13,13,13,13,13,13,13,13 f64 4
run staged_long_f64_d4k2 175,175,175,175 f64 2
run staged_narrow_f32_c3p8_k3 96,96,96,96,12 f32 3
# launch list of the default bench command (C2), per-launch durations, no replay
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_suite/launches_c2.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_suite/launches.log 2>&1; echo launches rc=$?
