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
run cols_f64_1024c_k0 1024,1024,1024 f64 0
run cols_f64_1024c_k1 1024,1024,1024 f64 1
run rows_f64_1024c_k2 1024,1024,1024 f64 2
run cols_u_f64_979c_k0 979,979,979 f64 0
run rows_u_f64_979c_k2 979,979,979 f64 2
run slabs_f32_c3p2_k3 96,96,96,96,48 f32 3
run rows_f32_c3p8_k4 96,96,96,96,12 f32 4
run slabs_u_f32_k1 20000,300,21 f32 1
run staged_f64_13p8_k6 13,13,13,13,13,13,13,13 f64 6
run staged_f64_13p8_k7 13,13,13,13,13,13,13,13 f64 7
run staged_f64_175p4_k3 175,175,175,175 f64 3
run staged_f64_63p5_k3 63,63,63,63,63 f64 3
run flat_f32_c3_k3 96,96,96,96,96 f32 3
run cols_bf16_c5p8_k1 4096,4096,512 bf16f32 1
run rows_bf16_c5p8_k2 4096,4096,512 bf16f32 2
run cols_f32f64_k0 512,512,512 f32f64 0
run rows_f16_k2 2048,2048,512 f16f32 2
# regimes the heuristics rarely pick, forced (TENVEC_B200_FORCE): narrow
# unaligned slabs, short rows, flat short rows; and the naive cross-check
run slabs_u_forced_f32 2000,3000,21 f32 1 7
run rows_short_forced_f32 4096,4096,16 f32 2 2
run flat_rows_forced_f32 4096,4096,24 f32 2 10
run naive_f64 256,256,256 f64 1 -1 --naive
# non-TVC kernels
python scripts/util_one.py > gpurun_out/ncu_suite/util_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:"k_(fold|norm|convert|fill|tvc_norm|axpby|select|read_stream)" -c 10 -o /tmp/p_util python scripts/util_one.py > gpurun_out/ncu_suite/ncu_util.log 2>&1
echo util rc=$?
ncu -i /tmp/p_util.ncu-rep --page raw --csv > /tmp/raw_util.csv 2>/dev/null
python - util "$KEYS" <<'PY'
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
