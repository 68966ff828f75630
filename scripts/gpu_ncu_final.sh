bash scripts/gpu_ncu_c2.sh
s=$(cat scripts/gpu_ncu_suite.sh); head=${s%%run cols_f64_1024c_k0*}
eval "$head"
run rows_f64_1024c_k2 1024,1024,1024 f64 2
run cols_f64_1024c_k0 1024,1024,1024 f64 0
