mkdir -p gpurun_out
run() {  # name shape mode k [env]
  name=$1; shape=$2; mode=$3; k=$4; envv=$5
  env $envv python scripts/tvc_one.py --shape $shape --mode $mode --k $k > gpurun_out/one_$name.log 2>&1 && \
  env $envv ncu --set full --clock-control none -k regex:"k_" -s 1 -c 1 -o /tmp/p_$name python scripts/tvc_one.py --shape $shape --mode $mode --k $k > gpurun_out/ncu_$name.log 2>&1
  echo $name rc=$?
  ncu -i /tmp/p_$name.ncu-rep --page raw --csv > gpurun_out/raw_$name.csv 2>/dev/null
  ncu -i /tmp/p_$name.ncu-rep --page details --csv > gpurun_out/details_$name.csv 2>/dev/null
}
for spec in "$@"; do run $spec; done
