# usage: bash scripts/gpu_ncu_one.sh name shape mode k  -> gpurun_out/ncu_one/<name>_{raw,details}.csv
mkdir -p gpurun_out/ncu_one
name=$1; shape=$2; mode=$3; k=$4
python scripts/tvc_one.py --shape $shape --mode $mode --k $k > gpurun_out/ncu_one/one_$name.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_(rows|cols|slabs|staged|flat)" -s 1 -c 1 -o /tmp/p_$name python scripts/tvc_one.py --shape $shape --mode $mode --k $k > gpurun_out/ncu_one/ncu_$name.log 2>&1
echo $name rc=$?
ncu -i /tmp/p_$name.ncu-rep --page raw --csv > gpurun_out/ncu_one/${name}_raw.csv 2>/dev/null
ncu -i /tmp/p_$name.ncu-rep --page details --csv > gpurun_out/ncu_one/${name}_details.csv 2>/dev/null
ncu -i /tmp/p_$name.ncu-rep --page source --csv > gpurun_out/ncu_one/${name}_source.csv 2>/dev/null
