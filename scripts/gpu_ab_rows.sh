mkdir -p gpurun_out
timeout 300 python scripts/tvc_modes_bench.py --set baseline > gpurun_out/rowsb1.jsonl 2>&1; echo a rc=$?
for m in 4 6; do
TENVEC_B200_LIB=$PWD/paper_2501_03121_b200/_lib/libtenvec_b200_rows$m.so timeout 300 python scripts/tvc_modes_bench.py --set baseline > gpurun_out/rowsb$m.jsonl 2>&1; echo $m rc=$?
done
