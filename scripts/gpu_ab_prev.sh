mkdir -p gpurun_out
for r in 1 2; do
timeout 300 python scripts/tvc_modes_bench.py --set table1 > gpurun_out/cur_$r.jsonl 2>&1; echo cur rc=$?
TENVEC_B200_LIB=$PWD/paper_2501_03121_b200/_lib/libtenvec_b200_prev.so timeout 300 python scripts/tvc_modes_bench.py --set table1 > gpurun_out/prev_$r.jsonl 2>&1; echo prev rc=$?
done
