mkdir -p gpurun_out
timeout 300 python scripts/tvc_modes_bench.py --set table1 > gpurun_out/unr4.jsonl 2>&1; echo a rc=$?
for u in 2 3; do
TENVEC_B200_LIB=$PWD/paper_2501_03121_b200/_lib/libtenvec_b200_unr$u.so timeout 300 python scripts/tvc_modes_bench.py --set table1 > gpurun_out/unr$u.jsonl 2>&1; echo $u rc=$?
done
