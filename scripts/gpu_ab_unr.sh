mkdir -p gpurun_out
timeout 300 python scripts/tvc_modes_bench.py --set table1 > gpurun_out/unr4.jsonl 2>&1; echo a rc=$?
TENVEC_B200_LIB=$PWD/paper_2501_03121_b200/_lib/libtenvec_b200_unr8.so timeout 300 python scripts/tvc_modes_bench.py --set table1 > gpurun_out/unr8.jsonl 2>&1; echo b rc=$?
