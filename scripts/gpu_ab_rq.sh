mkdir -p gpurun_out
for r in 1 2; do
timeout 300 python scripts/tvc_modes_bench.py --set baseline > gpurun_out/rq4_$r.jsonl 2>&1
for q in 6 8; do
TENVEC_B200_LIB=$PWD/paper_2501_03121_b200/_lib/libtenvec_b200_rq$q.so timeout 300 python scripts/tvc_modes_bench.py --set baseline > gpurun_out/rq${q}_$r.jsonl 2>&1
done
done
echo done
