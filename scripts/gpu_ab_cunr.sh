mkdir -p gpurun_out
for r in 1 2; do
timeout 300 python scripts/tvc_modes_bench.py --set baseline > gpurun_out/cu_base_$r.jsonl 2>&1
for v in c8u6 c1u12 c1u6; do
TENVEC_B200_LIB=$PWD/paper_2501_03121_b200/_lib/libtenvec_b200_$v.so timeout 300 python scripts/tvc_modes_bench.py --set baseline > gpurun_out/cu_${v}_$r.jsonl 2>&1
done
done
echo done
