mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python scripts/tvc_modes_bench.py --set table1 > gpurun_out/cur_1.jsonl 2>&1; echo cur rc=$?
TENVEC_B200_LIB=$PWD/paper_2501_03121_b200/_lib/libtenvec_b200_prev.so timeout 300 python scripts/tvc_modes_bench.py --set table1 > gpurun_out/prev_1.jsonl 2>&1; echo prev rc=$?
timeout 600 python scripts/tvc_modes_bench.py --set baseline > gpurun_out/cur_base.jsonl 2>&1; echo base rc=$?
python scripts/tall_probe.py > gpurun_out/tall.jsonl 2>&1; echo tall rc=$?
