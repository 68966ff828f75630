#!/bin/bash
# A/B of the SLABS split-K knobs on the tall views (scripts/tall_probe.py)
mkdir -p gpurun_out/tall
for cfg in "1 32" "2 32" "1 64" "2 64" "1 16" "2 128"; do
  set -- $cfg
  TENVEC_B200_SLAB_UNR=$1 TENVEC_B200_SLAB_SPLIT=$2 timeout 300 python scripts/tall_probe.py > gpurun_out/tall/unr$1_split$2.jsonl 2>&1
  echo "== unr=$1 split=$2"; grep -E '"slabs' gpurun_out/tall/unr$1_split$2.jsonl | python -c "import sys,json;[print(' ',d['shape'],d['mode'],d['regime'],d['ms'],d['gbs']) for d in map(json.loads,sys.stdin)]"
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
  --clock-control none -c 2000 --csv --log-file gpurun_out/tall/launches.csv python scripts/tall_probe.py > gpurun_out/tall/ncu.log 2>&1; echo ncu_rc=$?
