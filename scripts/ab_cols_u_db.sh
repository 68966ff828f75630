#!/bin/bash
# COLS_U register double buffer (JR = 8) A/B over the paper's Table-1 modes
mkdir -p gpurun_out/colsu
for db in 1 0; do
  TENVEC_B200_COLS_U_DB=$db timeout 900 python scripts/tvc_modes_bench.py --set table1 --reps 5 > gpurun_out/colsu/table1_db$db.jsonl 2>&1
done
python - <<'P'
import json
def load(f):
    out={}
    for l in open(f):
        try: d=json.loads(l)
        except Exception: continue
        out[(d['tensor'],d['k'])]=d
    return out
a=load('gpurun_out/colsu/table1_db1.jsonl'); b=load('gpurun_out/colsu/table1_db0.jsonl')
for key in a:
    if key in b and (a[key]['regime']=='cols_u' or abs(a[key]['gbs']-b[key]['gbs'])>100):
        print(key, a[key]['regime'], 'db1', a[key]['gbs'], 'db0', b[key]['gbs'])
import statistics
print('min db1', min(d['gbs'] for d in a.values()), 'min db0', min(d['gbs'] for d in b.values()))
print('mean db1', statistics.mean(d['gbs'] for d in a.values()), 'mean db0', statistics.mean(d['gbs'] for d in b.values()))
P
