#!/bin/bash
mkdir -p gpurun_out/final
timeout 1200 python scripts/tvc_modes_bench.py --set all --reps 5 > gpurun_out/final/modes_all.jsonl 2>&1; echo modes_rc=$?
timeout 300 python scripts/tall_probe.py > gpurun_out/final/tall_views.jsonl 2>&1; echo tall_rc=$?
python - <<'P'
import json, statistics
rows=[json.loads(l) for l in open('gpurun_out/final/modes_all.jsonl') if l.startswith('{')]
t1=[r for r in rows if r['tensor'].startswith('paper')]
g=[r['gbs'] for r in t1]
print('table1 n', len(g), 'min', min(g), 'max', max(g), 'mean', round(statistics.mean(g),1), 'sd%', round(100*statistics.pstdev(g)/statistics.mean(g),2), '>=6000', sum(x>=6000 for x in g))
for r in sorted(rows, key=lambda r: r['gbs'])[:6]: print(r['tensor'], r['k'], r['regime'], r['gbs'])
P
