#!/bin/bash
# ROWS lanes per row on C1 (bench.py --workload c1: cold L2, per-mode kernel times)
mkdir -p gpurun_out/rowg
for g in 0 16 8 0; do
  if [ $g = 0 ]; then unset TENVEC_B200_ROW_G; else export TENVEC_B200_ROW_G=$g; fi
  timeout 600 python bench.py --workload c1 --steps 20 --warmup 5 --hopm-workload none > gpurun_out/rowg/c1_g$g.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/rowg/c1_g$g.json').read().strip().splitlines()[-1])
print('G=$g', d['value'], d['ms_per_step'], [(m['k'],m['regime'],m['ms'],m['gbs']) for m in d.get('modes',[])])"
done
