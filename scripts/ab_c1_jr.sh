#!/bin/bash
# C1 COLS row phases (TENVEC_B200_COL_JR) A/B through bench.py --workload c1
mkdir -p gpurun_out/c1jr
for jr in 0 4 1 8; do
  if [ $jr = 0 ]; then unset TENVEC_B200_COL_JR; else export TENVEC_B200_COL_JR=$jr; fi
  timeout 600 python bench.py --workload c1 --steps 20 --warmup 5 --hopm-workload none > gpurun_out/c1jr/jr$jr.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/c1jr/jr$jr.json').read().strip().splitlines()[-1])
print('JR=$jr', d['value'], d['ms_per_step'], [(m['k'],m['regime'],m['ms'],m['gbs']) for m in d.get('modes',[])])"
done
