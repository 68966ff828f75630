#!/bin/bash
# aligned tall views: SLABS (default) vs STAGED_TALL forced
mkdir -p gpurun_out/tall
for f in 0 13; do
  if [ $f = 0 ]; then unset TENVEC_B200_FORCE; else export TENVEC_B200_FORCE=$f; fi
  timeout 300 python scripts/tall_probe.py > gpurun_out/tall/force_$f.jsonl 2>&1
  echo "== force=$f"; python -c "
import json
for l in open('gpurun_out/tall/force_$f.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(' ',d['shape'],d['k'],d['mode'],d['regime'],d['ms'],d['gbs'])"
done
