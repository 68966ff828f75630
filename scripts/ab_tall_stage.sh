#!/bin/bash
# STAGED_TALL tile size A/B (TENVEC_B200_STAGE_BYTES)
mkdir -p gpurun_out/tall
for sb in 49152 32768 24576; do
  TENVEC_B200_STAGE_BYTES=$sb timeout 300 python scripts/tall_probe.py > gpurun_out/tall/stage_$sb.jsonl 2>&1
  echo "== stage=$sb"; python -c "
import json
for l in open('gpurun_out/tall/stage_$sb.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    if d['regime']=='staged_tall': print(' ',d['shape'],d['k'],d['mode'],d['regime'],d['ms'],d['gbs'])"
done
