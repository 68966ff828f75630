#!/bin/bash
# STAGED_TALL (x preloaded per tile, unpredicated columns) vs the previous tall choice; then parity
mkdir -p gpurun_out/tall
for st in 1 0; do
  TENVEC_B200_STAGED_TALL=$st timeout 300 python scripts/tall_probe.py > gpurun_out/tall/v3_staged_tall_$st.jsonl 2>&1
  echo "== STAGED_TALL=$st"; python -c "
import json
for l in open('gpurun_out/tall/v3_staged_tall_$st.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(' ',d['shape'],d['k'],d['mode'],d['regime'],d['ms'],d['gbs'])"
done
timeout 1500 python -m pytest tests/test_gpu_tvc.py tests/test_gpu_guards.py tests/test_acceptance_b200.py -q -p no:cacheprovider -x 2>&1 | tail -3
