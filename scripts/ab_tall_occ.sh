#!/bin/bash
# STAGED_TALL occupancy A/B: default build (2 CTAs/SM, 48 KB stages) vs -DTV_TALL_OCC=3 (32 KB stages)
for cfg in "default 49152" "occ3 32768" "occ3 24576"; do
  set -- $cfg
  if [ $1 = occ3 ]; then export TENVEC_B200_LIB=$PWD/paper_2501_03121_b200/_lib/libtenvec_b200_occ3.so; else unset TENVEC_B200_LIB; fi
  TENVEC_B200_STAGE_BYTES=$2 timeout 300 python scripts/tall_probe.py 2>&1 | python -c "
import sys,json
print('== $1 $2')
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    if d['regime']=='staged_tall': print(' ',d['shape'],d['mode'],d['ms'],d['gbs'])"
done
