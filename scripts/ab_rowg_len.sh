#!/bin/bash
# ROWS lanes per row vs row length (aligned rows, >= 1 GB views), two passes
mkdir -p gpurun_out/rowg
V="f64:1048576,128:1 f32:2097152,256:1 bf16f32:2097152,512:1 f64:524288,256:1 f32:524288,512:1 bf16f32:1048576,1024:1 f64:349528,384:1 f64:262144,512:1 f32:262144,1024:1 bf16f32:524288,2048:1"
for pass in 1 2; do
for g in 0 8 16 32; do
  if [ $g = 0 ]; then unset TENVEC_B200_ROW_G; else export TENVEC_B200_ROW_G=$g; fi
  timeout 600 python scripts/time_views.py $V > gpurun_out/rowg/len_g${g}_p$pass.jsonl 2>&1
done
done
python - <<'P'
import json, collections
res=collections.defaultdict(dict)
for g in (0,8,16,32):
    for p in (1,2):
        for l in open(f'gpurun_out/rowg/len_g{g}_p{p}.jsonl'):
            try: d=json.loads(l)
            except Exception: continue
            key=(d['mode'],tuple(d['shape']))
            res[key].setdefault(g,[]).append(d['gbs'])
for key,v in res.items():
    print(key, {g: [round(x) for x in xs] for g,xs in sorted(v.items())})
P
