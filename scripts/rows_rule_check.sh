#!/bin/bash
# the new ROWS lane-group rule: row-length views, BASELINE views, benches, parity
mkdir -p gpurun_out/rowg
timeout 600 python scripts/time_views.py f64:1048576,128:1 f32:2097152,256:1 bf16f32:2097152,512:1 f64:524288,256:1 f32:524288,512:1 bf16f32:1048576,1024:1 f64:349528,384:1 f64:262144,512:1 f32:262144,1024:1 bf16f32:524288,2048:1 > gpurun_out/rowg/len_new.jsonl 2>&1
cat gpurun_out/rowg/len_new.jsonl
timeout 900 python scripts/tvc_modes_bench.py --set baseline --reps 5 > gpurun_out/rowg/baseline_new.jsonl 2>&1
grep '"rows' gpurun_out/rowg/baseline_new.jsonl
timeout 600 python bench.py --workload c1 --steps 20 --warmup 5 --hopm-workload none > gpurun_out/rowg/c1_new.json 2>/dev/null
python -c "
import json
d=json.loads(open('gpurun_out/rowg/c1_new.json').read().strip().splitlines()[-1])
print('c1', d['value'], d['ms_per_step'], d['parity']['status'], [(m['k'],m['regime'],m['ms'],m['gbs']) for m in d.get('modes',[])])"
timeout 900 python bench.py > gpurun_out/rowg/default_new.json 2>/dev/null
python -c "
import json
d=json.loads(open('gpurun_out/rowg/default_new.json').read().strip().splitlines()[-1])
print('c2', d['value'], d['parity']['status'], 'e2e', d['e2e']['value'], 'hopm', d['hopm']['value'], d['hopm']['parity']['status'], d['clocks'])"
timeout 900 python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/rowg/c5_new.json 2>/dev/null
python -c "
import json
d=json.loads(open('gpurun_out/rowg/c5_new.json').read().strip().splitlines()[-1])
print('c5', d['value'], d.get('parity',{}).get('status'), d.get('clocks'))"
timeout 1500 python -m pytest tests/test_gpu_tvc.py tests/test_gpu_hopm.py -q -p no:cacheprovider -x 2>&1 | tail -2
