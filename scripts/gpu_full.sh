#!/bin/bash
# What the driver runs at round end on one GPU: pytest -m gpu, smoke(), the default bench and the reference arm.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/gpu_all.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/gpu_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo ref_rc=$?
python - <<'P'
import json
d=json.loads(open('gpurun_out/bench_default.json').read().strip().splitlines()[-1])
print({k:d.get(k) for k in ('value','ms_per_step','gpu_launches','clocks')}, d['e2e']['value'] if d.get('e2e') else None, d.get('parity',{}).get('status'))
h=d.get('hopm') or {}
print('hopm', h.get('value'), (h.get('e2e') or {}).get('value'), (h.get('parity') or {}).get('status'))
r=json.loads(open('gpurun_out/bench_reference.json').read().strip().splitlines()[-1]); print('ref', r.get('value'), r.get('unit'))
P
