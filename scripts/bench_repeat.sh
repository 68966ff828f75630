#!/bin/bash
# the default bench line, three times back to back (run-to-run variance)
mkdir -p gpurun_out/rep
for i in 1 2 3 4; do
  timeout 900 python bench.py > gpurun_out/rep/default_$i.json 2> gpurun_out/rep/default_$i.err
  python -c "
import json
d=json.loads(open('gpurun_out/rep/default_$i.json').read().strip().splitlines()[-1])
print($i, d['value'], d['ms_per_step'], d['step_ms_rank0'], d['e2e']['value'], d['hopm']['value'])"
done
