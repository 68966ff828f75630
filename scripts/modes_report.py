import json, sys
f = sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/modes_quick.jsonl'
for l in open(f):
    try: d = json.loads(l)
    except ValueError: continue
    print(f"{d['tensor']:18s} k={d['k']} {d['regime']:10s} uvw={str(d['uvw']):26s} {d['ms']:8.3f}ms {d['gbs']:7.0f} GB/s")
