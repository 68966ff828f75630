"""Side-by-side GB/s of several tvc_modes_bench.py jsonl runs.

    python scripts/ab_table.py gpurun_out/a.jsonl gpurun_out/b.jsonl ...
"""
import json
import os
import sys


def load(f):
    d = {}
    for line in open(f):
        try:
            r = json.loads(line)
        except ValueError:
            continue
        d[(r["tensor"], r["mode"], r["k"])] = r
    return d


files = sys.argv[1:]
D = [load(f) for f in files]
names = [os.path.basename(f).rsplit(".", 1)[0][-12:] for f in files]
print(f"{'case':32s}" + "".join(f"{n:>15s}" for n in names))
for key in D[0]:
    cells = []
    for d in D:
        r = d.get(key)
        cells.append(f"{r['regime'][:6]}:{r['gbs']:5.0f}" if r else "-")
    print(f"{key[0][:16]:16s} {key[1]:8s} k={key[2]:<2d}  " + "".join(f"{c:>15s}" for c in cells))
