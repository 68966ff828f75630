import json, glob, sys
runs = {}
for f in sorted(glob.glob('gpurun_out/ab_*.jsonl')):
    tag = f.split('ab_')[1].split('.')[0]
    for l in open(f):
        try: d = json.loads(l)
        except ValueError: continue
        runs.setdefault((d['tensor'], d['k']), {})[tag] = (d['regime'], d['gbs'])
for key, r in runs.items():
    dflt = r.get('default')
    best = {}
    for tag, (reg, gbs) in r.items():
        if tag == 'default': continue
        if reg not in best or gbs > best[reg]: best[reg] = gbs
    alts = ' '.join(f"{reg}:{gbs:.0f}" for reg, gbs in sorted(best.items(), key=lambda t: -t[1]))
    flag = '' if not dflt or not best or dflt[1] >= 0.97 * max(best.values()) else '  <<<'
    print(f"{key[0]:18s} k={key[1]} default {dflt[0] if dflt else '-':10s} {dflt[1] if dflt else 0:6.0f} | {alts}{flag}")
