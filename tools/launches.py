"""Summarise an ncu gpu__time_duration launch list: per-kernel totals for the LAST step."""
import csv, collections, re, sys
path = sys.argv[1]
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            data.append((d['Kernel Name'], float(d['Metric Value'])))
ours = [(n, t) for n, t in data if 'rsvd::' in n]
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
per = len(ours) // nsteps
step = ours[-per:]
agg = collections.defaultdict(lambda: [0, 0.0])
for name, t in step:
    key = re.sub(r'\(.*', '', name).replace('void ', '')[:48]
    agg[key][0] += 1; agg[key][1] += t
tot = sum(v[1] for v in agg.values())
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:48s} {c:4d} launches {t/1e3:9.1f} us  {100*t/tot:5.1f}%  ({t/c/1e3:7.1f} us each)")
print(f"total {tot/1e3:.1f} us over {len(step)} launches (ncu: serialised, cold cache)")
