"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            data.append((d['Kernel Name'].split('(')[0][-48:], float(d['Metric Value']), d['Metric Unit']))
agg = collections.OrderedDict()
for n, v, u in data:
    agg.setdefault(n, []).append(v)
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tot = 0
for n, v in agg.items():
    vv = v[skip:] if len(v) > skip else v
    m = sum(vv) / len(vv)
    print(f"{n:50s} n={len(v):3d} mean={m/1000:9.2f} us  min={min(vv)/1000:9.2f}")
