"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import sys

agg = collections.defaultdict(lambda: [0, 0.0])
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get('Metric Name') != 'gpu__time_duration.sum':
        continue
    v = float(d['Metric Value'].replace(',', ''))
    v *= {'nsecond': 1e-6, 'usecond': 1e-3, 'msecond': 1.0, 'second': 1e3}.get(d.get('Metric Unit', 'nsecond'), 1e-6)
    name = d['Kernel Name'].split('(')[0]
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print(f"{'kernel':62s} {'launches':>8s} {'ms':>9s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[:62]:62s} {v[0]:8d} {v[1]:9.2f} {100 * v[1] / tot:5.1f}%")
print(f"{'total':62s} {sum(v[0] for v in agg.values()):8d} {tot:9.2f}")
