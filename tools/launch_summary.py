"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith('=='))]
hdr = rows[0]
ki, mi, vi = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value')
agg = OrderedDict()
for r in rows[1:]:
    if r[mi] != 'gpu__time_duration.sum':
        continue
    name = r[ki].split('(')[0].replace('void ', '').replace('<unnamed>::', '')
    t = float(r[vi].replace(',', ''))
    c, s = agg.get(name, (0, 0.0))
    agg[name] = (c + 1, s + t)
tot = sum(s for _, s in agg.values())
print(f"{'kernel':58s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}")
for name, (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{name[:58]:58s} {c:8d} {s / 1e6:10.3f} {100 * s / tot:6.1f}%")
print(f"{'TOTAL':58s} {sum(c for c, _ in agg.values()):8d} {tot / 1e6:10.3f}")
