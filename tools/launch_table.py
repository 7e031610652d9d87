"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split('(')[0].replace('void ', '').split('<')[0]
    v = float(r[vi].replace(',', ''))
    v = {'nsecond': v / 1000, 'ns': v / 1000, 'usecond': v, 'us': v, 'msecond': v * 1000, 'ms': v * 1000}[r[ui]]
    agg.setdefault(name, []).append(v)
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tot = sum(sum(v[skip:]) for v in agg.values())
print(f"{'kernel':24s} {'n':>5s} {'mean_us':>9s} {'min_us':>8s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1][skip:])):
    vv = v[skip:] or v
    print(f"{k:24s} {len(vv):5d} {sum(vv)/len(vv):9.2f} {min(vv):8.2f} {sum(vv)/tot:6.3f}")
