"""Per-kernel aggregate of an ncu --csv launch list with time and DRAM bytes
(`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum`).
Usage: python tools/launch_metrics.py launches.csv"""
import collections
import csv
import sys

UNITS = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1, 'usecond': 1, 'ms': 1e3, 'msecond': 1e3,
         'byte': 1, 'Kbyte': 1e3, 'KB': 1e3, 'Mbyte': 1e6, 'MB': 1e6, 'Gbyte': 1e9, 'GB': 1e9}
rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith('==')))
launch = {}
for r in rows:
    launch.setdefault((r['ID'], r['Kernel Name']), {})[r['Metric Name']] = \
        float(r['Metric Value'].replace(',', '')) * UNITS[r['Metric Unit']]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for (_, k), m in launch.items():
    a = agg[k.split('(')[0][:44]]
    a[0] += 1
    a[1] += m['gpu__time_duration.sum']
    a[2] += m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':44s} {'n':>4s} {'mean_us':>9s} {'MB':>8s} {'GB/s':>7s} {'share':>6s}")
for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:44s} {n:4d} {t / n:9.2f} {b / n / 1e6:8.2f} {b / t / 1e3:7.0f} {t / tot:6.3f}")
