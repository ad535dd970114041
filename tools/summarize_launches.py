"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
scale = {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3, 'second': 1e6, 's': 1e6}
agg = collections.defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split('(')[0].replace('void ', '').strip()
    agg[name].append(float(r[vi].replace(',', '')) * scale[r[ui]])
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':40s} {'launches':>8s} {'total_ms':>10s} {'mean_us':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:40]:40s} {len(v):8d} {sum(v) / 1e3:10.3f} {sum(v) / len(v):10.2f} {sum(v) / tot:6.3f}")
