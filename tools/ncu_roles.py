"""Stall reasons split into the consumer (address span of the DMMA loop copies) and the rest."""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--kernel-name', f'regex:{kern}',
                      '--launch-count', '1'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if 'Source' in r and 'Address' in r)
h = rows[hi]
seen, data = set(), []
for r in rows[hi + 1:]:
    if len(r) == len(h) and r[0].startswith('0x') and r[0] not in seen:
        seen.add(r[0]); data.append(r)
src = h.index('Source')
cols = [i for i, c in enumerate(h) if c.startswith('stall_') and 'Not Issued' not in c]
dm = [int(r[0], 16) for r in data if 'DMMA' in r[src]]
lo, hi_ = min(dm) - 0x400, max(dm) + 0x100
for name, sel in (('consumer', lambda a: lo <= a <= hi_), ('producer+rest', lambda a: not (lo <= a <= hi_))):
    t = collections.Counter()
    for r in data:
        if sel(int(r[0], 16)):
            for i in cols:
                t[h[i][6:]] += int(r[i] or 0)
    s = sum(t.values()) or 1
    print(f'{name:14s} samples {s:7d}: ' + ', '.join(f'{k} {v / s:.2f}' for k, v in t.most_common(8)))
