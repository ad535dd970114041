"""Stall-reason totals of one kernel, split by address range (e.g. producer vs consumer code),
plus the SASS of a window around a given address.  usage: ncu_stalls.py rep kernel [addr_lo addr_hi]"""
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
cols = [i for i, c in enumerate(h) if c.startswith('stall_') and 'Not Issued' not in c]
tot = collections.Counter()
for r in data:
    for i in cols:
        tot[h[i]] += int(r[i] or 0)
s = sum(tot.values()) or 1
print('stall totals:', ', '.join(f'{k[6:]} {v / s:.2f}' for k, v in tot.most_common(8)))
if len(sys.argv) > 4:
    lo, hi_ = int(sys.argv[3], 16), int(sys.argv[4], 16)
    ie = h.index('Instructions Executed'); src = h.index('Source')
    for r in data:
        a = int(r[0], 16) & 0xfffff
        if lo <= a <= hi_:
            top = sorted(((int(r[i] or 0), h[i][6:]) for i in cols), reverse=True)[:2]
            print(f'{a:05x} {r[ie]:>8s} {r[src][:70]:70s} {top}')
