"""Stall-reason totals of one kernel from an ncu report's source page, for the
launch with the most executed instructions (a capture may hold no-op launches,
e.g. window-mode residual passes of dependent snapshots), plus the SASS of a
window around given addresses.  usage: ncu_stalls.py rep kernel [addr_lo addr_hi]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--kernel-name', f'regex:{kern}'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
tables, cur, h = [], None, None
for r in rows:
    if 'Source' in r and 'Address' in r:
        h = r
        cur = []
        tables.append((h, cur))
    elif cur is not None and len(r) == len(h) and r[0].startswith('0x'):
        cur.append(r)


def executed(t):
    hh, data = t
    ie = hh.index('Instructions Executed') if 'Instructions Executed' in hh else None
    return sum(int(r[ie] or 0) for r in data) if ie is not None else 0


if not tables:
    print('no source table')
    sys.exit(0)
h, data = max(tables, key=executed)
seen, uniq = set(), []
for r in data:
    if r[0] not in seen:
        seen.add(r[0])
        uniq.append(r)
cols = [i for i, c in enumerate(h) if c.startswith('stall_') and 'Not Issued' not in c]
tot = collections.Counter()
for r in uniq:
    for i in cols:
        tot[h[i]] += int(r[i] or 0)
s = sum(tot.values()) or 1
print(f'launches in report: {len(tables)}; showing the one with {executed((h, data))} executed instructions')
print('stall totals:', ', '.join(f'{k[6:]} {v / s:.2f}' for k, v in tot.most_common(8)))
if len(sys.argv) > 4:
    lo, hi_ = int(sys.argv[3], 16), int(sys.argv[4], 16)
    ie = h.index('Instructions Executed'); src = h.index('Source')
    for r in uniq:
        a = int(r[0], 16) & 0xfffff
        if lo <= a <= hi_:
            top = sorted(((int(r[i] or 0), h[i][6:]) for i in cols), reverse=True)[:2]
            print(f'{a:05x} {r[ie]:>8s} {r[src][:70]:70s} {top}')
