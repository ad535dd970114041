"""Per-opcode instruction / stall shares and the top stall lines of one kernel's SASS source page."""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--kernel-name', f'regex:{kern}', '--launch-count', '1'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if 'Source' in r and 'Address' in r)
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0].startswith('0x')]
si, ie, src = h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed'), h.index('Source')
tot = sum(int(r[si]) for r in data) or 1
ti = sum(int(r[ie]) for r in data) or 1
print('samples', tot, 'instructions', ti)
op, ops = collections.Counter(), collections.Counter()
for r in data:
    w = r[src].split()
    o = w[1] if w and w[0].startswith('@') else (w[0] if w else '')
    o = o.split('.')[0]
    op[o] += int(r[ie])
    ops[o] += int(r[si])
for o, c in op.most_common(16):
    print(f'{o:10s} instr {c / ti:.3f} stall {ops[o] / tot:.3f}')
print('--- top stall lines (samples, executed, address, sass)')
for r in sorted(data, key=lambda r: -int(r[si]))[:ntop]:
    print(r[si], r[ie], r[0][-5:], r[src][:90])
