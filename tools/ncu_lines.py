"""Warp-stall samples and executed instructions per CUDA source line of one kernel
(ncu --page source --print-source sass,cuda; needs -lineinfo and --import-source on).

    python tools/ncu_lines.py report.ncu-rep kernel_regex [ntop]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass,cuda', '--kernel-name',
                      f'regex:{kern}', '--launch-count', '1'], capture_output=True, text=True).stdout
cur, hdr = None, None
acc = []
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == 'File Path':
        cur = r[1].split('/')[-1]
        continue
    if len(r) > 4 and r[0] == 'Line No':
        hdr = r
        si = hdr.index('Warp Stall Sampling (All Samples)')
        ie = hdr.index('Instructions Executed')
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].isdigit() or r[2] != '-':
        continue
    try:
        s, e = int(r[si]), int(r[ie])
    except ValueError:
        continue
    if s or e:
        acc.append((s, e, cur, int(r[0]), r[1].strip()[:100]))
tot_s = sum(a[0] for a in acc) or 1
tot_i = sum(a[1] for a in acc) or 1
print('samples', tot_s, 'warp instructions', tot_i)
print('share of samples, share of instructions, file:line')
for s, e, f, l, t in sorted(acc, key=lambda a: -a[0])[:ntop]:
    print(f'{s / tot_s:6.3f} {e / tot_i:6.3f}  {f}:{l}  {t}')
