"""Markdown table of the per-kernel ncu summaries written by tools/gpu_prof_r2.sh
(sum_*.txt from ncu_summary.py, stalls_*.txt from ncu_stalls.py): the longest captured
launch of every kernel.

    python tools/ncu_table.py gpurun_out/r02_prof4 > profiles/r02_q_ncu_kernels.md
"""
import glob
import os
import re
import sys

d = sys.argv[1]
rows = []
for f in sorted(glob.glob(os.path.join(d, 'sum_*.txt'))):
    cap = os.path.basename(f)[4:-4]
    stalls = ''
    sf = os.path.join(d, f'stalls_{cap}.txt')
    if os.path.exists(sf):
        for line in open(sf):
            if line.lower().startswith(('top', 'stall')):
                stalls = line.strip()
                break
        if not stalls:
            txt = open(sf).read().strip().splitlines()
            stalls = txt[-1][:120] if txt else ''
    best = {}
    cur = None
    for line in open(f):
        if line.startswith('== '):
            cur = {'name': line[3:].strip()}
            continue
        m = re.match(r'\s+(\S+)\s+([0-9.eE+-]+)\s*(.*)', line)
        if m and cur is not None:
            cur[m.group(1)] = (float(m.group(2)), m.group(3).strip())
            if m.group(1) == 'smsp__issue_active.avg.pct_of_peak_sustained_active':
                t = cur.get('gpu__time_duration.sum', (0, ''))
                us = t[0] * (1e3 if t[1].startswith('ms') else 1.0)
                key = cur['name']
                if key not in best or us > best[key][0]:
                    best[key] = (us, cur)
                cur = None
    for name, (us, c) in best.items():
        def g(k, fmt='{:.3g}'):
            v = c.get(k)
            return (fmt.format(v[0]) + (' ' + v[1] if v[1] and not v[1].startswith('%') else '')) if v else '-'
        rows.append((cap, name[:62], us, g('dram__bytes_read.sum'), g('dram__bytes_write.sum'),
                     g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', '{:.1f}'),
                     g('sm__warps_active.avg.pct_of_peak_sustained_active', '{:.1f}'),
                     g('smsp__issue_active.avg.pct_of_peak_sustained_active', '{:.1f}'),
                     g('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', '{:.1f}'),
                     g('launch__registers_per_thread', '{:.0f}'), g('launch__grid_size', '{:.0f}'),
                     g('launch__block_size', '{:.0f}'), stalls))
print('| capture | kernel | time (us) | DRAM read | DRAM write | DRAM % | warps active % | issue active % | '
      'fp64 pipe % | regs | grid | block | top stalls (capture) |')
print('|---|---|---|---|---|---|---|---|---|---|---|---|---|')
for r in rows:
    print('| ' + ' | '.join([r[0], '`' + r[1] + '`', f'{r[2]:.1f}'] + [str(x) for x in r[3:]]) + ' |')
