"""SASS instruction census of the sm_100a library: per kernel, the count of the
instructions that show which hardware path it uses (DMMA = fp64 tensor core,
UBLKCP = cp.async.bulk / TMA, SYNCS = mbarrier, LDGSTS = cp.async, BAR, DFMA...).

    python tools/sass_census.py [paper_1910_01260_b200/_lib/libstrom_b200.so] > profiles/r02_sass_census.txt
"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1910_01260_b200/_lib/libstrom_b200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
want = ["DMMA", "DFMA", "DADD", "DMUL", "UBLKCP", "UBLKPF", "SYNCS", "LDGSTS", "BAR", "SHFL", "LDS", "STS",
        "LDG", "STG", "MUFU", "ATOMG", "RED", "USETMAXREG"]
per = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        per[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m:
        op = m.group(1)
        for w in want:
            if op == w or op.startswith(w + "") and w in ("LDS", "STS", "LDG", "STG") and op == w:
                per[cur][w] += 1
        if op.startswith("DMMA"):
            per[cur]["DMMA"] += 0  # counted above via exact match
tot = collections.Counter()
rows = []
for fn, c in per.items():
    if not any(c[w] for w in want):
        continue
    dem = subprocess.run(["c++filt", fn], capture_output=True, text=True).stdout.strip()
    rows.append((dem[:70], c))
    tot.update(c)
print("kernel".ljust(72) + "".join(w.rjust(8) for w in want))
for name, c in rows:
    print(name.ljust(72) + "".join(str(c[w]).rjust(8) for w in want))
print("TOTAL".ljust(72) + "".join(str(tot[w]).rjust(8) for w in want))
print("\nno tcgen05 / UTCMMA: tcgen05 has no f64 kind; fp64 tensor math on sm_100a is mma.sync m8n8k4 (DMMA).")
