import os, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1910_01260_b200 import basis, workloads as wl
xt, _, _, _ = wl.cfg2_stream_torch(n=1 << 20, cols=500, rank=64, seed=0)
st0 = basis.isvd_init(xt[0], 1e-9, tol_sv=1e-9, r_max=64, cap_mode="truncate")
st100 = basis.ingest_simulation(st0, xt[1:100].T)
xh = np.asfortranarray(xt[100:].T.cpu().numpy())  # (n, 400) pageable, columns contiguous
for _ in range(3):
    basis.ingest_simulation(st100, xh).sigma.cpu()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    basis.ingest_simulation(st100, xh).sigma.cpu()
    ts.append(time.perf_counter() - t0)
print(os.environ.get('STROM_COPY_THREADS', 'default'), [round(t * 1e3, 1) for t in ts], 'snapshots/s at median', round(400 / sorted(ts)[2]))
