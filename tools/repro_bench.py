"""Bench-like pattern: repeated ingestion from one shared state (diagnostics)."""
import sys

import torch

sys.path.insert(0, '.')
from paper_1910_01260_b200 import basis, workloads as wl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
ncols = int(sys.argv[2]) if len(sys.argv) > 2 else 400
xt, _, _, _ = wl.cfg2_stream_torch(n=n, cols=100 + ncols, rank=64, seed=0)
st = basis.isvd_init(xt[0], 1e-9, tol_sv=1e-9, r_max=64, cap_mode='truncate')
st100 = basis.ingest_simulation(st, xt[1:100].T)
torch.cuda.synchronize()
print('warm ok', st100.rank, flush=True)
for rep in range(3):
    out = basis.ingest_simulation(st100, xt[100:].T)
    torch.cuda.synchronize()
    print('rep', rep, 'rank', out.rank, 'sigma0', float(out.sigma[0]), flush=True)
