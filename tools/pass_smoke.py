"""Time a few cfg2-size updates (diagnostics for the pass kernel)."""
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_1910_01260_b200 import basis, workloads as wl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
cols = int(sys.argv[2]) if len(sys.argv) > 2 else 12
xt_all, _, _, _ = wl.cfg2_stream_torch(n=n, cols=max(cols, 64), rank=64, seed=0)
xt = xt_all[:cols]
st = basis.isvd_init(xt[0], 1e-9, tol_sv=1e-9, r_max=64, cap_mode='truncate')
torch.cuda.synchronize()
print('init ok', flush=True)
t = time.time()
st1 = basis.isvd_update(st, xt[1])
torch.cuda.synchronize()
print('single update ok %.3f ms' % ((time.time() - t) * 1e3), st1.rank, flush=True)
t = time.time()
st2 = basis.ingest_simulation(st, xt[1:].T)
torch.cuda.synchronize()
print('ingest ok %.3f ms' % ((time.time() - t) * 1e3), st2.rank, flush=True)
