"""Single-update loop at cfg2 size, printing c/rank/flags (diagnostics)."""
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_1910_01260_b200 import basis, workloads as wl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
cols = int(sys.argv[2]) if len(sys.argv) > 2 else 140
xt, _, _, _ = wl.cfg2_stream_torch(n=n, cols=max(cols, 64), rank=64, seed=0)
st = basis.isvd_init(xt[0], 1e-9, tol_sv=1e-9, r_max=64, cap_mode='truncate')
for j in range(1, cols):
    t = time.time()
    st = basis.isvd_update(st, xt[j])
    inf = st.info()
    print(j, 'rank', inf.rank, 'c', inf.ncols_u, 'flags', inf.flags, '%.2f ms' % ((time.time() - t) * 1e3), flush=True)
