"""Single updates vs pipelined ingest vs the oracle on a small random stream (diagnostics)."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1910_01260_b200 import basis  # noqa: E402
from oracle import strom_oracle as so  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
cols = int(sys.argv[2]) if len(sys.argv) > 2 else 50
rng = np.random.default_rng(0)
x = rng.standard_normal((n, cols))
tol = 1e-8
ref = so.init(x[:, 0], tol)
st = basis.isvd_init(x[:, 0], tol)
print('init sigma dev', st.sigma.cpu().numpy(), 'ref', ref.sigma, flush=True)
for j in range(1, min(cols, 8)):
    d = so.Decision()
    ref = so.update(ref, x[:, j], d)
    st = basis.isvd_update(st, x[:, j])
    inf = st.info()
    s = st.sigma.cpu().numpy()
    print('single', j, 'rank', inf.rank, ref.rank, 'flags', inf.flags, 'c', inf.ncols_u, 'p %.6e %.6e' % (inf.last_p, d.p),
          'sig rel %.2e' % (np.max(np.abs(s - ref.sigma) / ref.sigma) if s.size == ref.sigma.size else -1), flush=True)
st0 = basis.isvd_init(x[:, 0], tol)
for k in (2, 3, 5, cols):
    sti = basis.ingest_simulation(st0, torch.as_tensor(x[:, 1:k], device='cuda'))
    ref = so.stream(x[:, :k], tol)
    s = sti.sigma.cpu().numpy()
    inf = sti.info()
    print('ingest', k, 'rank', inf.rank, ref.rank, 'flags', inf.flags, 'c', inf.ncols_u, 'p %.6e' % inf.last_p,
          'sig', s[:3], ref.sigma[:3], flush=True)
