"""Orthonormality drift of Phi over pure dependent steps: device vs the numpy device model."""
import sys

import numpy as np

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from paper_1910_01260_b200 import basis, workloads as wl  # noqa: E402
import device_model as dm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
RK = int(sys.argv[2]) if len(sys.argv) > 2 else 32
x, q, w, s = wl.cfg2_stream_numpy(n=n, cols=140, rank=RK, seed=5)
x = np.ascontiguousarray(x)
tol = 1e-6  # every in-span column below is dependent
st = basis.isvd_init(x[:, 0], tol, tol_sv=1e-9, r_max=RK, cap_mode='truncate')
m = dm.init(x[:, 0], tol, tol_sv=1e-9, r_max=RK)
for j in range(1, 40):
    st = basis.isvd_update(st, x[:, j])
    m = dm.update(m, x[:, j])
rng = np.random.default_rng(0)
for j in range(40, 140):
    phi = st.phi.cpu().numpy()
    xin = phi @ rng.standard_normal(phi.shape[1])  # exactly in span of the device basis
    st = basis.isvd_update(st, xin)
    m = dm.update(m, m.phi @ rng.standard_normal(m.r))
    if j % 10 == 0:
        ph = st.phi.cpu().numpy()
        e = ph.T @ ph - np.eye(ph.shape[1])
        em = m.phi.T @ m.phi - np.eye(m.r)
        inf = st.info()
        print(j, 'dev: dep', inf.flags & 1, 'trace(E) %+.3e maxabs %.2e | model trace %+.3e maxabs %.2e' %
              (np.trace(e), np.abs(e).max(), np.trace(em), np.abs(em).max()), flush=True)
