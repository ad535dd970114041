import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_1910_01260_b200 import basis
import device_model as dm
g = np.load('tests/golden/golden_isvd_small.npz')
u = g['heat_in']
st = basis.isvd_init(u[:, 0], tol_svd=0.0)
m = dm.init(u[:, 0], 0.0)
for j in range(1, u.shape[1]):
    st = basis.isvd_update(st, u[:, j])
    m = dm.update(m, u[:, j])
    inf = st.info()
    print(j, 'dev r', inf.rank, 'c', inf.ncols_u, 'flags', inf.flags, 'p %.2e' % inf.last_p, '| model r', m.r, 'c', m.U.shape[1], m.flags.get('dep'), m.flags.get('appended'), '%.2e' % m.flags.get('p', 0))
