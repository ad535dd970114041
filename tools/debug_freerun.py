"""Free-running device: is the device's p^2 biased relative to its own state? (diagnostics)"""
import sys

import numpy as np

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from paper_1910_01260_b200 import basis, workloads as wl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
cols = int(sys.argv[2]) if len(sys.argv) > 2 else 160
x, _, _, _ = wl.cfg2_stream_numpy(n=n, cols=cols)
x = np.ascontiguousarray(x)
st = basis.isvd_init(x[:, 0], 1e-9, tol_sv=1e-9, r_max=64, cap_mode='truncate')
for t in range(1, cols):
    if t >= 60:
        phi = st.phi.cpu().numpy()
        xt = x[:, t]
        ell = phi.T @ xt
        p2d = float(xt @ xt - ell @ ell)
        phl = phi.astype(np.longdouble)
        xl = xt.astype(np.longdouble)
        el = phl.T @ xl
        p2l = float(xl @ xl - el @ el)
        e = phi.T @ phi - np.eye(phi.shape[1])
        a = np.linalg.lstsq(phi, xt, rcond=None)[0]
        bias = -float(a @ e @ a)
    st = basis.isvd_update(st, x[:, t])
    inf = st.info()
    if t >= 60:
        ph2 = st.phi.cpu().numpy()
        e2 = ph2.T @ ph2 - np.eye(ph2.shape[1])
        print('   after: maxabs(E) %.2e trace(E) %+.2e  flags %d' % (np.abs(e2).max(), np.trace(e2), inf.flags))
        print('t %3d dev p2 %+.3e | numpy p2 on dev phi %+.3e | longdouble %+.3e | -a^T E a %+.3e | dep %d qr %d c %d'
              % (t, inf.last_p_sq, p2d, p2l, bias, inf.flags & 1, bool(inf.flags & 4), inf.ncols_u), flush=True)
u, w, lm = (t.cpu().numpy() for t in st.factors())
g = u.T @ u
li = np.linalg.inv(lm)
d = li @ g @ li.T - np.eye(g.shape[0])
print('representation: c', u.shape[1], 'max|L^-1 G L^-T - I| %.2e trace %+.2e' % (np.abs(d).max(), np.trace(d)))
e_small = w.T @ g @ w - np.eye(w.shape[1])
print('E small-space maxabs %.2e trace %+.2e' % (np.abs(e_small).max(), np.trace(e_small)))
