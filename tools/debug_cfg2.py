"""Free-running device iSVD vs the oracle on a scaled config-2 stream (diagnostics)."""
import sys

import numpy as np

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from paper_1910_01260_b200 import basis, workloads as wl  # noqa: E402
from oracle import strom_oracle as so  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
cols = int(sys.argv[2]) if len(sys.argv) > 2 else 300
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 0
x, _, _, _ = wl.cfg2_stream_numpy(n=n, cols=cols, seed=seed)
x = np.ascontiguousarray(x)
st = basis.isvd_init(x[:, 0], 1e-9, tol_sv=1e-9, r_max=64, cap_mode='truncate')
r = so.init(x[:, 0], 1e-9, tol_sv=1e-9, r_max=64, cap_mode='truncate')
c = dict(dq=0, rq=0, dd=0, rd=0, dt=0, rt=0)
for j in range(1, cols):
    st = basis.isvd_update(st, x[:, j])
    d = so.Decision()
    r = so.update(r, x[:, j], d)
    inf = st.info()
    c['dq'] += bool(inf.flags & 4); c['rq'] += d.qr; c['dd'] += bool(inf.flags & 1); c['rd'] += d.dependent
    c['dt'] += bool(inf.flags & 2); c['rt'] += d.truncated
    if j % 25 == 0 or j < 4:
        phi = st.phi.cpu().numpy()
        print(j, 'rank', inf.rank, r.rank, 'ncols', inf.ncols_u, c, 'p dev %.3e ref %.3e' % (inf.last_p, d.p),
              'orth dev %.2e ref %.2e' % (np.abs(phi.T @ phi - np.eye(inf.rank)).max(),
                                          np.abs(r.phi.T @ r.phi - np.eye(r.rank)).max()),
              'sig0 rel %.2e' % (abs(st.sigma[0].item() - r.sigma[0]) / r.sigma[0]), flush=True)
