"""Lock-step decision statistics on noise steps (diagnostics): device vs oracle from the oracle's state."""
import sys

import numpy as np

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from paper_1910_01260_b200 import basis, workloads as wl  # noqa: E402
from oracle import strom_oracle as so  # noqa: E402
from helpers import factor_state  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
cols = int(sys.argv[2]) if len(sys.argv) > 2 else 200
x, _, _, _ = wl.cfg2_stream_numpy(n=n, cols=cols)
x = np.ascontiguousarray(x)
ref = so.init(x[:, 0], 1e-9, tol_sv=1e-9, r_max=64, cap_mode='truncate')
agree = dis = dep_dev = dep_ref = 0
rows = []
for t in range(1, cols):
    d = so.Decision()
    nxt = so.update(ref, x[:, t], d)
    if t >= 70:
        u, w = factor_state(ref.phi)
        dev = basis.SvdState.from_factors(u, w, ref.sigma, ref.v, ref.k, 1e-9, 1e-9, 64, 'truncate')
        got = basis.isvd_update(dev, x[:, t])
        inf = got.info()
        dd = bool(inf.flags & 1)
        # exact-ish p^2 in long double from the oracle's phi
        phl = ref.phi.astype(np.longdouble)
        xl = x[:, t].astype(np.longdouble)
        ell = phl.T @ xl
        p2l = float(xl @ xl - ell @ ell)
        dep_dev += dd
        dep_ref += d.dependent
        agree += dd == d.dependent
        rows.append((t, d.p_sq, p2l, inf.last_p, dd, d.dependent))
    ref = nxt
print('steps', len(rows), 'agree', agree, 'dep dev', dep_dev, 'dep ref', dep_ref)
for r in rows[:40]:
    print('t %d ref p2 %+.3e  longdouble p2 %+.3e  dev p %.3e  dep dev %d ref %d' % r)
