"""Timeline of the persistent LU (strom_debug_lu_probe): per block column, when it
saw the previous panel, finished its update, published its panel; RHS CTA phases.

    python tools/lu_probe_timeline.py [n]
"""
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1910_01260_b200 import _capi, linalg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
rng = np.random.default_rng(0)
a = rng.standard_normal((n, n)) + 0.5 * np.sqrt(n) * np.eye(n)
b = rng.standard_normal(n)
nb = (n + 15) // 16 + 1
buf = torch.zeros(nb * 8 + 64, dtype=torch.int64, device='cuda')
for _ in range(3):
    linalg.solve_dense(a, b)
_capi.lib.strom_debug_lu_probe(_capi.C.c_void_p(buf.data_ptr()))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
linalg.solve_dense(a, b)
e1.record()
torch.cuda.synchronize()
_capi.lib.strom_debug_lu_probe(_capi.C.c_void_p(0))
print('solve_dense ms', e0.elapsed_time(e1))
B = buf.cpu().numpy()
P = B[:nb * 8].reshape(nb, 8).astype(np.float64)
CP = B[nb * 8:nb * 8 + 48].astype(np.float64)
t0 = P[:, 0][P[:, 0] > 0].min()
P = np.where(P > 0, (P - t0) / 1e3, np.nan)  # us
print('cta  start  wait_last  saw_last  factor_start  published  final')
for j in list(range(0, 6)) + list(range(nb - 6, nb)):
    print(j, ' '.join(f'{v:8.1f}' for v in P[j, :6]))
A = P[:-1]
upd = A[1:, 3] - A[1:, 2]      # last update (panel j-1 -> j), us
fac = A[:, 4] - A[:, 3]        # own panel factorisation
hand = A[1:, 2] - A[:-1, 4]    # publish(j-1) -> seen by j
print(f'median per step: handoff {np.nanmedian(hand):.2f} us, update {np.nanmedian(upd):.2f} us, '
      f'factor {np.nanmedian(fac):.2f} us')
print(f'RHS: forward done {P[-1, 3]:.1f} us, all fin seen {P[-1, 4]:.1f} us, back-sub done {P[-1, 5]:.1f} us')

cp = (CP - CP[0]) / 1e3
print('panel of CTA 1, per column (us from column 0 start): pre-barrier1, post-barrier1, post-barrier2')
for c in range(16):
    print(c, ' '.join(f'{cp[3 * c + k]:7.2f}' for k in range(3)))
