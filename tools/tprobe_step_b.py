"""Phase timestamps (clock64) inside k_step_b / the core SVD for steady-state cfg2
updates (strom_debug_tprobe).  Prints the median cycles per phase.

    python tools/tprobe_step_b.py [--cols 40]
"""
import argparse
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1910_01260_b200 import _capi, basis, workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument('--cols', type=int, default=40)
ap.add_argument('--pipelined', action='store_true')
ap.add_argument('--rmax', type=int, default=64)
ap.add_argument('--n', type=int, default=1 << 20)
ap.add_argument('--noise', type=float, default=1e-12)
ap.add_argument('--hadamard', action='store_true', help='the cfg5 stream (rank --rmax, sigma_i = 10^(-i/12))')
args = ap.parse_args()
warm = max(100, args.rmax + 40)
if args.hadamard:
    hs = wl.HadamardStream(args.n, 1000, args.rmax, decades_per=12.0, seed=0)
    ncol = warm + args.cols + 24
    xt = torch.cat([hs.batch(t0, min(16, ncol - t0)).T for t0 in range(0, ncol, 16)], 0).contiguous()
else:
    xt, _, _, _ = wl.cfg2_stream_torch(n=args.n, cols=warm + args.cols + 24, rank=args.rmax, seed=0, noise=args.noise)
st = basis.isvd_init(xt[0], 1e-9, tol_sv=1e-9, r_max=args.rmax, cap_mode='truncate')
st = basis.ingest_simulation(st, xt[1:warm].T)
buf = torch.zeros(512, dtype=torch.int64, device='cuda')
_capi.lib.strom_debug_tprobe(_capi.C.c_void_p(buf.data_ptr()))
rows = []
if args.pipelined:
    # the probes of the LAST update of a pipelined multi-column ingest (warm instruction cache,
    # neighbours running): one sample per call
    for q in range(args.cols):
        buf.zero_()
        basis.ingest_simulation(st, xt[warm:warm + 24 + q].T).rank
        torch.cuda.synchronize()
        rows.append(buf.cpu().numpy().copy())
else:
    for t in range(warm, warm + args.cols):
        buf.zero_()
        st = basis.ingest_simulation(st, xt[t:t + 1].T)
        torch.cuda.synchronize()
        b = buf.cpu().numpy()
        rows.append(b.copy())
_capi.lib.strom_debug_tprobe(_capi.C.c_void_p(0))
R = np.array(rows)
names = {0: 'B0 start', 1: 'B1 setup', 2: 'B2 core svd', 3: 'B3', 4: 'B4 N update', 5: 'B5 drift', 6: 'B6 qr'}
base = R[:, 0]
print('step_b phases (cycles from B0, median over updates; QR count %d)' % int((R[:, 7] > 0).sum()))
for k in range(1, 7):
    ok = R[:, k] > 0
    if ok.any():
        print(f'  {names.get(k, k):14s} {np.median(R[ok, k] - base[ok]):10.0f}')
print('QR kinds (1 CholeskyQR, 2 Householder):', sorted(set(int(v) for v in R[:, 7])), ' QR sub-phases pass 0 (cycles from B5):',
      [int(np.median(R[R[:, 280 + k] > 0, 280 + k] - R[R[:, 280 + k] > 0, 5])) if (R[:, 280 + k] > 0).any() else None for k in range(6)])
print('core svd phases (cycles from CORE_TP(0))')
c0 = R[:, 300]
for k in range(301, 308):
    ok = R[:, k] > 0
    if ok.any():
        print(f'  core {k - 300}: {np.median(R[ok, k] - c0[ok]):10.0f}')
it = R[:, 8:8 + args.rmax + 2]
print('root iterations: median over roots', np.median(it), ' max per update (median over updates)',
      np.median(it.max(axis=1)), ' max overall', it.max())
