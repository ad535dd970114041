"""Per-update timeline of window-mode iSVD ingestion (strom_debug_trace): median
microseconds of each phase relative to the update's k_decide_a start, and the
update-to-update period.

    python tools/trace_isvd.py [--cols 120]
"""
import argparse
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1910_01260_b200 import _capi, basis, workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument('--cols', type=int, default=120)
ap.add_argument('--uncapped', action='store_true', help='r_max = None (the cfg1 / cfg3 setting)')
ap.add_argument('--tol', type=float, default=1e-9)
args = ap.parse_args()
xt, _, _, _ = wl.cfg2_stream_torch(n=1 << 20, cols=100 + args.cols, rank=64, seed=0)
if args.uncapped:
    st = basis.isvd_init(xt[0], args.tol, tol_sv=args.tol)
else:
    st = basis.isvd_init(xt[0], args.tol, tol_sv=args.tol, r_max=64, cap_mode='truncate')
st = basis.ingest_simulation(st, xt[1:100].T)
basis.ingest_simulation(st, xt[100:].T).rank  # warm
buf = torch.zeros(args.cols * 16, dtype=torch.int64, device='cuda')
_capi.lib.strom_debug_trace(_capi.C.c_void_p(buf.data_ptr()), args.cols)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
out = basis.ingest_simulation(st, xt[100:].T)
e1.record()
torch.cuda.synchronize()
_capi.lib.strom_debug_trace(_capi.C.c_void_p(0), 0)
print(f'{args.cols} updates in {e0.elapsed_time(e1):.2f} ms = {e0.elapsed_time(e1) * 1e3 / args.cols:.1f} us each; '
      f'dependent {out.n_dependent - st.n_dependent}')
T = buf.cpu().numpy().reshape(args.cols, 16).astype(np.float64)
T[T == 0] = np.nan
names = ['A start', 'A end', 'resid start', 'resid end', 'B start', 'B end', 'second start', 'decide2 end',
         'stepb start', 'stepb svd done', 'stepb mid ok', 'stepb end', 'vupd start', 'resid reduced', 'wproj start',
         'prep_w end']
rel = (T - T[:, [0]]) / 1e3
print('phase (us from A start): median [p10, p90]   (n)')
for k in range(16):
    v = rel[:, k]
    v = v[np.isfinite(v)]
    if v.size:
        print(f'  {names[k]:15s} {np.median(v):8.1f} [{np.percentile(v, 10):7.1f}, {np.percentile(v, 90):7.1f}]  ({v.size})')
ind = np.isfinite(T[:, 3])
for label, sel in (('independent', ind), ('dependent', ~ind)):
    print(f'-- {label} updates only ({int(sel.sum())}): median [p10, p90]')
    for k in range(14):
        v = rel[sel, k]
        v = v[np.isfinite(v)]
        if v.size:
            print(f'  {names[k]:15s} {np.median(v):8.1f} [{np.percentile(v, 10):7.1f}, {np.percentile(v, 90):7.1f}]')
    nxt = (T[1:, 0] - T[:-1, 0]) / 1e3
    v = nxt[sel[:-1]]
    v = v[np.isfinite(v)]
    print(f'  next A start    {np.median(v):8.1f} [{np.percentile(v, 10):7.1f}, {np.percentile(v, 90):7.1f}]')
per = np.diff(T[:, 0]) / 1e3
print(f'A-to-A period: median {np.nanmedian(per):.1f} us, mean {np.nanmean(per):.1f}')
dep = np.isnan(T[:, 3])
print(f'period after dependent: {np.nanmedian(per[dep[:-1]]):.1f} us; after independent: '
      f'{np.nanmedian(per[~dep[:-1]]):.1f} us')
