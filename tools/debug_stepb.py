"""Phase timing of step B (clock64 probes) on steady-state cfg2 updates."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1910_01260_b200 import _capi, basis, workloads as wl
xt, _, _, _ = wl.cfg2_stream_torch(n=1 << 20, cols=130, rank=64, seed=0)
st = basis.isvd_init(xt[0], 1e-9, tol_sv=1e-9, r_max=64, cap_mode='truncate')
st = basis.ingest_simulation(st, xt[1:100].T)
buf = torch.zeros(320, dtype=torch.int64, device='cuda')
_capi.lib.strom_debug_tprobe(buf.data_ptr())
names = ['L/Li copy+wj', 'secular SVD', 'NS polish', 'trunc+W update', 'drift', 'QR', ]
for j in range(100, 130):
    buf.zero_()
    st = basis.isvd_update(st, xt[j])
    inf = st.info()
    t = buf.cpu().tolist()
    d = [(t[k + 1] - t[k]) / 1.965e3 for k in range(6)]
    print('   use_smem/qr path', t[7])
    cp = t[300:308]
    print('   core phases', ' '.join(f'{(cp[k+1]-cp[k])/1.965e3:.1f}' for k in range(7)), '(defl roots GE vec rot sort sign)')
    its = t[8:8 + inf.rank + 1]
    print('   iters max', max(its), 'mean', sum(its) / len(its), 'n>=99', sum(1 for v in its if v >= 99))
    q = t[280:292]
    if q[5] > 0:
        print('   qr phases', ' '.join(f'{(q[k+1]-q[k])/1.965e3:.1f}' for k in range(11)), '(gram chol inv gemm copy | ...)')
    print('upd', j, 'flags', inf.flags, 'c', inf.ncols_u, ' '.join(f'{n}={v:.1f}us' for n, v in zip(names, d) if v > 0))
_capi.lib.strom_debug_tprobe(None)
