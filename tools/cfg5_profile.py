"""Per-kernel event times of a short cfg5 run (n_s = 2^26, rank 100): which kernel sets the update time.

    python tools/cfg5_profile.py [--log2n 26] [--cols 160] [--timed-from 100]
"""
import argparse
import math
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

from paper_1910_01260_b200 import _capi, basis, workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument('--log2n', type=int, default=26)
ap.add_argument('--cols', type=int, default=160)
ap.add_argument('--timed-from', type=int, default=100)
ap.add_argument('--rank', type=int, default=100)
ap.add_argument('--call-cols', type=int, default=8, help='columns per timed ingest call')
args = ap.parse_args()
n, B = 1 << args.log2n, 8
dev = torch.device('cuda')
stream = wl.HadamardStream(n, 1000, args.rank, decades_per=12.0, seed=0)
buf = torch.empty((B, n), dtype=torch.float64, device=dev)
st = None
t = 0
KINDS = ["u_pass", "reorth_pass", "decide", "core_step", "v_update", "compact_prep", "compact_sweep", "spatial",
         "st", "lu", "window_pass"]
lib = _capi.lib
while t < args.cols:
    nb = min(B, args.cols - t)
    if st is not None:
        nb = 1 << int(math.floor(math.log2(nb)))
    if t >= args.timed_from and args.call_cols > B:
        nb = min(args.call_cols, args.cols - t)
        big = torch.empty((nb, n), dtype=torch.float64, device=dev)
        for j0 in range(0, nb, B):
            stream.batch(t + j0, min(B, nb - j0), out=big[j0:j0 + min(B, nb - j0)])
        x = big.T
    else:
        x = stream.batch(t, nb, out=buf[:nb])
    if t >= args.timed_from and not getattr(lib, '_on', False):
        torch.cuda.synchronize()
        lib.strom_profile_reset()
        lib.strom_profile_enable(1)
        lib._on = True
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()
        t_from = t
    if st is None:
        st = basis.isvd_init(x[:, 0].contiguous(), 1e-9, tol_sv=1e-9, r_max=args.rank, cap_mode='truncate')
        st = basis.ingest_simulation(st, x[:, 1:])
    else:
        st = basis.ingest_simulation(st, x)
    t += nb
e1 = torch.cuda.Event(enable_timing=True)
e1.record()
torch.cuda.synchronize()
lib.strom_profile_enable(0)
pl = (_capi.i64 * 16)()
pms = (_capi.dbl * 16)()
pby = (_capi.dbl * 16)()
lib.strom_profile_read(16, pl, pms, pby)
nupd = args.cols - t_from
print(f'{nupd} updates in {e0.elapsed_time(e1):.1f} ms = {e0.elapsed_time(e1) / nupd:.2f} ms each; rank {st.rank}')
for k, name in enumerate(KINDS):
    if pl[k]:
        gbs = pby[k] / (pms[k] / 1e3) / 1e9 if pms[k] > 0 and pby[k] > 0 else float('nan')
        print(f'  {name:14s} launches {pl[k]:5d}  {pms[k]:9.2f} ms  ({pms[k] / nupd:7.3f} ms/update)  {gbs:8.1f} GB/s')
