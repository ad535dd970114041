"""Short cfg2 ingestion run for ncu: warm state at 100 snapshots, then `--cols` updates."""
import argparse
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

from paper_1910_01260_b200 import basis, workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument('--n', type=int, default=1 << 20)
ap.add_argument('--cols', type=int, default=40)
ap.add_argument('--tol', type=float, default=1e-9)
args = ap.parse_args()
xt, _, _, _ = wl.cfg2_stream_torch(n=args.n, cols=100 + args.cols, rank=64, seed=0)
st = basis.isvd_init(xt[0], args.tol, tol_sv=args.tol, r_max=64, cap_mode='truncate')
st = basis.ingest_simulation(st, xt[1:100].T)
torch.cuda.synchronize()
out = basis.ingest_simulation(st, xt[100:].T)
torch.cuda.synchronize()
print('rank', out.rank, 'dependent', out.n_dependent, 'truncated', out.n_truncated)
