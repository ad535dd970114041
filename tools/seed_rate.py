"""cfg2 ingestion rate (snapshots 101-500) on the torch-seed streams of bench.py's `seeds` key.

    python tools/seed_rate.py [--seeds 1 2] [--reps 3]
"""
import argparse
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

import numpy as np  # noqa: E402

from paper_1910_01260_b200 import _capi, basis, workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument('--seeds', type=int, nargs='*', default=[1, 2])
ap.add_argument('--reps', type=int, default=3)
ap.add_argument('--trace', action='store_true', help='device trace: gap between a core step\'s end and the next decision')
args = ap.parse_args()
for seed in args.seeds:
    xt, _, _, _ = wl.cfg2_stream_torch(n=1 << 20, cols=500, rank=64, seed=seed)
    q, r = torch.linalg.qr(xt[:100].T)
    w, s, vt = torch.linalg.svd(r)
    st = basis.SvdState((q @ w[:, :64]).contiguous(), s[:64], vt.T[:, :64].contiguous(), 100, 1e-9, tol_sv=1e-9,
                        r_max=64, cap_mode='truncate')
    cols = xt[100:].T
    out = basis.ingest_simulation(st, cols)
    out.rank
    rates = []
    gaps = []
    for _ in range(args.reps):
        if args.trace:
            buf = torch.zeros(400 * 16, dtype=torch.int64, device='cuda')
            _capi.lib.strom_debug_trace(_capi.C.c_void_p(buf.data_ptr()), 400)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = basis.ingest_simulation(st, cols)
        e1.record()
        torch.cuda.synchronize()
        rates.append(400 / (e0.elapsed_time(e1) / 1e3))
        if args.trace:
            _capi.lib.strom_debug_trace(_capi.C.c_void_p(0), 0)
            T = buf.cpu().numpy().reshape(400, 16).astype(np.float64)
            T[T == 0] = np.nan
            g = (T[1:, 0] - T[:-1, 11]) / 1e3  # next A start - this core step's end
            g = g[np.isfinite(g)]
            gaps.append((round(float(np.median(g)), 1), round(float(np.percentile(g, 90)), 1), round(float(g.sum()) / 1e3, 2)))
    if gaps:
        print('  step-end -> next-decision gap (median us, p90 us, total ms):', gaps)
    print(f'seed {seed}: {[round(v) for v in rates]} snapshots/s, dependent {out.n_dependent - st.n_dependent}, '
          f'truncated {out.n_truncated - st.n_truncated}')
    del xt, cols, st, out
    torch.cuda.empty_cache()
