"""Transport-proxy configuration (BASELINE.json configs[2]) on one B200.

64^3 cells x 4 directions (2^20 dofs), backward Euler dt = 0.01, 100 steps, four
source amplitudes.  Snapshots come from the device full-order march
(fom_march: cooperative BiCGSTAB kernel, system.py:150-163) and are ingested by
the device iSVD (tol 1e-8) straight from HBM, sample-major like
pipeline.train; then the per-mode temporal bases (n_t = 2: the system is linear
in the amplitude).  The reference cannot produce these
snapshots (SuperLU at 32^3 x 4 took 209 s); parity is checked at 12^3 x 4 in
tests/test_gpu_fom.py.

    python tools/cfg3_transport.py [--nc 64] > out.json
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1910_01260_b200 import (LinearDynamicalSystem, TimeGrid, basis, fom_march,  # noqa: E402
                                   workloads as wl)

ap = argparse.ArgumentParser()
ap.add_argument("--nc", type=int, default=wl.CFG3_NC)
ap.add_argument("--steps", type=int, default=wl.CFG3_NT)
ap.add_argument("--ns", type=int, default=10)
args = ap.parse_args()
t_all = time.time()
t0 = time.time()
a = wl.cfg3_operator(args.nc)
t_op = time.time() - t0
grid = TimeGrid(np.full(args.steps, wl.CFG3_DT))
st = None
fom_s, ingest_ms, iters = [], [], []
for amp in wl.CFG3_AMPLITUDES:
    d = wl.cfg3_system(amp, nc=args.nc, a=a)
    sys_ = LinearDynamicalSystem(a=d.a, b=d.b, c=d.c, x0=d.x0, input_signal=d.inputs, constant_input=True)
    sys_.device_arrays()
    res = fom_march(sys_, grid)
    fom_s.append(res.wall_time)
    iters += res.iterations
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if st is None:
        st = basis.isvd_init(res.states[:, 0], wl.CFG3_TOL, tol_sv=wl.CFG3_TOL)
        st = basis.ingest_simulation(st, res.states[:, 1:])
    else:
        st = basis.ingest_simulation(st, res.states)
    e1.record()
    torch.cuda.synchronize()
    ingest_ms.append(e0.elapsed_time(e1))
    del res
n_s = min(args.ns, st.rank)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
bs = basis.build_basis_set(st, n_s, 2, args.steps, len(wl.CFG3_AMPLITUDES))
e1.record()
torch.cuda.synchronize()
nsnap = args.steps * len(wl.CFG3_AMPLITUDES)
n = a.shape[0]
sig = st.sigma.cpu().numpy()
out = {
    "config": f"cfg3 transport proxy: {args.nc}^3 cells x 4 directions ({n} dofs), sigma_t 1, sigma_s 0.5, "
              f"backward Euler dt {wl.CFG3_DT}, {args.steps} steps, amplitudes {list(wl.CFG3_AMPLITUDES)}, "
              "iSVD tol 1e-8",
    "operator_build_s_host": t_op,
    "fom": {"s_per_sample": fom_s, "ms_per_step": float(np.mean(fom_s)) / args.steps * 1e3,
            "bicgstab_iterations_mean": float(np.mean(iters)), "bicgstab_iterations_max": int(np.max(iters)),
            "solver": "BiCGSTAB on the left-Jacobi-preconditioned step system, relative residual 1e-13, one cooperative kernel per march"},
    "isvd": {"snapshots": nsnap, "ingest_ms": ingest_ms, "snapshots_per_s": nsnap / (sum(ingest_ms) / 1e3),
             "rank": st.rank, "counters": {"n_dependent": st.n_dependent, "n_truncated": st.n_truncated},
             "sigma_head": sig[:8].tolist(), "sigma_tail": sig[-3:].tolist()},
    "temporal_bases": {"n_s": n_s, "n_t": 2, "ms": e0.elapsed_time(e1),
                       "orthonormality_defect": float(bs.orthonormality_defect())},
    "wall_s": time.time() - t_all,
}
print(json.dumps(out), flush=True)
