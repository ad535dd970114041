"""ncu targets beyond the cfg2 stream (tools/profile_isvd.py): the cfg4 operator build,
its dense solve and reconstruct_states, and the cfg1 temporal bases.

    python tools/prof_targets.py st|cfg1 [reps]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1910_01260_b200 import (BasisSet, LinearDynamicalSystem, TimeGrid, basis, spacetime, spatial,  # noqa: E402
                                   workloads as wl)

what = sys.argv[1] if len(sys.argv) > 1 else "st"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
if what == "st":
    d = wl.cfg4_inputs()
    sys_ = LinearDynamicalSystem(a=d.a, b=d.b, c=d.c, x0=d.x0, input_signal=d.inputs, constant_input=True)
    phi = torch.as_tensor(np.asfortranarray(d.phi_s).T.copy(), device="cuda").T
    bs = BasisSet(phi, torch.as_tensor(np.stack(d.temporal), device="cuda"), n_mu=20)
    grid = TimeGrid(d.dt)
    for _ in range(reps):
        srom = spatial.build_spatial_rom(sys_, bs, ref_mode="zero")
        rom = spacetime.build_st_rom(srom, bs, grid, sys_.input_signal, True)
        x = spacetime.solve_st_rom(rom)
        states = spacetime.reconstruct_states(bs, x)
        torch.cuda.synchronize()
        del states
    print("st ok", float(x[0]))
elif what == "cfg1":
    grid = TimeGrid(wl.cfg1_dt())
    mats = []
    for nu in wl.CFG1_TRAIN_NU:
        dd = wl.cfg1_system(nu)
        s_ = LinearDynamicalSystem(a=dd.a, b=dd.b, c=dd.c, x0=dd.x0, input_signal=dd.inputs, constant_input=True)
        from paper_1910_01260_b200 import fom_march
        mats.append(fom_march(s_, grid).states)
    st = basis.isvd_init(mats[0][:, 0], wl.CFG1_TOL, tol_sv=wl.CFG1_TOL)
    st = basis.ingest_simulation(st, mats[0][:, 1:])
    for m in mats[1:]:
        st = basis.ingest_simulation(st, m)
    for _ in range(reps):
        bs = basis.build_basis_set(st, wl.CFG1_NS, wl.CFG1_NTMODES, wl.CFG1_NT, 4)
    torch.cuda.synchronize()
    print("cfg1 ok", st.rank)
