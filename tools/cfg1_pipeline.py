"""Config 1 (BASELINE.json configs[0]) end to end on the device, beside the CPU oracle.

Four training marches (fom_march on the device) -> iSVD (tol 1e-8) -> temporal
bases (n_s 10, n_t 4) -> spatial ROM at the test viscosity -> ST operator ->
dense solve -> lifted states, compared with the full-order test march.  Times
are CUDA-event medians over repeats after a warm-up; the CPU column runs the
same stages through the oracle (the reference's algorithm, NumPy/SciPy).

    python tools/cfg1_pipeline.py > out.json
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import strom_oracle as so  # noqa: E402
from paper_1910_01260_b200 import (LinearDynamicalSystem, TimeGrid, basis, fom_march, spacetime,  # noqa: E402
                                   spatial, workloads as wl)


def lds(d):
    return LinearDynamicalSystem(a=d.a, b=d.b, c=d.c, x0=d.x0, input_signal=d.inputs, constant_input=True)


grid = TimeGrid(wl.cfg1_dt())
train = [lds(wl.cfg1_system(nu)) for nu in wl.CFG1_TRAIN_NU]
test = lds(wl.cfg1_system(wl.CFG1_TEST_NU))
for s_ in train + [test]:
    s_.device_arrays()
grid.dt_device()


def run():
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    ev[0].record()
    mats = [fom_march(s_, grid).states for s_ in train]
    ev[1].record()
    st = basis.isvd_init(mats[0][:, 0], wl.CFG1_TOL, tol_sv=wl.CFG1_TOL)
    st = basis.ingest_simulation(st, mats[0][:, 1:])
    for m in mats[1:]:
        st = basis.ingest_simulation(st, m)
    ev[2].record()
    bs = basis.build_basis_set(st, wl.CFG1_NS, wl.CFG1_NTMODES, wl.CFG1_NT, len(wl.CFG1_TRAIN_NU))
    ev[3].record()
    srom = spatial.build_spatial_rom(test, bs, ref_mode="zero")
    rom = spacetime.build_st_rom(srom, bs, grid, test.input_signal, True)
    ev[4].record()
    x_st = spacetime.solve_st_rom(rom)
    states = spacetime.reconstruct_states(bs, x_st)
    ev[5].record()
    torch.cuda.synchronize()
    return [ev[i].elapsed_time(ev[i + 1]) for i in range(5)], ev[0].elapsed_time(ev[5]), st, states


run()
runs = [run() for _ in range(5)]
stage = [statistics.median(r[0][i] for r in runs) for i in range(5)]
total = statistics.median(r[1] for r in runs)
st, states = runs[-1][2], runs[-1][3]
fom_test = fom_march(test, grid).states
rel = (torch.linalg.norm(states - fom_test, dim=0) / torch.linalg.norm(fom_test, dim=0)).cpu().numpy()

# CPU: the same stages through the oracle (one run)
t = [time.perf_counter()]
dt = grid.dt
mats = [so.fom_march(d.a, d.b, d.x0, dt, d.inputs) for d in map(wl.cfg1_system, wl.CFG1_TRAIN_NU)]
t.append(time.perf_counter())
u = np.hstack(mats)
ref = so.stream(u, wl.CFG1_TOL, tol_sv=wl.CFG1_TOL)
t.append(time.perf_counter())
phi_s, temporal, _ = so.basis_set(ref, wl.CFG1_NS, wl.CFG1_NTMODES, wl.CFG1_NT, 4)
t.append(time.perf_counter())
d = wl.cfg1_system(wl.CFG1_TEST_NU)
o = so.spatial_rom(d.a, d.b, d.c, d.x0, phi_s, "zero")
a_st = so.st_matrix(o.a_hat, temporal, dt)
f_st = so.st_input(o.b_hat, temporal, dt, d.inputs, True)
i_st = so.st_init(o.x0_hat, temporal)
t.append(time.perf_counter())
x_ref = so.st_solve(a_st, f_st, i_st)
t.append(time.perf_counter())
cpu = [1e3 * (t[i + 1] - t[i]) for i in range(5)]
names = ["fom_4x100_steps", "isvd_400_snapshots", "temporal_bases", "st_operator_build", "st_solve_and_lift"]
print(json.dumps({
    "config": "cfg1: 1D periodic advection-diffusion, n_s=1024, 4 training nu x 100 backward-Euler steps, "
              "tol 1e-8, n_s=10 spatial x n_t=4 temporal modes, test nu=0.025",
    "device_ms": dict(zip(names, stage)), "device_total_ms": total,
    "device_us_per_snapshot_isvd": stage[1] * 1e3 / 400,
    "cpu_oracle_ms": dict(zip(names, cpu)), "cpu_total_ms": sum(cpu), "cpu_cores": os.cpu_count(),
    "rank": st.rank,
    "st_rom_rel_err_vs_fom": {"max": float(rel.max()), "final": float(rel[-1])},
}), flush=True)
