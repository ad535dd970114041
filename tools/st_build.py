"""cfg4 ST-ROM operator build, repeated (diagnostics / ncu target)."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1910_01260_b200 import (BasisSet, LinearDynamicalSystem, TimeGrid, spacetime, spatial,  # noqa: E402
                                   workloads as wl)

layout = sys.argv[1] if len(sys.argv) > 1 else "cm"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
d = wl.cfg4_inputs()
sys_ = LinearDynamicalSystem(a=d.a, b=d.b, c=d.c, x0=d.x0, input_signal=d.inputs, constant_input=True)
dev = torch.device("cuda")
if layout == "cm":
    phi = torch.as_tensor(np.asfortranarray(d.phi_s).T.copy(), device=dev).T
else:
    phi = torch.as_tensor(np.ascontiguousarray(d.phi_s), device=dev)
bs = BasisSet(phi, torch.as_tensor(np.stack(d.temporal), device=dev), n_mu=20)
grid = TimeGrid(d.dt)
sys_.device_arrays()
grid.dt_device()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    srom = spatial.build_spatial_rom(sys_, bs, ref_mode="zero")
    rom = spacetime.build_st_rom(srom, bs, grid, sys_.input_signal, True)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(layout, 'build ms', ['%.3f' % t for t in ts], flush=True)
