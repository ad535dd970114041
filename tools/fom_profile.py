"""One cfg1 training march (n = 1024, 100 steps) for an ncu capture of the
single-CTA k_fom_march: python tools/fom_profile.py [nu_index]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1910_01260_b200 import LinearDynamicalSystem, TimeGrid, fom_march, workloads as wl  # noqa: E402

nu = wl.CFG1_TRAIN_NU[int(sys.argv[1]) if len(sys.argv) > 1 else 0]
d = wl.cfg1_system(nu)
s = LinearDynamicalSystem(a=d.a, b=d.b, c=d.c, x0=d.x0, input_signal=d.inputs, constant_input=True)
grid = TimeGrid(wl.cfg1_dt())
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = fom_march(s, grid)
    e1.record()
    torch.cuda.synchronize()
its = sum(res.iterations)
print(f"nu {nu}: {e0.elapsed_time(e1):.3f} ms, {its} iterations, {1e3 * e0.elapsed_time(e1) / its:.2f} us/iteration")
