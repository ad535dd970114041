"""Time linalg.solve_dense (device LU) on a well-conditioned n x n system."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1910_01260_b200 import linalg  # noqa: E402

for n in (40, 500, 1000, 1200):
    rng = np.random.default_rng(n)
    a = torch.as_tensor(rng.standard_normal((n, n)) + n * np.eye(n) * 0.05, device="cuda")
    b = torch.as_tensor(rng.standard_normal(n), device="cuda")
    x = linalg.solve_dense(a, b)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x = linalg.solve_dense(a, b)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res = float(torch.linalg.norm(a @ x - b) / torch.linalg.norm(b))
    print(f"n={n} solve ms median {sorted(ts)[2]:.3f} residual {res:.2e}")
