import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_1910_01260_b200 import linalg
n = 40
rng = np.random.default_rng(n)
an = rng.standard_normal((n, n)) + n * np.eye(n) * 0.05
bn = rng.standard_normal(n)
a = torch.as_tensor(an, device="cuda")
b = torch.as_tensor(bn, device="cuda")
xr = np.linalg.solve(an, bn)
for rep in range(4):
    x = linalg.solve_dense(a, b)
    xn = x.cpu().numpy()
    print(rep, np.max(np.abs(xn - xr)), float(torch.linalg.norm(a @ x - b)), np.linalg.norm(an @ xn - bn),
          np.max(np.abs(a.cpu().numpy() - an)), x.shape, x.stride(), x.is_contiguous())
