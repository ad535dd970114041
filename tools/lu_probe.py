import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1910_01260_b200 import linalg
n = 1000
rng = np.random.default_rng(n)
a = torch.as_tensor(rng.standard_normal((n, n)) + n * np.eye(n) * 0.05, device="cuda")
b = torch.as_tensor(rng.standard_normal(n), device="cuda")
for _ in range(2):
    x = linalg.solve_dense(a, b)
torch.cuda.synchronize()
print("ok")
