"""Split the dense solve at n = 1000 into the LU factorisation and the two
triangular solves (C ABI strom_dense_lu / strom_dense_lu_solve), CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1910_01260_b200 import _capi as capi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
rng = np.random.default_rng(n)
a0 = torch.as_tensor((rng.standard_normal((n, n)) + n * np.eye(n) * 0.05).T.copy(), device="cuda")  # column-major
b0 = torch.as_tensor(rng.standard_normal(n), device="cuda")
piv = torch.empty(n, dtype=torch.int32, device="cuda")
tf, ts = [], []
for _ in range(7):
    a = a0.clone()
    x = b0.clone()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    capi.call("strom_dense_lu", n, a.data_ptr(), piv.data_ptr(), capi.stream_ptr())
    e[1].record()
    capi.call("strom_dense_lu_solve", n, a.data_ptr(), piv.data_ptr(), x.data_ptr(), 1, capi.stream_ptr())
    e[2].record()
    torch.cuda.synchronize()
    tf.append(e[0].elapsed_time(e[1]))
    ts.append(e[1].elapsed_time(e[2]))
print(f"n={n}: factor {sorted(tf)[3]:.3f} ms, solve {sorted(ts)[3]:.3f} ms")
