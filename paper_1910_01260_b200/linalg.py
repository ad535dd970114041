"""Dense fp64 kernels of the reference ``strom.linalg`` (linalg.py:19-108), on the device.

``thin_svd`` and ``qr`` keep the reference's deterministic sign conventions
(largest-|.| entry of each left singular vector >= 0; diag(R) >= 0) and
``solve_dense`` its pivot floor and error message.  All run as sm_100a
kernels; inputs may be numpy arrays or tensors, outputs are CUDA tensors.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _capi as capi
from ._tensors import F64, colmajor, device, to_dev
from .errors import ConvergenceError, SingularMatrixError  # noqa: F401  (re-exported names)

__all__ = ["SingularMatrixError", "ConvergenceError", "thin_svd", "qr", "solve_dense", "kron"]


def _cm(m: torch.Tensor) -> torch.Tensor:
    """Column-major copy of a 2-D tensor as a flat storage owner (always a copy:
    ``t().contiguous()`` would alias an (n, 1) input, and the kernels work in place)."""
    out = torch.empty((m.shape[1], m.shape[0]), dtype=m.dtype, device=m.device)
    out.copy_(m.t())
    return out  # (cols, rows) row-major == (rows, cols) column-major


def thin_svd(m):
    """Thin SVD ``m = w @ diag(sigma) @ v.T`` with deterministic signs (linalg.py:41-57)."""
    m = to_dev(m)
    if m.dim() != 2 or min(m.shape) < 1:
        raise ValueError(f"need a non-empty 2-D matrix, got shape {tuple(m.shape)}")
    if not bool(torch.isfinite(m).all()):
        raise ValueError("matrix has non-finite entries")
    rows, cols = m.shape
    kmin = min(rows, cols)
    dev = device()
    w = torch.empty((kmin, rows), dtype=F64, device=dev)   # column-major rows x kmin
    s = torch.empty((kmin,), dtype=F64, device=dev)
    v = torch.empty((kmin, cols), dtype=F64, device=dev)   # column-major cols x kmin
    a = _cm(m)
    capi.call("strom_thin_svd", rows, cols, a.data_ptr(), w.data_ptr(), s.data_ptr(), v.data_ptr(),
              capi.stream_ptr())
    return w.t(), s, v.t()


def _temporal_batch(v_cm: torch.Tensor, k: int, r: int, n_steps: int, n_mu: int, n_s: int, n_t: int):
    """All n_s temporal SVDs in one launch; v_cm is the k x r matrix column-major (r, k) storage."""
    dev = device()
    psi = torch.empty((n_s, n_steps, n_t), dtype=F64, device=dev)
    ranks = torch.empty((n_s,), dtype=torch.int32, device=dev)
    sig = torch.empty((n_s, min(n_steps, n_mu)), dtype=F64, device=dev)
    capi.call("strom_temporal_bases", v_cm.data_ptr(), k, r, n_steps, n_mu, n_s, n_t, psi.data_ptr(),
              ranks.data_ptr(), sig.data_ptr(), capi.stream_ptr())
    return psi, ranks.cpu(), sig


def qr(m):
    """Reduced QR with diag(R) >= 0 (linalg.py:60-72); single-CTA Householder on the device."""
    m = to_dev(m)
    if m.dim() != 2 or m.shape[0] < m.shape[1]:
        raise ValueError(f"need rows >= cols, got shape {tuple(m.shape)}")
    rows, cols = m.shape
    q = _cm(m)
    r = torch.zeros((cols, cols), dtype=F64, device=device())  # column-major
    capi.call("strom_qr", rows, cols, q.data_ptr(), rows, r.data_ptr(), capi.stream_ptr())
    return q.t(), r.t()


def solve_dense(a, b):
    """Solve a x = b by LU with partial pivoting (linalg.py:75-99).

    Raises SingularMatrixError naming the first pivot with |U_ii| <= 1e-14 ||a||_F.
    """
    a = to_dev(a)
    b = to_dev(b)
    if a.dim() != 2 or a.shape[0] != a.shape[1]:
        raise ValueError(f"matrix must be square, got shape {tuple(a.shape)}")
    if b.shape[0] != a.shape[0]:
        raise ValueError(f"dimension mismatch: {tuple(a.shape)} vs {tuple(b.shape)}")
    n = a.shape[0]
    vec = b.dim() == 1
    bm = b.reshape(n, -1)
    nrhs = bm.shape[1]
    lu = _cm(a)
    x = _cm(bm)
    capi.call("strom_dense_solve", n, lu.data_ptr(), x.data_ptr(), nrhs, None, None, capi.stream_ptr())
    x = x.t()
    return x.reshape(n) if vec else x


def kron(a, b):
    """Kronecker product (linalg.py:102-108); oracle helper, not on the hot path."""
    a, b = to_dev(a), to_dev(b)
    if not (bool(torch.isfinite(a).all()) and bool(torch.isfinite(b).all())):
        raise ValueError("kron factors must be finite")
    return torch.kron(a, b)


class AdjointConsistencyError(Exception):
    """``apply_adjoint`` is not the transpose of ``apply`` (linalg.py:27-28)."""


def largest_singular_value(apply, apply_adjoint, dim_in: int, dim_out: int, tol: float = 1e-8,
                           max_iter: int = 10_000, seed: int = 0) -> float:
    """Largest singular value of a linear map by power iteration on A^T A (linalg.py:111-171).

    Same protocol as the reference: three random adjoint-consistency probes,
    then sweeps until the estimate is stable to ``tol`` twice in a row; the
    start vectors come from ``numpy.random.default_rng(seed)`` in the
    reference's draw order, and the applies run on device vectors.
    """
    from .errors import ConvergenceError

    rng = np.random.default_rng(seed)

    def dev(x):
        return torch.as_tensor(x, dtype=F64, device=device())

    for _ in range(3):
        v = rng.standard_normal(dim_in)
        w = rng.standard_normal(dim_out)
        v /= np.linalg.norm(v)
        w /= np.linalg.norm(w)
        lhs = float(torch.dot(apply(dev(v)), dev(w)))
        rhs = float(torch.dot(dev(v), apply_adjoint(dev(w))))
        if abs(lhs - rhs) > 1e-10 * max(1.0, abs(lhs), abs(rhs)):
            raise AdjointConsistencyError(f"<Av, w> = {lhs:.16e} but <v, A^T w> = {rhs:.16e}")
    v = rng.standard_normal(dim_in)
    v = dev(v / np.linalg.norm(v))
    sigma, stable, gap = 0.0, 0, np.inf
    for _ in range(max_iter):
        t = apply_adjoint(apply(v))
        lam = float(torch.linalg.norm(t))
        if lam == 0.0:
            v = rng.standard_normal(dim_in)
            v = dev(v / np.linalg.norm(v))
            t = apply_adjoint(apply(v))
            lam = float(torch.linalg.norm(t))
            if lam == 0.0:
                return 0.0
        new_sigma = float(np.sqrt(lam))
        v = t / lam
        gap = abs(new_sigma - sigma)
        if gap <= tol * max(new_sigma, np.finfo(float).tiny):
            stable += 1
            if stable >= 2:
                return new_sigma
        else:
            stable = 0
        sigma = new_sigma
    raise ConvergenceError(f"power iteration failed to converge in {max_iter} iterations "
                           f"(last estimate {sigma:.6e}, last gap {gap:.3e})")
