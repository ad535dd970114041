"""Tensor plumbing: everything the kernels see is float64 CUDA memory."""

from __future__ import annotations

import numpy as np
import torch

F64 = torch.float64


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1910_01260_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def to_dev(a, *, contiguous: bool = True) -> torch.Tensor:
    """float64 CUDA tensor view/copy of a numpy array, python sequence or tensor."""
    if isinstance(a, torch.Tensor):
        t = a.to(device=device(), dtype=F64)
    else:
        t = torch.as_tensor(np.asarray(a, dtype=np.float64), device=device())
    return t.contiguous() if contiguous else t


def colmajor(a: torch.Tensor) -> tuple[torch.Tensor, int]:
    """Return (storage-owning tensor, leading dimension) with columns contiguous.

    ``a`` is (rows, cols); the result T satisfies a[:, j] == T.flatten()[j*ld : j*ld+rows].
    """
    rows = a.shape[0]
    if a.dim() != 2:
        raise ValueError("expected a 2-D matrix")
    if a.stride(0) == 1 and a.stride(1) >= max(rows, 1):
        return a, a.stride(1)
    t = a.t().contiguous()  # (cols, rows) row-major == column-major of a
    return t.t(), rows


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def as_numpy(t) -> np.ndarray:
    if isinstance(t, torch.Tensor):
        return t.detach().cpu().numpy()
    return np.asarray(t)
