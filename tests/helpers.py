"""Comparison helpers shared by the parity tests (test infrastructure)."""

from __future__ import annotations

import numpy as np

EPS = np.finfo(float).eps


def npy(t) -> np.ndarray:
    try:
        import torch

        if isinstance(t, torch.Tensor):
            return t.detach().cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(t)


def align_columns(a: np.ndarray, b: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Flip columns of a so that each has a non-negative inner product with b's; returns (a', signs)."""
    s = np.sign(np.sum(a * b, axis=0))
    s[s == 0] = 1.0
    return a * s, s


def max_rel(a, b) -> float:
    """max |a - b| / max(1e-300, max |b|) -- the 'relative max-abs' of SURVEY 8(c)."""
    a, b = npy(a), npy(b)
    scale = max(float(np.max(np.abs(b))) if b.size else 0.0, 1e-300)
    return float(np.max(np.abs(a - b))) / scale if b.size else 0.0


def sigma_rel(a, b) -> np.ndarray:
    a, b = npy(a), npy(b)
    return np.abs(a - b) / np.abs(b)


def principal_sine(a: np.ndarray, b: np.ndarray) -> float:
    """sin of the largest principal angle between span(a) and span(b)."""
    qa, _ = np.linalg.qr(a)
    qb, _ = np.linalg.qr(b)
    m = qb - qa @ (qa.T @ qb)
    return float(np.linalg.norm(m, 2))


def factor_state(phi: np.ndarray):
    """Orthonormal factor U and coefficients W with phi = U W (numpy QR), for lock-step loading."""
    if phi.shape[1] == 0:
        return phi, np.zeros((0, 0))
    q, r = np.linalg.qr(phi, mode="reduced")
    return q, r
