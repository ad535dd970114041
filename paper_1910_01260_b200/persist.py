"""STROMMAT matrix files for device bases (reference persist.py:1-73,
pipeline.py:127-176 save_bases / load_basis).

The on-disk layout is the reference's, byte for byte: an 8-byte magic
``STROMMAT``, a little-endian u32 version (1), u64 rows, u64 cols, then
rows*cols little-endian binary64 values in column-major order.  Files written
here are read by the reference and vice versa.

Device tensors are written without a transposition: the bases live column-major
in HBM (``BasisSet.phi_s``; temporal blocks are transposed views when needed),
so the payload is one device-to-host copy into a pinned buffer, validated for
finiteness on the device first.  ``read_matrix`` keeps the reference's return
type (a C-contiguous NumPy array); ``read_matrix_device`` returns a
column-major CUDA tensor straight from the payload.
"""

from __future__ import annotations

import os
import struct
from pathlib import Path

import numpy as np
import torch

from ._tensors import F64, device

MAGIC = b"STROMMAT"
VERSION = 1
HEADER_SIZE = 28
_HEADER = struct.Struct("<8sIQQ")


class MatrixFileError(Exception):
    """Raised for malformed, truncated, or non-finite matrix files (persist.py:31-32)."""


def _payload_f(m) -> tuple[int, int, np.ndarray | torch.Tensor]:
    """(rows, cols, column-major payload) of a 1-D/2-D array or tensor."""
    if isinstance(m, torch.Tensor):
        t = m.detach()
        if t.dim() == 1:
            t = t[:, None]
        if t.dim() != 2 or t.numel() == 0:
            raise MatrixFileError(f"refusing to write empty or non-2-D matrix of shape {tuple(t.shape)}")
        t = t.to(F64)
        if not bool(torch.isfinite(t).all()):
            raise MatrixFileError("refusing to write non-finite entries")
        rows, cols = t.shape
        colmajor = t.T.contiguous() if not (t.stride(0) == 1 and t.stride(1) == rows) else t.T
        if colmajor.is_cuda:
            host = torch.empty(colmajor.shape, dtype=F64, pin_memory=True)
            host.copy_(colmajor)
            return rows, cols, host.numpy()
        return rows, cols, colmajor.numpy()
    a = np.asarray(m, dtype="<f8")
    if a.ndim == 1:
        a = a[:, None]
    if a.ndim != 2 or a.size == 0:
        raise MatrixFileError(f"refusing to write empty or non-2-D matrix of shape {a.shape}")
    if not np.all(np.isfinite(a)):
        raise MatrixFileError("refusing to write non-finite entries")
    return a.shape[0], a.shape[1], np.asfortranarray(a).T


def write_matrix(path, m) -> None:
    """Write a 2-D float64 matrix (NumPy array or torch tensor, host or device)."""
    rows, cols, payload = _payload_f(m)
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(MAGIC, VERSION, rows, cols))
        fh.write(np.ascontiguousarray(payload, dtype="<f8").tobytes(order="C"))


def _read_checked(path) -> tuple[int, int, np.ndarray]:
    size = os.stat(path).st_size
    if size < HEADER_SIZE:
        raise MatrixFileError(f"{path}: file too short for a header ({size} bytes)")
    with open(path, "rb") as fh:
        magic, version, rows, cols = _HEADER.unpack(fh.read(HEADER_SIZE))
        if magic != MAGIC:
            raise MatrixFileError(f"{path}: bad magic {magic!r}")
        if version != VERSION:
            raise MatrixFileError(f"{path}: unsupported version {version}")
        if rows == 0 or cols == 0:
            raise MatrixFileError(f"{path}: degenerate shape {rows}x{cols}")
        expected = HEADER_SIZE + 8 * rows * cols
        if size != expected:
            raise MatrixFileError(f"{path}: payload truncated or padded ({size} bytes, expected {expected})")
        data = np.fromfile(fh, dtype="<f8", count=rows * cols)
    if data.size != rows * cols:
        raise MatrixFileError(f"{path}: short read of payload")
    return rows, cols, data


def read_matrix(path) -> np.ndarray:
    """Read a matrix (persist.py:54-73): validated header, C-contiguous NumPy result."""
    rows, cols, data = _read_checked(path)
    m = data.reshape((rows, cols), order="F")
    if not np.all(np.isfinite(m)):
        raise MatrixFileError(f"{path}: non-finite values in payload")
    return np.ascontiguousarray(m)


def read_matrix_device(path) -> torch.Tensor:
    """Read a matrix straight into HBM as a column-major (rows, cols) CUDA tensor."""
    rows, cols, data = _read_checked(path)
    host = torch.from_numpy(data).pin_memory()
    t = host.to(device(), non_blocking=True).reshape(cols, rows).T
    if not bool(torch.isfinite(t).all()):
        raise MatrixFileError(f"{path}: non-finite values in payload")
    return t


def save_bases(state, basis, bases_dir) -> list[str]:
    """Persist the basis set and the SVD state's sigma and V (pipeline.py:127-142)."""
    bases_dir = Path(bases_dir)
    bases_dir.mkdir(parents=True, exist_ok=True)
    written = []

    def put(name, matrix):
        write_matrix(bases_dir / name, matrix)
        written.append(name)

    put("phi_s.strommat", basis.phi_s)
    for i, psi in enumerate(basis.temporal):
        put(f"psi_{i:04d}.strommat", psi)
    put("sigma.strommat", state.sigma[:, None])
    put("v.strommat", state.v)
    return written


def load_basis(bases_dir, n_s: int | None = None, n_t: int | None = None):
    """Load a stored basis into HBM, optionally sliced (pipeline.py:145-176)."""
    from .basis import BasisSet

    bases_dir = Path(bases_dir)
    phi_path = bases_dir / "phi_s.strommat"
    if not phi_path.exists():
        raise FileNotFoundError(f"no trained basis at {bases_dir} (run `strom train` first)")
    phi_s = read_matrix_device(phi_path)
    psi_paths = sorted(bases_dir.glob("psi_*.strommat"))
    temporal = [read_matrix_device(p) for p in psi_paths]
    if len(temporal) != phi_s.shape[1]:
        raise ValueError(f"{bases_dir}: found {len(temporal)} temporal bases for {phi_s.shape[1]} spatial modes")
    stored_nt = temporal[0].shape[1]
    n_s = phi_s.shape[1] if n_s is None else n_s
    n_t = stored_nt if n_t is None else n_t
    if n_s > phi_s.shape[1] or n_t > stored_nt:
        raise ValueError(f"requested n_s={n_s}, n_t={n_t} but stored basis has n_s={phi_s.shape[1]}, "
                         f"n_t={stored_nt}")
    n_steps = temporal[0].shape[0]
    v_path = bases_dir / "v.strommat"
    # read_matrix, as the reference does (pipeline.py:171): it validates the payload too
    n_mu = read_matrix(v_path).shape[0] // n_steps if v_path.exists() else n_t
    return BasisSet(phi_s=phi_s[:, :n_s], temporal=tuple(t[:, :n_t] for t in temporal[:n_s]), n_mu=n_mu)
