"""Spatial Galerkin reduced operators on the B200 (reference spatial.py:22-67).

``build_spatial_rom`` runs ONE fused kernel: the CSR product A Phi is formed
tile by tile in shared memory and immediately contracted with Phi on the fp64
tensor cores, together with the extra right-hand columns B, C, x0 - x_ref and
A x_ref, so A Phi never touches HBM.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _capi as capi
from ._tensors import F64, device, to_dev
from .basis import BasisSet
from .system import LinearDynamicalSystem

REF_MODES = ("zero", "initial_state")


@dataclass(frozen=True)
class SpatialRom:
    """Reduced operators of one parameter instance (spatial.py:22-42)."""

    a_hat: torch.Tensor
    b_hat: torch.Tensor
    c_hat: torch.Tensor
    x_ref: torch.Tensor
    x_ref_hat: torch.Tensor
    x0_hat: torch.Tensor
    y_ref: torch.Tensor
    ref_mode: str

    @property
    def n_s(self) -> int:
        return self.a_hat.shape[0]


def _phi_strides(phi: torch.Tensor) -> tuple[torch.Tensor, int, int]:
    if phi.stride(1) == 1 or phi.stride(0) == 1:
        return phi, phi.stride(0), phi.stride(1)
    phi = phi.contiguous()
    return phi, phi.stride(0), phi.stride(1)


def spatial_reduce(dev: dict, phi: torch.Tensor, extra: torch.Tensor | None, xref: torch.Tensor | None,
                   stream=None) -> torch.Tensor:
    """Phi^T [A Phi | extra | A xref] as one (n_s x q) tensor (C ABI strom_spatial_reduce_csr)."""
    n, ns = phi.shape
    phi, rs, cs = _phi_strides(phi)
    ne = 0 if extra is None else extra.shape[1]
    ext_ptr, ext_ld = None, n
    if extra is not None:
        ecm = extra.t().contiguous()  # column-major N x ne
        ext_ptr = ecm.data_ptr()
    q = ns + ne + (1 if xref is not None else 0)
    out = torch.empty((ns, q), dtype=F64, device=phi.device)
    capi.call("strom_spatial_reduce_csr", n, dev["indptr"].data_ptr(), dev["indices"].data_ptr(),
              dev["data"].data_ptr(), dev["index_bits"], phi.data_ptr(), rs, cs, ns, ext_ptr, ext_ld, ne,
              None if xref is None else xref.data_ptr(), out.data_ptr(),
              capi.stream_ptr(stream))
    if extra is not None:
        del ecm
    return out


def build_spatial_rom(sys: LinearDynamicalSystem, basis: BasisSet,
                      ref_mode: str = "initial_state") -> SpatialRom:
    """Project the system operators onto the spatial basis (spatial.py:45-67)."""
    if ref_mode not in REF_MODES:
        raise ValueError(f"ref_mode must be one of {REF_MODES}, got {ref_mode!r}")
    phi = basis.phi_s
    if phi.shape[0] != sys.n_states:
        raise ValueError(f"basis has {phi.shape[0]} rows but the system has {sys.n_states} states")
    dev = sys.device_arrays()
    n, ns = phi.shape
    m, p = dev["b"].shape[1], dev["c"].shape[1]
    if ref_mode == "initial_state":
        x_ref = dev["x0"]
        x0_minus = torch.zeros_like(x_ref)
        xref_col = x_ref
    else:
        x_ref = torch.zeros(n, dtype=F64, device=phi.device)
        x0_minus = dev["x0"]
        xref_col = None  # A 0 = 0 exactly: no column
    extra = torch.cat([dev["b"], dev["c"], x0_minus[:, None]], dim=1)
    z = spatial_reduce(dev, phi, extra, xref_col)
    a_hat = z[:, :ns].contiguous()
    b_hat = z[:, ns:ns + m].contiguous()
    c_hat = z[:, ns + m:ns + m + p].contiguous()
    x0_hat = z[:, ns + m + p].contiguous()
    x_ref_hat = z[:, -1].contiguous() if xref_col is not None else torch.zeros(ns, dtype=F64, device=phi.device)
    y_ref = dev["c"].T @ x_ref
    return SpatialRom(a_hat=a_hat, b_hat=b_hat, c_hat=c_hat, x_ref=x_ref, x_ref_hat=x_ref_hat,
                      x0_hat=x0_hat, y_ref=y_ref, ref_mode=ref_mode)
