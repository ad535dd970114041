"""Spatial Galerkin reduced operators on the B200 (reference spatial.py:22-67).

``build_spatial_rom`` runs ONE fused kernel: the CSR product A Phi is formed
tile by tile in shared memory and immediately contracted with Phi on the fp64
tensor cores, together with the extra right-hand columns B, C, x0 - x_ref and
A x_ref, so A Phi never touches HBM.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
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


def spatial_reduce(dev: dict, phi: torch.Tensor, extra_cm: torch.Tensor | None, ne: int,
                   xref: torch.Tensor | None, stream=None) -> torch.Tensor:
    """Phi^T [A Phi | extra | A xref] as one (n_s x q) tensor (C ABI strom_spatial_reduce_csr).

    ``extra_cm`` holds the extra right-hand columns column-major, as the rows of a
    C-contiguous (>= ne, N) tensor; the first ``ne`` are used."""
    n, ns = phi.shape
    phi, rs, cs = _phi_strides(phi)
    ext_ptr, ext_ld = None, n
    if extra_cm is not None and ne > 0:
        assert extra_cm.is_contiguous() and extra_cm.shape[1] == n
        ext_ptr = extra_cm.data_ptr()
    else:
        ne = 0
    q = ns + ne + (1 if xref is not None else 0)
    out = torch.empty((ns, q), dtype=F64, device=phi.device)
    ell = dev.get("ell")
    if ell is not None and rs == 1 and ns <= 64 and q <= 64:
        # column-major Phi: warp-specialised gather from the tiled-ELL operator
        capi.call("strom_spatial_reduce_ell", n, ell["k"], ell["idx"].data_ptr(), ell["val"].data_ptr(),
                  ell["reach"], phi.data_ptr(), cs, ns, ext_ptr, ext_ld, ne,
                  None if xref is None else xref.data_ptr(), out.data_ptr(), capi.stream_ptr(stream))
        return out
    capi.call("strom_spatial_reduce_csr", n, dev["indptr"].data_ptr(), dev["indices"].data_ptr(),
              dev["data"].data_ptr(), dev["index_bits"], phi.data_ptr(), rs, cs, ns, ext_ptr, ext_ld, ne,
              None if xref is None else xref.data_ptr(), out.data_ptr(),
              capi.stream_ptr(stream))
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
    # extras: dev["bcx0"] is [B | C | x0] column-major.  With x_ref = x0 the
    # x0 - x_ref column is exactly zero (x0_hat = 0) and A x_ref is one more
    # gathered column; with x_ref = 0 the A x_ref column is exactly zero.
    if ref_mode == "initial_state":
        x_ref = dev["x0"]
        z = spatial_reduce(dev, phi, dev["bcx0"], m + p, x_ref)
        x0_hat = torch.zeros(ns, dtype=F64, device=phi.device)
        x_ref_hat = z[:, -1].contiguous()
    else:
        x_ref = torch.zeros(n, dtype=F64, device=phi.device)
        z = spatial_reduce(dev, phi, dev["bcx0"], m + p + 1, None)
        x0_hat = z[:, ns + m + p].contiguous()
        x_ref_hat = torch.zeros(ns, dtype=F64, device=phi.device)
    a_hat = z[:, :ns].contiguous()
    b_hat = z[:, ns:ns + m].contiguous()
    c_hat = z[:, ns + m:ns + m + p].contiguous()
    y_ref = dev["c"].T @ x_ref if ref_mode == "initial_state" else torch.zeros(p, dtype=F64, device=phi.device)
    return SpatialRom(a_hat=a_hat, b_hat=b_hat, c_hat=c_hat, x_ref=x_ref, x_ref_hat=x_ref_hat,
                      x0_hat=x0_hat, y_ref=y_ref, ref_mode=ref_mode)


def srom_march(rom: SpatialRom, grid, inputs) -> torch.Tensor:
    """March the reduced coordinates over the grid; column k-1 holds xhat_k (spatial.py:68-85).

    One device LU of I - dt A_hat per distinct dt (``strom_dense_lu``), two
    triangular solves per step (``strom_dense_lu_solve``), like the
    reference's ``lu_factor`` / ``lu_solve`` cache.
    """
    n_s, nt = rom.n_s, grid.n_steps
    dev = rom.a_hat.device
    traj = torch.empty((nt, n_s), dtype=F64, device=dev)
    eye = torch.eye(n_s, dtype=F64, device=dev)
    factors = {}
    x = rom.x0_hat
    if not bool(torch.isfinite(rom.a_hat).all()):  # scipy lu_factor(check_finite=True), spatial.py:80
        raise ValueError("array must not contain infs or NaNs")
    for k in range(nt):
        dt = float(grid.dt[k])
        fac = factors.get(dt)
        if fac is None:
            lu = (eye - dt * rom.a_hat).T.contiguous()  # column-major
            piv = torch.empty(n_s, dtype=torch.int32, device=dev)
            capi.call("strom_dense_lu", n_s, lu.data_ptr(), piv.data_ptr(), capi.stream_ptr())
            fac = factors[dt] = (lu, piv)
        f = torch.as_tensor(np.atleast_1d(np.asarray(inputs(k + 1), dtype=float)), dtype=F64, device=dev)
        xk = traj[k]
        torch.add(x + dt * rom.x_ref_hat, rom.b_hat @ f, alpha=dt, out=xk)
        capi.call("strom_dense_lu_solve", n_s, fac[0].data_ptr(), fac[1].data_ptr(), xk.data_ptr(), 1,
                  capi.stream_ptr())
        x = xk
    return traj.T


def srom_output(rom: SpatialRom, x_hat) -> torch.Tensor:
    """y = C_hat^T xhat + C^T x_ref, for a vector or a trajectory (spatial.py:88-92)."""
    x_hat = to_dev(x_hat)
    y = rom.c_hat.T @ x_hat
    return y + (rom.y_ref if x_hat.dim() == 1 else rom.y_ref[:, None])


def reconstruct_states(rom: SpatialRom, basis: BasisSet, x_hat) -> torch.Tensor:
    """Lift reduced coordinates: x_ref + Phi_s xhat (spatial.py:95-100; not the
    space-time ``reconstruct_states`` that the package exports)."""
    x_hat = to_dev(x_hat)
    lifted = basis.phi_s @ x_hat
    return lifted + (rom.x_ref if x_hat.dim() == 1 else rom.x_ref[:, None])
