"""Space-time reduced operators from the block structure, on the B200.

Mirror of the reference ``strom.spacetime`` (pkg/src/strom/spacetime.py).  The
space-time basis column (spatial mode i, temporal mode j) is psi_i^j (x) phi_i;
every reduced space-time operator collapses onto the spatial operators through
the diagonals E_k^(j), so the full-size basis never exists.  The whole
assembly (A_st, f_st, x0_st) is one C-ABI call: a DMMA temporal Gram with the
Hadamard-with-A_hat and diagonal terms fused into its epilogue, plus one small
kernel for the vectors.  The solve is the device LU of ``linalg.solve_dense``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _capi as capi
from . import linalg
from ._tensors import F64, colmajor, device, to_dev
from .basis import BasisSet
from .errors import SingularMatrixError
from .spatial import SpatialRom
from .system import InputSignal, TimeGrid


def temporal_diag(basis: BasisSet, k: int, j: int) -> torch.Tensor:
    """Diagonal of E_k^(j): entry i is mode i's j-th temporal vector at step k (spacetime.py:25-34)."""
    if not 0 <= k < basis.n_steps:
        raise IndexError(f"time step {k} out of range [0, {basis.n_steps})")
    if not 0 <= j < basis.n_t:
        raise IndexError(f"temporal mode {j} out of range [0, {basis.n_t})")
    return basis.temporal_stack()[:, k, j]


def _inputs_matrix(srom: SpatialRom, grid: TimeGrid, inputs: InputSignal, constant_input: bool):
    m = srom.b_hat.shape[1]
    if constant_input:
        f = np.atleast_1d(np.asarray(inputs(1), dtype=float)).reshape(m)
    else:
        f = np.stack([np.atleast_1d(np.asarray(inputs(k + 1), dtype=float)).reshape(m)
                      for k in range(grid.n_steps)])
    return torch.as_tensor(f, dtype=F64, device=device()).contiguous()


def _assemble(srom: SpatialRom, basis: BasisSet, grid: TimeGrid, inputs, constant_input: bool,
              want_matrix: bool, want_vectors: bool):
    if basis.n_steps != grid.n_steps:
        raise ValueError(f"basis covers {basis.n_steps} steps but the grid has {grid.n_steps}")
    n_s, n_t, nsteps = basis.n_s, basis.n_t, basis.n_steps
    nt_total = n_s * n_t
    dev = device()
    psi = basis.temporal_stack().contiguous()
    dt = grid.dt_device()
    a_hat = srom.a_hat.contiguous()
    a_st = torch.empty((nt_total, nt_total), dtype=F64, device=dev) if want_matrix else None
    f_st = x0_st = f = b_hat = x0_hat = None
    m = srom.b_hat.shape[1]
    if want_vectors:
        f_st = torch.empty(nt_total, dtype=F64, device=dev)
        x0_st = torch.empty(nt_total, dtype=F64, device=dev)
        b_hat = srom.b_hat.contiguous()
        x0_hat = srom.x0_hat.contiguous()
        f = (_inputs_matrix(srom, grid, inputs, constant_input) if inputs is not None
             else torch.zeros(max(m, 1), dtype=F64, device=dev))
    capi.call("strom_st_assemble", a_hat.data_ptr(), psi.data_ptr(), dt.data_ptr(), nsteps, n_s, n_t,
              None if b_hat is None else b_hat.data_ptr(), m, None if f is None else f.data_ptr(),
              1 if (constant_input or inputs is None) else 0,
              None if x0_hat is None else x0_hat.data_ptr(),
              None if a_st is None else a_st.data_ptr(), None if f_st is None else f_st.data_ptr(),
              None if x0_st is None else x0_st.data_ptr(), capi.stream_ptr())
    return a_st, f_st, x0_st


def build_st_matrix(srom: SpatialRom, basis: BasisSet, grid: TimeGrid) -> torch.Tensor:
    """Reduced space-time system matrix from its (j', j) blocks (spacetime.py:43-69)."""
    a_st, _, _ = _assemble(srom, basis, grid, None, True, True, False)
    return a_st


def build_st_input(srom: SpatialRom, basis: BasisSet, grid: TimeGrid, inputs: InputSignal,
                   constant_input: bool = False) -> torch.Tensor:
    """Block j = sum_k dt_k E_k^(j) (B_hat f_k) (spacetime.py:72-99)."""
    if basis.n_steps != grid.n_steps:
        raise ValueError(f"basis covers {basis.n_steps} steps but the grid has {grid.n_steps}")
    _, f_st, _ = _assemble(srom, basis, grid, inputs, constant_input, False, True)
    return f_st


def build_st_init(srom: SpatialRom, basis: BasisSet) -> torch.Tensor:
    """Every block j = E_1^(j) x0_hat -- the reference code's choice (spacetime.py:102-115)."""
    grid = TimeGrid(np.ones(basis.n_steps))
    _, _, x0_st = _assemble(srom, basis, grid, None, True, False, True)
    return x0_st


@dataclass(frozen=True)
class SpaceTimeRom:
    """Assembled reduced space-time system plus the basis to lift solutions (spacetime.py:118-125)."""

    a_st_hat: torch.Tensor
    f_st_hat: torch.Tensor
    x0_st_hat: torch.Tensor
    basis: BasisSet


def build_st_rom(srom: SpatialRom, basis: BasisSet, grid: TimeGrid, inputs: InputSignal,
                 constant_input: bool = False) -> SpaceTimeRom:
    """Matrix, input and initial vector in one device call (spacetime.py:128-151)."""
    if srom.ref_mode != "zero" and bool((srom.x_ref != 0.0).any()):
        raise ValueError("space-time assembly needs a zero-reference spatial ROM; "
                         "rebuild it with ref_mode='zero'")
    a_st, f_st, x0_st = _assemble(srom, basis, grid, inputs, constant_input, True, True)
    return SpaceTimeRom(a_st_hat=a_st, f_st_hat=f_st, x0_st_hat=x0_st, basis=basis)


def solve_st_rom(rom: SpaceTimeRom) -> torch.Tensor:
    """Solve the dense reduced space-time system (spacetime.py:154-162) with the device LU."""
    try:
        return linalg.solve_dense(rom.a_st_hat, rom.f_st_hat + rom.x0_st_hat)
    except SingularMatrixError as exc:
        raise SingularMatrixError(
            f"reduced space-time matrix is singular ({exc}); "
            "try smaller n_s or n_t, or better-conditioned bases") from exc


def reconstruct_step(basis: BasisSet, x_hat_st, k: int) -> torch.Tensor:
    """x_k = Phi_s sum_j E_k^(j) xhat^(j) (spacetime.py:165-177)."""
    if not 0 <= k < basis.n_steps:
        raise IndexError(f"time step {k} out of range [0, {basis.n_steps})")
    x_hat_st = to_dev(x_hat_st)
    blocks = x_hat_st.reshape(basis.n_t, basis.n_s)
    coeffs = (basis.temporal_stack()[:, k, :] * blocks.T).sum(dim=1)
    return basis.phi_s @ coeffs


def reconstruct_states(basis: BasisSet, x_hat_st) -> torch.Tensor:
    """Lift the reduced space-time solution at every step: N_s x N_t (spacetime.py:180-186).

    One coefficient kernel (C = sum_j E^(j) xhat^(j), n_s x N_t) and one DMMA
    tall GEMM Phi_s C (``strom_st_reconstruct``); the result is row-major like
    the reference's array.
    """
    x_hat_st = to_dev(x_hat_st).contiguous()
    ns, nt, nsteps = basis.n_s, basis.n_t, basis.n_steps
    if x_hat_st.numel() != ns * nt:
        raise ValueError(f"space-time solution has {x_hat_st.numel()} entries, expected n_s*n_t = {ns * nt}")
    phi, ldphi = colmajor(basis.phi_s)
    psi = basis.temporal_stack().contiguous()
    n = phi.shape[0]
    out = torch.empty((n, nsteps), dtype=F64, device=phi.device)
    capi.call("strom_st_reconstruct", n, ns, nt, nsteps, phi.data_ptr(), ldphi, psi.data_ptr(),
              x_hat_st.data_ptr(), out.data_ptr(), nsteps, capi.stream_ptr())
    return out


ST_VERIFICATION_CAP = 20_000  # system.py:23


def explicit_st_basis(basis: BasisSet, cap: int = ST_VERIFICATION_CAP) -> torch.Tensor:
    """The space-time basis, column i + n_s j = psi_i^j (x) phi_i (spacetime.py:189-210).

    A verification oracle only, refused above ``cap`` rows like the
    reference's: at production size it is exactly what the block-structured
    assembly avoids.  Built on the device as one broadcast product.
    """
    from .errors import CapExceededError

    n_rows = basis.phi_s.shape[0] * basis.n_steps
    if n_rows > cap:
        raise CapExceededError(f"explicit space-time basis would have {n_rows} rows, above the "
                               f"verification cap {cap}; it exists only as a testing oracle")
    psi = basis.temporal_stack()                          # (n_s, N_t, n_t)
    phi = basis.phi_s                                     # (N, n_s)
    # [k, r, j, i] = psi[i, k, j] * phi[r, i]  ->  rows k N + r, columns j n_s + i
    out = psi.permute(1, 2, 0)[:, None, :, :] * phi[None, :, None, :]
    return out.reshape(basis.n_steps * phi.shape[0], basis.n_t * basis.n_s)
