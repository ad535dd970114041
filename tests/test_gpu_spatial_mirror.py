"""The reference's spatial-ROM test cases (pkg/tests/test_spatial.py) against
the device path: build_spatial_rom, srom_march, srom_output and the spatial
reconstruct_states (spatial.py:45-100)."""

import numpy as np
import pytest
import scipy.sparse as sp
import torch

from paper_1910_01260_b200 import BasisSet, LinearDynamicalSystem, TimeGrid, basis, fom_march, spatial
from paper_1910_01260_b200 import workloads as wl
from paper_1910_01260_b200.spatial import SpatialRom

from helpers import npy

pytestmark = pytest.mark.gpu


def heat1d(nx, kappa):
    """The reference's heat1d generator (problems.py:86-112): kappa u_xx, Dirichlet,
    unit indicator source on the middle third, nodal-mean output."""
    h = 1.0 / (nx + 1)
    s = kappa / h**2
    a = sp.diags_array([np.full(nx - 1, s), np.full(nx, -2.0 * s), np.full(nx - 1, s)], offsets=(-1, 0, 1),
                       format="csr")
    x = (np.arange(nx) + 1) * h
    b = ((x >= 1.0 / 3.0) & (x <= 2.0 / 3.0)).astype(float)
    return LinearDynamicalSystem(a=a, b=sp.csr_array(b[:, None]), c=np.full((nx, 1), 1.0 / nx), x0=np.zeros(nx),
                                 input_signal=lambda k: np.array([1.0]), constant_input=True)


def full_basis(n, n_steps=1):
    return BasisSet(np.eye(n), tuple(np.ones((n_steps, 1)) for _ in range(n)), 1)


def trained_basis(sys_, grid, n_s):
    states = fom_march(sys_, grid).states
    st = basis.ingest_simulation(basis.isvd_init(states[:, 0], tol_svd=0.0), states[:, 1:])
    return basis.build_basis_set(st, n_s, 1, grid.n_steps, 1)


def _t(v):
    return torch.as_tensor(np.asarray(v, dtype=float), device="cuda")


def test_square_basis_is_similarity(cuda):
    rng = np.random.default_rng(1)
    d = wl.random_stable_system(rng, 6)
    sys_ = LinearDynamicalSystem(a=d["a"], b=d["b"], c=d["c"], x0=d["x0"], input_signal=d["inputs"])
    q = wl.haar(rng, 6, 6)
    rom = spatial.build_spatial_rom(sys_, BasisSet(q, tuple(np.ones((1, 1)) for _ in range(6)), 1), ref_mode="zero")
    np.testing.assert_allclose(npy(rom.a_hat), q.T @ d["a"].toarray() @ q, atol=1e-12)


def test_frozen_dynamics_and_scalar_recursion(cuda):
    rom = SpatialRom(a_hat=_t(np.zeros((2, 2))), b_hat=_t(np.zeros((2, 1))), c_hat=_t(np.zeros((2, 1))),
                     x_ref=_t(np.zeros(4)), x_ref_hat=_t(np.zeros(2)), x0_hat=_t([1.0, -1.0]), y_ref=_t(np.zeros(1)),
                     ref_mode="zero")
    traj = npy(spatial.srom_march(rom, TimeGrid.uniform(0.1, 5), lambda k: np.zeros(1)))
    np.testing.assert_allclose(traj, np.tile([[1.0], [-1.0]], (1, 5)))
    a, b, f, dt = -0.7, 0.4, 1.3, 0.2
    rom = SpatialRom(a_hat=_t([[a]]), b_hat=_t([[b]]), c_hat=_t(np.ones((1, 1))), x_ref=_t(np.zeros(1)),
                     x_ref_hat=_t(np.zeros(1)), x0_hat=_t([0.5]), y_ref=_t(np.zeros(1)), ref_mode="zero")
    traj = npy(spatial.srom_march(rom, TimeGrid.uniform(dt, 4), lambda k: np.array([f])))
    x = 0.5
    for k in range(4):
        x = (x + dt * b * f) / (1.0 - dt * a)
        assert traj[0, k] == pytest.approx(x, rel=1e-14)


def test_identity_basis_matches_fom_and_outputs(cuda):
    sys_ = heat1d(7, 1.0)
    grid = TimeGrid.uniform(0.02, 9)
    bs = full_basis(7, grid.n_steps)
    rom = spatial.build_spatial_rom(sys_, bs, ref_mode="zero")
    traj = spatial.srom_march(rom, grid, sys_.input_signal)
    fom = fom_march(sys_, grid)
    rec = spatial.reconstruct_states(rom, bs, traj)
    assert float((rec - fom.states).abs().max()) <= 1e-9 * max(1.0, float(fom.states.abs().max()))
    np.testing.assert_allclose(npy(spatial.srom_output(rom, traj)), npy(fom.outputs), atol=1e-9)


def test_output_zero_case_and_selector(cuda):
    rng = np.random.default_rng(5)
    d = wl.random_stable_system(rng, 6)
    phi, temporal = wl.random_basis(rng, 6, 4, 2, 1)
    sys_ = LinearDynamicalSystem(a=d["a"], b=d["b"], c=d["c"], x0=d["x0"], input_signal=d["inputs"])
    rom = spatial.build_spatial_rom(sys_, BasisSet(phi, temporal, 1), ref_mode="zero")
    assert np.array_equal(npy(spatial.srom_output(rom, np.zeros(2))), np.zeros(1))
    rng = np.random.default_rng(6)
    d = wl.random_stable_system(rng, 5)
    sel = np.zeros((5, 1))
    sel[3, 0] = 1.0
    sys_ = LinearDynamicalSystem(a=d["a"], b=d["b"], c=sel, x0=d["x0"], input_signal=d["inputs"])
    bs = full_basis(5)
    rom = spatial.build_spatial_rom(sys_, bs, ref_mode="zero")
    x_hat = rng.standard_normal(5)
    np.testing.assert_allclose(npy(spatial.srom_output(rom, x_hat)), [x_hat[3]], atol=1e-14)


def test_galerkin_residual_orthogonal_to_basis(cuda):
    sys_ = heat1d(10, 1.0)
    grid = TimeGrid.uniform(0.02, 10)
    bs = trained_basis(sys_, grid, 3)
    rom = spatial.build_spatial_rom(sys_, bs, ref_mode="zero")
    rec = npy(spatial.reconstruct_states(rom, bs, spatial.srom_march(rom, grid, sys_.input_signal)))
    a, b, phi = sys_.a.toarray(), sys_.b.toarray(), npy(bs.phi_s)
    x_prev = sys_.x0
    for k in range(grid.n_steps):
        dt = float(grid.dt[k])
        r = rec[:, k] - dt * (a @ rec[:, k]) - x_prev - dt * (b @ sys_.input_signal(k + 1))  # system.step_residual
        assert np.max(np.abs(phi.T @ r)) <= 1e-9
        x_prev = rec[:, k]


def test_exactness_when_span_contains_trajectory(cuda):
    sys_ = heat1d(9, 1.1)
    grid = TimeGrid.uniform(0.02, 14)
    fom = fom_march(sys_, grid).states
    bs = trained_basis(sys_, grid, min(9, int(np.linalg.matrix_rank(npy(fom)))))
    rom = spatial.build_spatial_rom(sys_, bs, ref_mode="initial_state")
    rec = spatial.reconstruct_states(rom, bs, spatial.srom_march(rom, grid, sys_.input_signal))
    rel = torch.linalg.norm(rec - fom, dim=0) / torch.linalg.norm(fom, dim=0)
    assert float(rel.max()) <= 1e-9
