"""A-posteriori bounds (reference bounds.py) and the matrix-free space-time
inverse (system.py:195-275) on the device, against the reference's own outputs
(tests/golden/golden_bounds.npz, make_golden.gen_bounds).  Stage-isolated: the
approximate trajectories are the reference's.  Dense norms (n <= 256) to
1e-10; power-iteration constants (n = 300, tol 1e-8, same seeded start
vectors) to 1e-7."""

import numpy as np
import pytest
import scipy.sparse as sp
import torch

from paper_1910_01260_b200 import LinearDynamicalSystem, TimeGrid, bounds, linalg, system

from conftest import load_golden
from helpers import npy

pytestmark = pytest.mark.gpu


def heat1d(nx, kappa=1.0):
    h = 1.0 / (nx + 1)
    s = kappa / h**2
    a = sp.diags_array([np.full(nx - 1, s), np.full(nx, -2.0 * s), np.full(nx - 1, s)], offsets=(-1, 0, 1),
                       format="csr")
    x = (np.arange(nx) + 1) * h
    b = ((x >= 1.0 / 3.0) & (x <= 2.0 / 3.0)).astype(float)
    return LinearDynamicalSystem(a=a, b=sp.csr_array(b[:, None]), c=np.full((nx, 1), 1.0 / nx), x0=np.zeros(nx),
                                 input_signal=lambda k: np.array([1.0]), constant_input=True)


def _rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - b)) / max(np.max(np.abs(b)), 1e-300))


def test_st_inverse_applies_match_reference(cuda):
    g = load_golden("golden_bounds.npz")
    sys_ = LinearDynamicalSystem(a=sp.csr_array(g["inv_a"]), b=sp.csr_array(g["inv_b"]), c=np.zeros((10, 1)),
                                 x0=np.zeros(10), input_signal=lambda k: np.zeros(1))
    grid = TimeGrid(g["inv_dt"])
    assert _rel(npy(system.st_apply_inverse(sys_, grid, g["inv_v"])), g["inv_fwd"]) <= 1e-12
    assert _rel(npy(system.st_apply_inverse_adjoint(sys_, grid, g["inv_v"])), g["inv_adj"]) <= 1e-12
    with pytest.raises(ValueError):
        system.st_apply_inverse(sys_, grid, np.zeros(59))


@pytest.mark.parametrize("direct", [True, False])
def test_krylov_and_direct_inverse_agree(cuda, direct):
    """Sparse operator: the Krylov march over the ELL forms of A and A^T and the
    dense StepSolver path give the same applies; adjoint consistency holds."""
    sys_ = heat1d(40)
    grid = TimeGrid(np.full(5, 2e-4))
    apply, apply_adj = system.st_inverse_operator(sys_, grid, direct=direct)
    rng = np.random.default_rng(3)
    v = torch.as_tensor(rng.standard_normal(200), device="cuda")
    w = torch.as_tensor(rng.standard_normal(200), device="cuda")
    lhs, rhs = float(torch.dot(apply(v), w)), float(torch.dot(v, apply_adj(w)))
    assert abs(lhs - rhs) <= 1e-11 * max(1.0, abs(lhs))
    ref_apply, _ = system.st_inverse_operator(sys_, grid, direct=True)
    assert _rel(npy(apply(v)), npy(ref_apply(v))) <= 1e-11


@pytest.mark.parametrize("tag,nx,dt,nt", [("small", 12, 1e-3, 10), ("large", 300, 2e-6, 6)])
def test_bounds_match_reference(cuda, tag, nx, dt, nt):
    g = load_golden("golden_bounds.npz")
    heat = heat1d(nx)
    grid = TimeGrid.uniform(dt, nt)
    assert _rel(npy(system.st_residual(heat, grid, g[f"{tag}_approx_st"])), g[f"{tag}_st_res"]) <= 1e-9
    ctol = 1e-10 if nx <= bounds.DENSE_NORM_CUTOFF else 1e-7
    for name, fn, arg in (("residual", bounds.residual_error_bound, g[f"{tag}_approx"]),
                          ("rom", bounds.rom_error_bound, g[f"{tag}_approx"]),
                          ("st", bounds.space_time_error_bound, g[f"{tag}_approx_st"])):
        rep = fn(heat, grid, arg)
        assert _rel(rep.step_errors, g[f"{tag}_{name}_errors"]) <= 1e-8, name
        assert _rel(rep.constants, g[f"{tag}_{name}_constants"]) <= ctol, name
        assert _rel(rep.step_bounds, g[f"{tag}_{name}_bounds"]) <= max(ctol, 1e-9) * 10, name
        assert rep.valid == bool(g[f"{tag}_{name}_valid"][0])


def test_preconditions_and_power_iteration_guards(cuda):
    heat = heat1d(12)
    grid = TimeGrid.uniform(0.02, 3)  # dt above 1/||A||_2
    with pytest.raises(bounds.PreconditionError):
        bounds.rom_error_bound(heat, grid, np.zeros((12, 3)))
    a = torch.eye(4, dtype=torch.float64, device="cuda")
    with pytest.raises(linalg.AdjointConsistencyError):
        linalg.largest_singular_value(lambda v: a @ v, lambda v: 2.0 * (a @ v), 4, 4)
    assert linalg.largest_singular_value(lambda v: 0.0 * v, lambda v: 0.0 * v, 4, 4) == 0.0
    assert abs(linalg.largest_singular_value(lambda v: 3.0 * v, lambda v: 3.0 * v, 5, 5) - 3.0) <= 1e-12


def test_csr_apply_matches_scipy(cuda):
    """The library SpMM (C ABI strom_csr_spmm) behind the residual evaluations and
    operator_norm's sparse applies (reference system.py:249-275, bounds.py:60-70):
    vector and multi-column right-hand sides, a rectangular operator, empty rows."""
    import scipy.sparse as sp

    from paper_1910_01260_b200.system import csr_apply

    rng = np.random.default_rng(4)
    for (n, ncol, m) in ((1, 1, 1), (300, 300, 1), (257, 190, 7), (1000, 1000, 33)):
        a = sp.random(n, ncol, density=0.05, random_state=int(rng.integers(1 << 30)), format="csr")
        a.sort_indices()
        csr = dict(indptr=torch.as_tensor(a.indptr.astype(np.int32), device="cuda"),
                   indices=torch.as_tensor(a.indices.astype(np.int32), device="cuda"),
                   data=torch.as_tensor(a.data, device="cuda"), index_bits=32, shape=a.shape)
        x = rng.standard_normal((ncol, m))
        ref = a @ x
        got = csr_apply(csr, torch.as_tensor(x, device="cuda")).cpu().numpy()
        scale = max(1.0, np.max(np.abs(ref)))
        assert np.max(np.abs(got - ref)) <= 1e-13 * scale
        v = csr_apply(csr, torch.as_tensor(x[:, 0].copy(), device="cuda")).cpu().numpy()
        assert v.shape == (n,) and np.max(np.abs(v - ref[:, 0])) <= 1e-13 * scale
        csr64 = dict(csr, indptr=csr["indptr"].to(torch.int64), indices=csr["indices"].to(torch.int64), index_bits=64)
        got64 = csr_apply(csr64, torch.as_tensor(x, device="cuda")).cpu().numpy()
        np.testing.assert_array_equal(got64, got)
    with pytest.raises(ValueError):
        csr_apply(csr, torch.zeros(3, dtype=torch.float64, device="cuda"))
