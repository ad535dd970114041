"""The dense LU solve (reference linalg.py:75-99: scipy lu_factor + lu_solve with the
1e-14 ||A||_F pivot floor) on its two device paths: the persistent dataflow
kernel (every 16-column block column in one co-resident CTA; n <= ~1700) and the
blocked multi-launch LU above that.  Parity with the oracle (scipy getrf/getrs)
at 1e-10 relative on x, pivots identical to getrf's on well-separated inputs, the
finite-input check and the singular-pivot message."""

import os

import numpy as np
import pytest
import scipy.linalg
import torch

from oracle import strom_oracle as so
from paper_1910_01260_b200 import SingularMatrixError, _capi, linalg

from helpers import max_rel, npy

pytestmark = pytest.mark.gpu


def _system(n, seed, nrhs=None):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n)) + 0.5 * np.sqrt(n) * np.eye(n)
    b = rng.standard_normal(n) if nrhs is None else rng.standard_normal((n, nrhs))
    return a, b


@pytest.mark.parametrize("n", [1, 2, 15, 16, 17, 100, 999, 1000, 1200, 1700, 2100])
def test_solve_vs_oracle(cuda, n):
    a, b = _system(n, n)
    x = npy(linalg.solve_dense(a, b))
    ref = so.solve_dense(a, b)
    assert max_rel(x, ref) <= 1e-10
    assert np.linalg.norm(a @ x - b) <= 1e-12 * (np.linalg.norm(a) * np.linalg.norm(x) + np.linalg.norm(b))


@pytest.mark.parametrize("nrhs", [2, 16, 17, 40])
def test_multiple_rhs(cuda, nrhs):
    a, b = _system(300, 7, nrhs)
    x = npy(linalg.solve_dense(a, b))
    assert x.shape == (300, nrhs)
    assert max_rel(x, scipy.linalg.solve(a, b)) <= 1e-10


@pytest.mark.parametrize("n", [64, 700])
def test_factor_matches_getrf(cuda, n):
    """strom_dense_lu: the same pivots as LAPACK getrf and the same packed L\\U."""
    a, _ = _system(n, 3)
    lu_ref, piv_ref = scipy.linalg.lu_factor(a)
    lu = torch.as_tensor(a.T.copy(), device="cuda")  # column-major copy
    piv = torch.empty(n, dtype=torch.int32, device="cuda")
    _capi.call("strom_dense_lu", n, lu.data_ptr(), piv.data_ptr(), _capi.stream_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(npy(piv), piv_ref)
    assert max_rel(npy(lu).T, lu_ref) <= 1e-12


def test_pivot_ties_take_the_first_row(cuda):
    a = np.array([[1.0, 2.0, 0.0], [-1.0, 1.0, 3.0], [1.0, 0.0, 1.0]])
    lu_ref, piv_ref = scipy.linalg.lu_factor(a)
    lu = torch.as_tensor(a.T.copy(), device="cuda")
    piv = torch.empty(3, dtype=torch.int32, device="cuda")
    _capi.call("strom_dense_lu", 3, lu.data_ptr(), piv.data_ptr(), _capi.stream_ptr())
    assert np.array_equal(npy(piv), piv_ref)
    assert max_rel(npy(lu).T, lu_ref) <= 1e-15


@pytest.mark.parametrize("n", [2, 40, 1000])
def test_singular_pivot_message(cuda, n):
    a, b = _system(n, 5)
    a[:, n - 1] = a[:, 0]  # rank n - 1: the last pivot collapses
    with pytest.raises(SingularMatrixError, match="pivot"):
        linalg.solve_dense(a, b)
    with pytest.raises(SingularMatrixError, match="pivot 1"):
        linalg.solve_dense(np.array([[1.0, 2.0], [2.0, 4.0]]), np.ones(2))


@pytest.mark.parametrize("bad", [np.nan, np.inf])
def test_nonfinite_inputs_raise_like_scipy(cuda, bad):
    a, b = _system(50, 9)
    a2 = a.copy()
    a2[:, 3] = bad  # a whole NaN column too: the pivot search must not pick an invalid row
    with pytest.raises(ValueError, match="infs or NaNs"):
        linalg.solve_dense(a2, b)
    b2 = b.copy()
    b2[7] = bad
    with pytest.raises(ValueError, match="infs or NaNs"):
        linalg.solve_dense(a, b2)
    # the device is still healthy afterwards
    assert max_rel(npy(linalg.solve_dense(a, b)), so.solve_dense(a, b)) <= 1e-10


def test_persistent_and_blocked_paths_agree(cuda, monkeypatch):
    a, b = _system(500, 11)
    x1 = npy(linalg.solve_dense(a, b))
    monkeypatch.setenv("STROM_LU_LEGACY", "1")
    x2 = npy(linalg.solve_dense(a, b))
    assert max_rel(x1, x2) <= 1e-12
