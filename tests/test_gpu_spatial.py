"""Spatial reduction paths (spatial.py:57-64): the tiled-ELL fast path and the
CSR paths against the CPU oracle's Phi^T [A Phi | B | C | x0 | A x_ref].

Bar: reduced operators <= 1e-12 relative max-abs.  Edge
cases: empty rows, rows at every length up to the ELL width (4, 8, 16),
rows too long for ELL (CSR fallback), a ragged last 64-row tile, n < 64,
n_s not a multiple of 8, q = 64 exactly, negative and forward reach.
"""

import numpy as np
import pytest
import scipy.sparse as sp
import torch

from oracle import strom_oracle as so
from paper_1910_01260_b200 import BasisSet, LinearDynamicalSystem, spatial, workloads as wl

from helpers import max_rel, npy

pytestmark = pytest.mark.gpu


def _random_csr(rng, n, max_row, empty_frac=0.1, band=None):
    rows, cols, vals = [], [], []
    for r in range(n):
        if rng.random() < empty_frac:
            continue
        k = int(rng.integers(1, max_row + 1))
        if band is None:
            c = rng.choice(n, size=min(k, n), replace=False)
        else:
            c = np.unique(np.clip(r + rng.integers(-band, band + 1, size=k), 0, n - 1))
        rows += [r] * len(c)
        cols += list(c)
        vals += list(rng.standard_normal(len(c)))
    return sp.csr_array((vals, (rows, cols)), shape=(n, n))


def _system(rng, a, m=1, p=1):
    n = a.shape[0]
    return LinearDynamicalSystem(a=a, b=sp.csr_array(rng.standard_normal((n, m))), c=rng.standard_normal((n, p)),
                                 x0=rng.standard_normal(n), input_signal=lambda k: np.ones(m))


def _check(sys_, phi, ref_mode, expect_ell):
    dev = sys_.device_arrays()
    assert ("ell" in dev) == expect_ell
    bs = BasisSet(phi, tuple(np.eye(2) for _ in range(phi.shape[1])), 1)
    rom = spatial.build_spatial_rom(sys_, bs, ref_mode=ref_mode)
    ref = so.spatial_rom(sys_.a, sys_.b, sys_.c, sys_.x0, phi, ref_mode)
    for name in ("a_hat", "b_hat", "c_hat", "x0_hat", "x_ref_hat"):
        got, want = npy(getattr(rom, name)), getattr(ref, name)
        scale = max(np.max(np.abs(want)), 1e-300)
        assert np.max(np.abs(got - want)) <= 1e-12 * scale, name


@pytest.mark.parametrize("n,max_row,ns,band", [
    (1000, 4, 10, 3), (4099, 8, 50, 40), (777, 16, 13, 100), (63, 8, 7, None), (5000, 7, 60, None),
])
@pytest.mark.parametrize("ref_mode", ["zero", "initial_state"])
def test_ell_path_matches_oracle(cuda, n, max_row, ns, band, ref_mode):
    rng = np.random.default_rng(n + max_row)
    a = _random_csr(rng, n, max_row, band=band)
    phi = wl.haar(rng, n, ns)  # q = ns + 3 extra columns (+1 A x_ref) <= 64: the ELL path
    _check(_system(rng, a), phi, ref_mode, expect_ell=True)


def test_long_rows_fall_back_to_csr(cuda):
    rng = np.random.default_rng(3)
    a = _random_csr(rng, 600, 40, empty_frac=0.0)
    assert np.diff(a.indptr).max() > 16
    _check(_system(rng, a), wl.haar(rng, 600, 20), "zero", expect_ell=False)


def test_ell_equals_csr_bitwise_structure(cuda):
    """The ELL path and the CSR path agree to rounding on a cfg4-like stencil (10^3)."""
    a = wl.cfg4_operator(10, seed=1)
    rng = np.random.default_rng(5)
    sys_ = _system(rng, a)
    dev = sys_.device_arrays()
    assert dev["ell"]["k"] == 6 and dev["ell"]["reach"] == 100
    phi = torch.as_tensor(np.asfortranarray(wl.haar(rng, 1000, 50)).T.copy(), device="cuda").T
    ext = dev["bcx0"]
    z_ell = spatial.spatial_reduce(dev, phi, ext, 3, None)
    saved = dev.pop("ell")
    try:
        z_csr = spatial.spatial_reduce(dev, phi, ext, 3, None)
    finally:
        dev["ell"] = saved
    assert max_rel(npy(z_ell), npy(z_csr)) <= 1e-13
