"""reconstruct_states / reconstruct_step on the device (reference spacetime.py:165-186)
against the oracle: the DMMA tall GEMM Phi_s C with C[i, k] = sum_j Psi_i[k, j]
xhat[j n_s + i], at ragged sizes (N, N_t, n_s not multiples of the tiles) and at
BASELINE config 4's full size (N = 10^6, n_s = 50, n_t = 20, N_t = 500)."""

import numpy as np
import pytest
import torch

from oracle import strom_oracle as so
from paper_1910_01260_b200 import BasisSet, spacetime, workloads as wl

from helpers import max_rel, npy

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,ns,nt,nsteps", [(1, 1, 1, 1), (37, 3, 2, 5), (1000, 7, 3, 65), (4097, 13, 5, 129),
                                            (300, 50, 20, 500)])
def test_ragged_sizes(cuda, n, ns, nt, nsteps):
    rng = np.random.default_rng(n + ns)
    phi, temporal = wl.random_basis(rng, n, nsteps, ns, nt) if n >= ns and nsteps >= nt else (
        rng.standard_normal((n, ns)), tuple(rng.standard_normal((nsteps, nt)) for _ in range(ns)))
    xhat = rng.standard_normal(ns * nt)
    bs = BasisSet(phi, temporal, n_mu=1)
    got = spacetime.reconstruct_states(bs, xhat)
    ref = so.st_reconstruct(phi, temporal, xhat)
    assert got.shape == (n, nsteps) and got.is_contiguous()
    assert max_rel(got, ref) <= 1e-13
    for k in (0, nsteps - 1):
        assert max_rel(spacetime.reconstruct_step(bs, xhat, k), ref[:, k]) <= 1e-13


def test_rejects_wrong_solution_length(cuda):
    bs = BasisSet(np.eye(4)[:, :2], (np.eye(3)[:, :1], np.eye(3)[:, :1]), n_mu=1)
    with pytest.raises(ValueError, match="n_s\\*n_t"):
        spacetime.reconstruct_states(bs, np.ones(3))


def test_cfg4_full_size(cuda):
    d = wl.cfg4_inputs()
    xhat = np.random.default_rng(12).standard_normal(50 * 20)
    phi_cm = torch.as_tensor(np.asfortranarray(d.phi_s).T.copy(), device="cuda").T
    bs = BasisSet(phi_cm, torch.as_tensor(np.stack(d.temporal), device="cuda"), n_mu=20)
    got = spacetime.reconstruct_states(bs, xhat)
    ref = so.st_reconstruct(d.phi_s, d.temporal, xhat)
    assert max_rel(got, ref) <= 1e-12
