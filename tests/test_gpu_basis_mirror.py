"""The reference's basis test cases (pkg/tests/test_basis.py) not already in
test_gpu_isvd.py, against the device path: ingest edge cases, batch POD, the
temporal-snapshot layout, and build_basis_set against the batch pipeline."""

import numpy as np
import pytest
import scipy.sparse as sp
import torch

from paper_1910_01260_b200 import BasisError, LinearDynamicalSystem, TimeGrid, basis, fom_march, linalg

from helpers import npy

pytestmark = pytest.mark.gpu


def heat1d(nx, kappa):
    h = 1.0 / (nx + 1)
    s = kappa / h**2
    a = sp.diags_array([np.full(nx - 1, s), np.full(nx, -2.0 * s), np.full(nx - 1, s)], offsets=(-1, 0, 1),
                       format="csr")
    x = (np.arange(nx) + 1) * h
    b = ((x >= 1.0 / 3.0) & (x <= 2.0 / 3.0)).astype(float)
    return LinearDynamicalSystem(a=a, b=sp.csr_array(b[:, None]), c=np.full((nx, 1), 1.0 / nx), x0=np.zeros(nx),
                                 input_signal=lambda k: np.array([1.0]), constant_input=True)


def trained(kappas, nx=10, nt=15):
    grid = TimeGrid.uniform(0.02, nt)
    mats = [fom_march(heat1d(nx, k), grid).states for k in kappas]
    st = basis.ingest_simulation(basis.isvd_init(mats[0][:, 0], tol_svd=0.0), mats[0][:, 1:])
    for m in mats[1:]:
        st = basis.ingest_simulation(st, m)
    return st, torch.cat(mats, dim=1)


def _sign_dist(a, b):
    return min(float(torch.linalg.norm(a - b)), float(torch.linalg.norm(a + b)))


class TestIngest:
    def test_zero_simulation_rejected_columns(self, cuda):
        st = basis.ingest_simulation(basis.isvd_init(np.zeros(6), tol_svd=1e-8), np.zeros((6, 4)))
        assert st.rank == 0 and st.k == 5 and st.n_rejected == 5

    def test_single_column_equals_one_update(self, cuda):
        rng = np.random.default_rng(6)
        x0, x1 = rng.standard_normal(8), rng.standard_normal(8)
        st = basis.isvd_init(x0, tol_svd=1e-8)
        a = basis.ingest_simulation(st, x1[:, None])
        b = basis.isvd_update(st, x1)
        assert torch.equal(a.sigma, b.sigma) and torch.equal(a.phi, b.phi)

    def test_rank_matches_batch_over_two_samples(self, cuda):
        grid = TimeGrid.uniform(0.02, 20)
        u = torch.cat([fom_march(heat1d(12, k), grid).states for k in (0.8, 1.6)], dim=1)
        st = basis.ingest_simulation(basis.isvd_init(u[:, 0], tol_svd=0.0), u[:, 1:])
        _, sigma, _ = linalg.thin_svd(u)
        assert st.rank == sigma.numel() == 12
        lead = sigma > 1e-6 * sigma[0]
        np.testing.assert_allclose(npy(st.sigma[lead]), npy(sigma[lead]), rtol=1e-8)


class TestBatchPod:
    def test_orthogonal_columns(self, cuda):
        u = np.zeros((4, 2))
        u[0, 0], u[1, 1] = 3.0, 2.0
        phi, sigma, _ = basis.batch_pod(u, 2)
        np.testing.assert_allclose(npy(sigma[:2]), [3.0, 2.0])
        np.testing.assert_allclose(np.abs(npy(phi)), np.eye(4)[:, :2])

    def test_rejections(self, cuda):
        with pytest.raises(BasisError):
            basis.batch_pod(np.eye(3), 0)
        with pytest.raises(BasisError, match="rank 1"):
            basis.batch_pod(np.outer(np.arange(1.0, 5.0), np.ones(3)), 2)

    def test_projection_error_is_singular_tail(self, cuda):
        u = np.random.default_rng(7).standard_normal((20, 8))
        phi, sigma, _ = basis.batch_pod(u, 3)
        phi, sigma = npy(phi), npy(sigma)
        err_sq = np.linalg.norm(u - phi @ (phi.T @ u)) ** 2
        assert abs(err_sq - np.sum(sigma[3:] ** 2)) <= 1e-10


class TestTemporalSnapshots:
    def test_slicing(self, cuda):
        v = np.arange(12.0).reshape(6, 2)
        assert np.array_equal(npy(basis.temporal_snapshots(v, 0, 6, 1))[:, 0], v[:, 0])
        v = np.arange(1.0, 7.0)[:, None]
        assert np.array_equal(npy(basis.temporal_snapshots(v, 0, 3, 2)), [[1.0, 4.0], [2.0, 5.0], [3.0, 6.0]])
        v = np.random.default_rng(8).standard_normal((12, 3))
        assert np.array_equal(npy(basis.temporal_snapshots(v, 2, 4, 3)).T.ravel(), v[:, 2])
        with pytest.raises(IndexError):
            basis.temporal_snapshots(np.ones((6, 2)), 2, 3, 2)


class TestBuildBasisSet:
    def test_single_sample_temporal_is_normalized_slice(self, cuda):
        st, _ = trained([1.0])
        bs = basis.build_basis_set(st, 3, 1, 15, 1)
        for i in range(3):
            sl = st.v[:, i]
            assert _sign_dist(bs.temporal[i][:, 0], sl / torch.linalg.norm(sl)) <= 1e-12

    def test_matches_batch_pipeline_and_pod(self, cuda):
        st, u = trained([0.7, 1.0, 1.9])
        bs = basis.build_basis_set(st, 3, 2, 15, 3)
        assert bs.orthonormality_defect() <= 1e-10
        pod = basis.basis_set_from_pod(u, 3, 2, 15, 3)
        for inc, ref in zip(bs.temporal, pod.temporal):
            for j in range(2):
                assert _sign_dist(inc[:, j], ref[:, j]) <= 1e-7
        for i in range(3):
            assert _sign_dist(bs.phi_s[:, i], pod.phi_s[:, i]) <= 1e-7

    def test_dimension_errors_and_stack_layout(self, cuda):
        st, _ = trained([1.0])
        with pytest.raises(BasisError, match="rank"):
            basis.build_basis_set(st, 99, 1, 15, 1)
        with pytest.raises(BasisError, match="ceiling"):
            basis.build_basis_set(st, 2, 2, 15, 1)
        st, _ = trained([0.7, 1.9])
        bs = basis.build_basis_set(st, 2, 2, 15, 2)
        stack = bs.temporal_stack()
        assert tuple(stack.shape) == (2, 15, 2) and torch.equal(stack[1], bs.temporal[1])


def test_large_host_arrays_are_staged_exactly(cuda):
    """_tensors.h2d_numpy: host arrays of 32 MB and more go through alternating pinned
    buffers; C and Fortran order, sizes that are not a multiple of the chunk, other dtypes."""
    from paper_1910_01260_b200._tensors import h2d_numpy, to_dev

    rng = np.random.default_rng(0)
    a = rng.standard_normal((70_001, 97))                     # 54 MB, C order
    t = h2d_numpy(a)
    assert t.shape == a.shape and t.is_contiguous()
    np.testing.assert_array_equal(t.cpu().numpy(), a)
    f = np.asfortranarray(a)                                   # Fortran order: strides kept
    tf = h2d_numpy(f)
    assert tf.shape == f.shape and tf.stride() == (1, f.shape[0])
    np.testing.assert_array_equal(tf.cpu().numpy(), f)
    i = rng.integers(0, 1 << 30, 9_000_003).astype(np.int32)   # 36 MB of int32
    np.testing.assert_array_equal(h2d_numpy(i).cpu().numpy(), i)
    np.testing.assert_array_equal(to_dev(a[:, ::2]).cpu().numpy(), a[:, ::2])  # strided: plain path
    ro = a.copy()
    ro.flags.writeable = False
    np.testing.assert_array_equal(h2d_numpy(ro).cpu().numpy(), ro)
