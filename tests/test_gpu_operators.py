"""Parity of the device temporal bases, spatial/space-time operators, and dense
kernels with the CPU oracle and the reference golden vectors.

Bars (SURVEY 8(c), P2 stage-isolated): temporal bases sign-aligned <= 1e-11;
reduced operators <= 1e-12 relative max-abs; ST solution <= 1e-10 relative;
block assembly vs explicit Kronecker projection <= 1e-11 (verify.py:158).
"""

import numpy as np
import pytest
import scipy.sparse as sp
import torch

from oracle import strom_oracle as so
from paper_1910_01260_b200 import (BasisSet, LinearDynamicalSystem, SingularMatrixError, TimeGrid, basis,
                                   linalg, spacetime, spatial, workloads as wl)

from conftest import load_golden
from helpers import align_columns, max_rel, npy

pytestmark = pytest.mark.gpu


# ------------------------------------------------------------------ linalg (test_linalg.py)
class TestDenseKernels:
    def test_thin_svd_kats(self, cuda):
        w, s, v = linalg.thin_svd(np.diag([3.0, 2.0]))
        assert np.array_equal(npy(s), [3.0, 2.0])
        assert np.array_equal(npy(w), np.eye(2)) and np.array_equal(npy(v), np.eye(2))
        _, s, _ = linalg.thin_svd(np.eye(2))
        np.testing.assert_allclose(npy(s), [1.0, 1.0])

    def test_thin_svd_golden(self, cuda):
        g = load_golden("golden_linalg.npz")
        for key in ("rand64", "rand87", "wide", "core10"):
            m = g[f"svd_{key}_in"]
            w, s, v = (npy(t) for t in linalg.thin_svd(m))
            np.testing.assert_allclose(s, g[f"svd_{key}_s"], rtol=1e-13, atol=1e-15)
            # same sign rule -> same vectors, not just up to sign
            assert max_rel(w, g[f"svd_{key}_w"]) <= 1e-12
            assert max_rel(v, g[f"svd_{key}_v"]) <= 1e-12
            assert np.linalg.norm(m - w @ np.diag(s) @ v.T) <= 1e-12 * np.linalg.norm(m)

    def test_thin_svd_rejects_nonfinite(self, cuda):
        with pytest.raises(ValueError):
            linalg.thin_svd(np.array([[np.nan, 1.0]]))

    def test_qr(self, cuda):
        g = load_golden("golden_linalg.npz")
        for key in ("qr83", "qr34"):
            q, r = linalg.qr(g[f"{key}_in"])
            assert max_rel(npy(q), g[f"{key}_q"]) <= 1e-13
            assert max_rel(npy(r), g[f"{key}_r"]) <= 1e-13
        q, r = linalg.qr(np.eye(3))
        np.testing.assert_allclose(npy(q), np.eye(3)); np.testing.assert_allclose(npy(r), np.eye(3))
        m = np.ones((4, 2))
        q, r = linalg.qr(m)
        assert np.linalg.norm(m - npy(q) @ npy(r)) <= 1e-12 * np.linalg.norm(m)

    def test_solve(self, cuda):
        g = load_golden("golden_linalg.npz")
        x = npy(linalg.solve_dense(g["solve_a"], g["solve_b"]))
        assert max_rel(x, g["solve_x"]) <= 1e-13
        np.testing.assert_allclose(npy(linalg.solve_dense(np.diag([2.0, 4.0]), np.array([2.0, 8.0]))), [1.0, 2.0])
        with pytest.raises(SingularMatrixError, match="pivot 1"):
            linalg.solve_dense(np.array([[1.0, 2.0], [2.0, 4.0]]), np.ones(2))

    @pytest.mark.parametrize("n", [40, 333, 1000])
    def test_solve_sizes(self, cuda, n):
        rng = np.random.default_rng(n)
        a = rng.standard_normal((n, n)) + 0.5 * np.sqrt(n) * np.eye(n)
        b = rng.standard_normal(n)
        x = npy(linalg.solve_dense(a, b))
        ref = so.solve_dense(a, b)
        assert max_rel(x, ref) <= 1e-10
        assert np.linalg.norm(a @ x - b) <= 1e-10 * (np.linalg.norm(a) * np.linalg.norm(x) + np.linalg.norm(b))


# ------------------------------------------------------------------ temporal bases
class TestTemporalBases:
    def test_stage_isolated_vs_oracle(self, cuda):
        """P2: temporal SVDs of the oracle's own V (cfg1)."""
        g = load_golden("golden_isvd_small.npz")
        st = so.stream(g["tb_in"], 0.0)
        _, temporal, ranks = so.basis_set(st, 3, 2, 15, 3)
        v_cm = torch.as_tensor(np.asfortranarray(st.v).T.copy(), device="cuda")  # (r, k) == col-major k x r
        psi, dranks, _ = linalg._temporal_batch(v_cm, st.v.shape[0], st.rank, 15, 3, 3, 2)
        assert list(npy(dranks)) == ranks
        for i in range(3):
            assert np.max(np.abs(npy(psi[i]) - temporal[i])) <= 1e-11  # same sign rule: no alignment

    def test_cfg1_temporal_stage_isolated(self, cuda):
        g = load_golden("golden_cfg1.npz")
        dt = wl.cfg1_dt()
        u = np.hstack([so.fom_march(d.a, d.b, d.x0, dt, d.inputs) for d in map(wl.cfg1_system, wl.CFG1_TRAIN_NU)])
        st = so.stream(u, wl.CFG1_TOL, tol_sv=wl.CFG1_TOL)
        _, temporal, ranks = so.basis_set(st, 10, 4, 100, 4)
        v_cm = torch.as_tensor(np.ascontiguousarray(st.v.T), device="cuda")
        psi, dranks, _ = linalg._temporal_batch(v_cm, st.v.shape[0], st.rank, 100, 4, 10, 4)
        assert list(npy(dranks)) == ranks
        assert np.max(np.abs(npy(psi) - np.stack(temporal))) <= 1e-11
        assert np.max(np.abs(npy(psi) - g["temporal"])) <= 1e-11

    def test_build_basis_set_errors_and_layout(self, cuda):
        g = load_golden("golden_isvd_small.npz")
        st = basis.ingest_simulation(basis.isvd_init(g["tb_in"][:, 0], 0.0), g["tb_in"][:, 1:])
        bs = basis.build_basis_set(st, 3, 2, 15, 3)
        assert tuple(bs.temporal_stack().shape) == (3, 15, 2)
        assert bs.orthonormality_defect() <= 1e-10
        for i in range(3):
            pa, _ = align_columns(npy(bs.temporal[i]), g["tb_temporal"][i])
            assert np.max(np.abs(pa - g["tb_temporal"][i])) <= 1e-7  # incremental-vs-batch level (test_basis.py:242)
        with pytest.raises(basis.BasisError, match="rank"):
            basis.build_basis_set(st, 99, 1, 15, 3)
        with pytest.raises(basis.BasisError, match="ceiling"):
            basis.build_basis_set(st, 2, 4, 15, 3)

    def test_temporal_snapshot_slicing(self, cuda):
        v = np.arange(1.0, 7.0)[:, None]
        t = basis.temporal_snapshots(v, 0, 3, 2)
        assert np.array_equal(npy(t), [[1.0, 4.0], [2.0, 5.0], [3.0, 6.0]])
        with pytest.raises(IndexError):
            basis.temporal_snapshots(np.ones((6, 2)), 2, 3, 2)


# ------------------------------------------------------------------ spatial + space-time
def _lds_from_golden(g, p):
    f = g[p + "f"]
    return LinearDynamicalSystem(a=sp.csr_array(g[p + "a"]), b=sp.csr_array(g[p + "b"]), c=g[p + "c"],
                                 x0=g[p + "x0"], input_signal=lambda k: f[:, k - 1])


class TestBlockAssembly:
    @pytest.mark.parametrize("trial", range(5))
    def test_vs_golden_and_kronecker(self, cuda, trial):
        g = load_golden("golden_blocks.npz")
        p = f"t{trial}_"
        sys_ = _lds_from_golden(g, p)
        grid = TimeGrid(g[p + "dt"])
        bs = BasisSet(g[p + "phi"], tuple(g[p + "temporal"]), n_mu=2)
        srom = spatial.build_spatial_rom(sys_, bs, ref_mode="zero")
        assert max_rel(srom.a_hat, g[p + "a_hat"]) <= 1e-12
        assert max_rel(srom.b_hat, g[p + "b_hat"]) <= 1e-12
        assert max_rel(srom.x0_hat, g[p + "x0_hat"]) <= 1e-12
        a = spacetime.build_st_matrix(srom, bs, grid)
        f = spacetime.build_st_input(srom, bs, grid, sys_.input_signal)
        i0 = spacetime.build_st_init(srom, bs)
        assert max_rel(a, g[p + "a_blk"]) <= 1e-12
        assert max_rel(f, g[p + "f_blk"]) <= 1e-12
        assert max_rel(i0, g[p + "i_blk"]) <= 1e-12
        assert np.max(np.abs(npy(a) - g[p + "a_exp"])) <= 1e-11
        assert np.max(np.abs(npy(f) - g[p + "f_exp"])) <= 1e-11
        assert np.max(np.abs(npy(i0) - g[p + "i_exp"])) <= 1e-11
        rom = spacetime.build_st_rom(srom, bs, grid, sys_.input_signal)
        assert max_rel(spacetime.solve_st_rom(rom), g[p + "x_st"]) <= 1e-10

    def test_collapses_to_single_block(self, cuda):
        a_hat = np.array([[-2.0, 0.3], [0.1, -1.5]])
        bs = BasisSet(np.eye(2), (np.ones((1, 1)), np.ones((1, 1))), n_mu=1)
        srom = spatial.SpatialRom(a_hat=torch.as_tensor(a_hat, device="cuda"),
                                  b_hat=torch.zeros((2, 1), dtype=torch.float64, device="cuda"),
                                  c_hat=None, x_ref=None, x_ref_hat=None,
                                  x0_hat=torch.zeros(2, dtype=torch.float64, device="cuda"), y_ref=None,
                                  ref_mode="zero")
        out = spacetime.build_st_matrix(srom, bs, TimeGrid.uniform(0.25, 1))
        np.testing.assert_allclose(npy(out), np.eye(2) - 0.25 * a_hat, atol=1e-14)

    def test_constant_path_equals_general(self, cuda):
        rng = np.random.default_rng(8)
        phi, temporal = wl.random_basis(rng, 6, 7, 3, 2)
        bs = BasisSet(phi, temporal, n_mu=2)
        b_hat = rng.standard_normal((3, 2))
        srom = spatial.SpatialRom(a_hat=torch.zeros((3, 3), dtype=torch.float64, device="cuda"),
                                  b_hat=torch.as_tensor(b_hat, device="cuda"), c_hat=None, x_ref=None,
                                  x_ref_hat=None, x0_hat=torch.zeros(3, dtype=torch.float64, device="cuda"),
                                  y_ref=None, ref_mode="zero")
        grid = TimeGrid(rng.uniform(0.05, 0.2, 7))
        f = rng.standard_normal(2)
        gen = spacetime.build_st_input(srom, bs, grid, lambda k: f, constant_input=False)
        fast = spacetime.build_st_input(srom, bs, grid, lambda k: f, constant_input=True)
        assert float((gen - fast).abs().max()) <= 1e-13

    def test_initial_state_reference_zeroes_x0hat(self, cuda):
        rng = np.random.default_rng(1)
        d = wl.random_stable_system(rng, 8)
        sys_ = LinearDynamicalSystem(a=d["a"], b=d["b"], c=d["c"], x0=d["x0"], input_signal=d["inputs"])
        phi, temporal = wl.random_basis(rng, 8, 4, 3, 2)
        rom = spatial.build_spatial_rom(sys_, BasisSet(phi, temporal, 2), ref_mode="initial_state")
        assert torch.equal(rom.x0_hat, torch.zeros(3, dtype=torch.float64, device="cuda"))
        with pytest.raises(ValueError, match="zero-reference"):
            spacetime.build_st_rom(rom, BasisSet(phi, temporal, 2), TimeGrid.uniform(0.1, 4), d["inputs"])

    def test_triple_product_extended_precision(self, cuda):
        rng = np.random.default_rng(2)
        d = wl.random_stable_system(rng, 12)
        sys_ = LinearDynamicalSystem(a=d["a"], b=d["b"], c=d["c"], x0=d["x0"], input_signal=d["inputs"])
        phi, temporal = wl.random_basis(rng, 12, 4, 3, 2)
        rom = spatial.build_spatial_rom(sys_, BasisSet(phi, temporal, 2), ref_mode="zero")
        phi_ld = phi.astype(np.longdouble)
        expected = (phi_ld.T @ d["a"].toarray().astype(np.longdouble) @ phi_ld).astype(float)
        assert np.max(np.abs(npy(rom.a_hat) - expected)) <= 1e-12

    def test_errors(self, cuda):
        rng = np.random.default_rng(3)
        d = wl.random_stable_system(rng, 5)
        sys_ = LinearDynamicalSystem(a=d["a"], b=d["b"], c=d["c"], x0=d["x0"], input_signal=d["inputs"])
        phi, temporal = wl.random_basis(rng, 6, 4, 2, 1)
        with pytest.raises(ValueError):
            spatial.build_spatial_rom(sys_, BasisSet(phi, temporal, 1))
        phi, temporal = wl.random_basis(rng, 5, 4, 2, 1)
        with pytest.raises(ValueError):
            spatial.build_spatial_rom(sys_, BasisSet(phi, temporal, 1), ref_mode="average")
        rom = spatial.build_spatial_rom(sys_, BasisSet(phi, temporal, 1), ref_mode="zero")
        with pytest.raises(ValueError):
            spacetime.build_st_matrix(rom, BasisSet(phi, temporal, 1), TimeGrid.uniform(0.1, 5))

    def test_scalar_solve_kat(self, cuda):
        bs = BasisSet(np.ones((1, 1)), (np.ones((1, 1)),), n_mu=1)
        rom = spacetime.SpaceTimeRom(torch.tensor([[4.0]], dtype=torch.float64, device="cuda"),
                                     torch.tensor([2.0], dtype=torch.float64, device="cuda"),
                                     torch.tensor([6.0], dtype=torch.float64, device="cuda"), bs)
        np.testing.assert_allclose(npy(spacetime.solve_st_rom(rom)), [2.0])


class TestCfg4:
    def test_small_instance_vs_golden(self, cuda):
        g = load_golden("golden_cfg4_small.npz")
        d = wl.cfg4_inputs(nx=10, n_s=8, n_t=4, n_steps=20, dt=1e-3)
        sys_ = LinearDynamicalSystem(a=d.a, b=d.b, c=d.c, x0=d.x0, input_signal=d.inputs, constant_input=True)
        bs = BasisSet(d.phi_s, d.temporal, n_mu=4)
        grid = TimeGrid(d.dt)
        srom = spatial.build_spatial_rom(sys_, bs, ref_mode="zero")
        for key in ("a_hat", "b_hat", "c_hat", "x0_hat"):
            assert max_rel(getattr(srom, key), g[key]) <= 1e-12, key
        rom = spacetime.build_st_rom(srom, bs, grid, sys_.input_signal, True)
        assert max_rel(rom.a_st_hat, g["a_st"]) <= 1e-12
        assert max_rel(rom.f_st_hat, g["f_st"]) <= 1e-12
        assert max_rel(rom.x0_st_hat, g["x0_st"]) <= 1e-12
        assert np.max(np.abs(npy(rom.a_st_hat) - g["a_exp"])) <= 1e-11
        assert max_rel(spacetime.solve_st_rom(rom), g["x_st"]) <= 1e-10

    def test_kronecker_check_instance(self, cuda):
        """BASELINE configs[3]'s stated check instance: 20^3 cells, N_t = 50, n_s = 50,
        n_t = 20, against the reference's explicit Kronecker assembly
        (spacetime.py:189-210, system.py:166-194, the verify.py:124-158 bar 1e-11)
        stored as seeded samples + checksums (tests/golden/golden_cfg4_kron.npz)."""
        g = load_golden("golden_cfg4_kron.npz")
        d = wl.cfg4_inputs(nx=20, n_s=50, n_t=20, n_steps=50, dt=1e-3)
        sys_ = LinearDynamicalSystem(a=d.a, b=d.b, c=d.c, x0=d.x0, input_signal=d.inputs, constant_input=True)
        bs = BasisSet(d.phi_s, d.temporal, n_mu=20)
        grid = TimeGrid(d.dt)
        srom = spatial.build_spatial_rom(sys_, bs, ref_mode="zero")
        for key in ("a_hat", "b_hat", "x0_hat"):
            assert max_rel(getattr(srom, key), g[key]) <= 1e-12, key
        rom = spacetime.build_st_rom(srom, bs, grid, sys_.input_signal, True)
        a = npy(rom.a_st_hat)
        idx = g["sample_idx"]
        assert max_rel(a.ravel()[idx], g["a_blk_sample"]) <= 1e-12
        assert np.max(np.abs(a.ravel()[idx] - g["a_exp_sample"])) <= 1e-11
        assert np.max(np.abs(np.diag(a) - g["a_exp_diag"])) <= 1e-11
        assert np.max(np.abs(a.sum(axis=1) - g["a_exp_rowsum"])) <= 1e-10
        assert np.max(np.abs(a.sum(axis=0) - g["a_exp_colsum"])) <= 1e-10
        assert abs(np.linalg.norm(a) - float(g["a_exp_fro"])) <= 1e-11 * float(g["a_exp_fro"])
        assert np.max(np.abs(npy(rom.f_st_hat) - g["f_exp"])) <= 1e-11
        assert np.max(np.abs(npy(rom.x0_st_hat) - g["i_exp"])) <= 1e-11
        assert max_rel(spacetime.solve_st_rom(rom), g["x_st"]) <= 1e-10

    def test_full_size_vs_oracle(self, cuda):
        """BASELINE config 4 at full size (N = 10^6, n_s = 50, n_t = 20, N_t = 500)."""
        d = wl.cfg4_inputs()
        sys_ = LinearDynamicalSystem(a=d.a, b=d.b, c=d.c, x0=d.x0, input_signal=d.inputs, constant_input=True)
        bs = BasisSet(d.phi_s, d.temporal, n_mu=20)
        grid = TimeGrid(d.dt)
        srom = spatial.build_spatial_rom(sys_, bs, ref_mode="zero")
        rom = spacetime.build_st_rom(srom, bs, grid, sys_.input_signal, True)
        ref = so.spatial_rom(d.a, d.b, d.c, d.x0, d.phi_s, "zero")
        assert max_rel(srom.a_hat, ref.a_hat) <= 1e-12
        assert max_rel(srom.b_hat, ref.b_hat) <= 1e-12
        assert max_rel(srom.x0_hat, ref.x0_hat) <= 1e-12
        a_st = so.st_matrix(ref.a_hat, d.temporal, d.dt)
        f_st = so.st_input(ref.b_hat, d.temporal, d.dt, d.inputs, True)
        x0_st = so.st_init(ref.x0_hat, d.temporal)
        assert max_rel(rom.a_st_hat, a_st) <= 1e-12
        assert max_rel(rom.f_st_hat, f_st) <= 1e-12
        assert max_rel(rom.x0_st_hat, x0_st) <= 1e-12
        x_ref = so.st_solve(a_st, f_st, x0_st)
        assert max_rel(spacetime.solve_st_rom(rom), x_ref) <= 1e-10


class TestCfg1EndToEnd:
    def test_st_rom_solution(self, cuda):
        """Free-running config 1: device iSVD -> bases -> operators -> solve vs the reference.

        North-star bar 1e-8 on the ST-ROM solution, or 10x the reference's own
        reduction-order envelope when that is larger."""
        from test_gpu_isvd import cfg1_snapshots

        g = load_golden("golden_cfg1.npz")
        dt = wl.cfg1_dt()
        u = cfg1_snapshots()
        t = wl.cfg1_system(wl.CFG1_TEST_NU)

        def ref_states(rows):
            st = so.stream(u[rows], wl.CFG1_TOL, tol_sv=wl.CFG1_TOL)
            phi_s, temporal, _ = so.basis_set(st, wl.CFG1_NS, wl.CFG1_NTMODES, wl.CFG1_NT, 4)
            a = t.a[rows][:, rows]
            o = so.spatial_rom(a, t.b[rows], t.c[rows], t.x0[rows], phi_s, "zero")
            xs = so.st_solve(so.st_matrix(o.a_hat, temporal, dt), so.st_input(o.b_hat, temporal, dt, t.inputs, True),
                             so.st_init(o.x0_hat, temporal))
            out = np.empty((u.shape[0], wl.CFG1_NT))
            out[rows] = so.st_reconstruct(phi_s, temporal, xs)
            return out

        base = np.arange(u.shape[0])
        ref = ref_states(base)
        env = 0.0
        for sd in (0, 1, 2):
            perm = np.random.default_rng(sd).permutation(u.shape[0])
            env = max(env, float(np.max(np.linalg.norm(ref_states(perm) - ref, axis=0) / np.linalg.norm(ref, axis=0))))
        st = basis.isvd_init(u[:, 0], wl.CFG1_TOL, tol_sv=wl.CFG1_TOL)
        st = basis.ingest_simulation(st, torch.as_tensor(u[:, 1:], device="cuda"))
        bs = basis.build_basis_set(st, wl.CFG1_NS, wl.CFG1_NTMODES, wl.CFG1_NT, 4)
        sys_ = LinearDynamicalSystem(a=t.a, b=t.b, c=t.c, x0=t.x0, input_signal=t.inputs, constant_input=True)
        srom = spatial.build_spatial_rom(sys_, bs, ref_mode="zero")
        rom = spacetime.build_st_rom(srom, bs, TimeGrid(dt), sys_.input_signal, True)
        states = npy(spacetime.reconstruct_states(bs, spacetime.solve_st_rom(rom)))
        rel = float(np.max(np.linalg.norm(states - ref, axis=0) / np.linalg.norm(ref, axis=0)))
        print(f"cfg1 ST-ROM states rel vs reference {rel:.2e}; reference reduction-order envelope {env:.2e}")
        assert np.allclose(ref.sum(axis=0), g["states_colsum"], rtol=1e-12)
        assert rel <= max(1e-8, 10 * env)


def test_solve_dense_leaves_inputs_untouched(cuda):
    """solve_dense is pure like the reference's (linalg.py:75-99): a 1-D right-hand side
    must not be overwritten by the in-place device solve."""
    rng = np.random.default_rng(40)
    a = torch.as_tensor(rng.standard_normal((40, 40)) + 2.0 * np.eye(40), device="cuda")
    b = torch.as_tensor(rng.standard_normal(40), device="cuda")
    a0, b0 = a.clone(), b.clone()
    x1 = linalg.solve_dense(a, b)
    x2 = linalg.solve_dense(a, b)
    assert torch.equal(a, a0) and torch.equal(b, b0) and torch.equal(x1, x2)
    assert float(torch.linalg.norm(a @ x1 - b)) <= 1e-12 * float(torch.linalg.norm(b))
