"""Pin the CPU oracle against golden vectors produced by the real reference.

The fixtures come from tests/golden/make_golden.py (which imports the
reference's ``strom``).  The oracle performs the same numpy operations in the
same order, so on this image it reproduces them bit for bit; the tolerance
below only absorbs a different OpenBLAS kernel selection on another host.
"""

import numpy as np
import pytest

from oracle import strom_oracle as so
from paper_1910_01260_b200 import workloads as wl

from conftest import load_golden

TIGHT = 1e-13


def _close(a, b, tol=TIGHT):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    scale = max(1.0, float(np.max(np.abs(b)))) if b.size else 1.0
    assert np.max(np.abs(a - b), initial=0.0) <= tol * scale


def _check_state(st, g, prefix, tol=TIGHT):
    _close(st.sigma, g[f"{prefix}_sigma"], tol)
    _close(st.phi, g[f"{prefix}_phi"], tol)
    _close(st.v, g[f"{prefix}_v"], tol)
    cnt = [st.k, st.n_rejected, st.n_dependent, st.n_truncated, st.n_restarts]
    assert cnt == list(g[f"{prefix}_counters"])


class TestLinalg:
    def test_thin_svd(self):
        g = load_golden("golden_linalg.npz")
        for key in ("rand64", "rand87", "wide", "diag", "eye", "core10"):
            w, s, v = so.thin_svd(g[f"svd_{key}_in"])
            _close(w, g[f"svd_{key}_w"]); _close(s, g[f"svd_{key}_s"]); _close(v, g[f"svd_{key}_v"])

    def test_diag_kat_exact(self):
        w, s, v = so.thin_svd(np.diag([3.0, 2.0]))
        assert np.array_equal(w, np.eye(2)) and np.array_equal(v, np.eye(2))

    def test_qr(self):
        g = load_golden("golden_linalg.npz")
        for key in ("qr83", "qr34", "qr_ones"):
            q, r = so.qr_pos(g[f"{key}_in"])
            _close(q, g[f"{key}_q"]); _close(r, g[f"{key}_r"])
        assert np.all(np.diag(so.qr_pos(g["qr83_in"])[1]) >= 0)

    def test_solve(self):
        g = load_golden("golden_linalg.npz")
        _close(so.solve_dense(g["solve_a"], g["solve_b"]), g["solve_x"])
        with pytest.raises(so.OracleSingularMatrixError, match="pivot 1"):
            so.solve_dense(np.array([[1.0, 2.0], [2.0, 4.0]]), np.ones(2))


class TestIsvdKat:
    def test_kats(self):
        g = load_golden("golden_isvd_small.npz")
        _check_state(so.init(np.array([0.0, 2.0, 0.0]), 1e-8), g, "kat_init")
        st = so.update(so.init(np.array([1.0, 0, 0]), 1e-8), np.array([0.0, 1.0, 0]))
        _check_state(st, g, "kat_e1e2")
        e1 = np.array([1.0, 0, 0])
        _check_state(so.update(so.init(e1, 1e-8), e1), g, "kat_e1e1")

    def test_rejections(self):
        st = so.init(np.zeros(3), 1e-8)
        assert st.rank == 0 and st.phi.shape == (3, 0) and st.v.shape == (1, 0)
        assert so.init(np.array([0.5, 0.0]), 0.5).rank == 0
        st = so.ingest(so.init(np.zeros(6), 1e-8), np.zeros((6, 4)))
        assert st.rank == 0 and st.k == 5 and st.n_rejected == 5


class TestIsvdStreams:
    @pytest.mark.parametrize("prefix,tol,kw", [
        ("rand", 0.0, {}), ("orth", 1e-10, {}), ("heat", 0.0, {}), ("tb", 0.0, {}),
    ])
    def test_stream(self, prefix, tol, kw):
        g = load_golden("golden_isvd_small.npz")
        st = so.stream(g[f"{prefix}_in"], tol, **kw)
        _check_state(st, g, prefix)

    def test_duplicates(self):
        g = load_golden("golden_isvd_small.npz")
        x = g["dup_in"]
        st = so.init(x, 0.0)
        for _ in range(5):
            st = so.update(st, x)
        _check_state(st, g, "dup")

    def test_truncate_and_restart(self):
        g = load_golden("golden_isvd_small.npz")
        st = so.stream(g["trunc_in"], 1e-10, r_max=5, cap_mode="truncate")
        _check_state(st, g, "trunc")
        cols = g["restart_in"]
        st = so.update(so.init(cols[:, 0], 1e-10, r_max=2), cols[:, 1])
        with pytest.warns(RuntimeWarning, match="r_max"):
            st = so.update(st, cols[:, 2])
        _check_state(st, g, "restart")

    def test_inspan(self):
        g = load_golden("golden_isvd_small.npz")
        cols = g["inspan_in"]
        st = so.stream(cols[:, :3], 1e-6)
        st = so.update(st, cols[:, 3])
        _check_state(st, g, "inspan")
        assert st.n_dependent == 1

    def test_temporal_bases(self):
        g = load_golden("golden_isvd_small.npz")
        st = so.stream(g["tb_in"], 0.0)
        phi_s, temporal, _ = so.basis_set(st, 3, 2, 15, 3)
        _close(phi_s, g["tb_phi_s"])
        _close(np.stack(temporal), g["tb_temporal"])
        with pytest.raises(so.OracleBasisError, match="rank"):
            so.basis_set(st, 99, 1, 15, 3)
        with pytest.raises(so.OracleBasisError, match="ceiling"):
            so.basis_set(st, 2, 4, 15, 3)


class TestCfg1Pipeline:
    def test_full_pipeline(self):
        g = load_golden("golden_cfg1.npz")
        dt = wl.cfg1_dt()
        mats = []
        for nu in wl.CFG1_TRAIN_NU:
            d = wl.cfg1_system(nu)
            mats.append(so.fom_march(d.a, d.b, d.x0, dt, d.inputs))
        u = np.hstack(mats)
        # the snapshot producer itself is pinned by checksums
        _close(u.sum(axis=0), g["u_colsum"]); _close(np.abs(u).sum(axis=0), g["u_abssum"])
        _close(u[::97, ::7], g["u_sample"])
        st = so.init(u[:, 0], wl.CFG1_TOL, tol_sv=wl.CFG1_TOL)
        ranks = [st.rank]
        for c in range(1, u.shape[1]):
            st = so.update(st, u[:, c])
            ranks.append(st.rank)
        assert ranks == list(g["ranks"])
        _close(st.sigma, g["sigma"]); _close(st.phi[:, :10], g["phi10"]); _close(st.v[:, :10], g["v10"])
        assert [st.k, st.n_rejected, st.n_dependent, st.n_truncated, st.n_restarts] == list(g["counters"])
        with pytest.raises(so.OracleBasisError, match="ceiling"):
            so.basis_set(st, wl.CFG1_NS, 5, wl.CFG1_NT, 4)
        phi_s, temporal, _ = so.basis_set(st, wl.CFG1_NS, wl.CFG1_NTMODES, wl.CFG1_NT, 4)
        _close(phi_s, g["phi_s"]); _close(np.stack(temporal), g["temporal"])
        t = wl.cfg1_system(wl.CFG1_TEST_NU)
        sr = so.spatial_rom(t.a, t.b, t.c, t.x0, phi_s, "zero")
        _close(sr.a_hat, g["a_hat"]); _close(sr.x0_hat, g["x0_hat"])
        a_st = so.st_matrix(sr.a_hat, temporal, dt)
        f_st = so.st_input(sr.b_hat, temporal, dt, t.inputs, True)
        x0_st = so.st_init(sr.x0_hat, temporal)
        _close(a_st, g["a_st"]); _close(f_st, g["f_st"]); _close(x0_st, g["x0_st"])
        _close(so.st_solve(a_st, f_st, x0_st), g["x_st"], 1e-12)


class TestBlockAssembly:
    @pytest.mark.parametrize("trial", range(5))
    def test_blocks(self, trial):
        g = load_golden("golden_blocks.npz")
        p = f"t{trial}_"
        f = g[p + "f"]
        sr = so.spatial_rom(g[p + "a"], g[p + "b"], g[p + "c"], g[p + "x0"], g[p + "phi"], "zero")
        _close(sr.a_hat, g[p + "a_hat"]); _close(sr.b_hat, g[p + "b_hat"])
        temporal = tuple(g[p + "temporal"])
        dt = g[p + "dt"]
        a_st = so.st_matrix(sr.a_hat, temporal, dt)
        f_st = so.st_input(sr.b_hat, temporal, dt, lambda k: f[:, k - 1])
        i_st = so.st_init(sr.x0_hat, temporal)
        _close(a_st, g[p + "a_blk"]); _close(f_st, g[p + "f_blk"]); _close(i_st, g[p + "i_blk"])
        # block assembly == explicit Kronecker projection (verify.py:158 threshold 1e-11)
        assert np.max(np.abs(a_st - g[p + "a_exp"])) <= 1e-11
        assert np.max(np.abs(f_st - g[p + "f_exp"])) <= 1e-11
        assert np.max(np.abs(i_st - g[p + "i_exp"])) <= 1e-11
        _close(so.st_solve(a_st, f_st, i_st), g[p + "x_st"], 1e-12)


class TestCfg4Small:
    def test_small_instance(self):
        g = load_golden("golden_cfg4_small.npz")
        d = wl.cfg4_inputs(nx=10, n_s=8, n_t=4, n_steps=20, dt=1e-3)
        assert d.a.nnz == int(g["a_nnz"]) == 7 * 1000 - 6 * 100
        sr = so.spatial_rom(d.a, d.b, d.c, d.x0, d.phi_s, "zero")
        _close(sr.a_hat, g["a_hat"]); _close(sr.b_hat, g["b_hat"]); _close(sr.x0_hat, g["x0_hat"])
        a_st = so.st_matrix(sr.a_hat, d.temporal, d.dt)
        f_st = so.st_input(sr.b_hat, d.temporal, d.dt, d.inputs, True)
        x0_st = so.st_init(sr.x0_hat, d.temporal)
        _close(a_st, g["a_st"]); _close(f_st, g["f_st"]); _close(x0_st, g["x0_st"])
        assert np.max(np.abs(a_st - g["a_exp"])) <= 1e-11
        phi_st = so.explicit_st_basis(d.phi_s, d.temporal)
        a_x, f_x, i_x = so.assemble_st(d.a, d.b, d.x0, d.dt, d.inputs)
        assert np.max(np.abs(phi_st.T @ (a_x @ phi_st) - a_st)) <= 1e-11
        assert np.max(np.abs(phi_st.T @ f_x - f_st)) <= 1e-11
        assert np.max(np.abs(phi_st.T @ i_x - x0_st)) <= 1e-11


class TestCfg4KroneckerInstance:
    def test_baseline_check_instance(self):
        """BASELINE configs[3]'s check instance (20^3 cells, N_t = 50, n_s = 50,
        n_t = 20): the oracle's block assembly against the reference's explicit
        Kronecker assembly (golden samples + checksums, make_golden.gen_cfg4_kron)."""
        g = load_golden("golden_cfg4_kron.npz")
        d = wl.cfg4_inputs(nx=20, n_s=50, n_t=20, n_steps=50, dt=1e-3)
        assert d.a.nnz == int(g["a_nnz"]) == 7 * 20**3 - 6 * 20**2
        assert float(d.a.data.sum()) == float(g["a_datasum"])
        sr = so.spatial_rom(d.a, d.b, d.c, d.x0, d.phi_s, "zero")
        _close(sr.a_hat, g["a_hat"]); _close(sr.b_hat, g["b_hat"]); _close(sr.x0_hat, g["x0_hat"])
        a_st = so.st_matrix(sr.a_hat, d.temporal, d.dt)
        f_st = so.st_input(sr.b_hat, d.temporal, d.dt, d.inputs, True)
        x0_st = so.st_init(sr.x0_hat, d.temporal)
        idx = g["sample_idx"]
        _close(a_st.ravel()[idx], g["a_blk_sample"])
        assert np.max(np.abs(a_st.ravel()[idx] - g["a_exp_sample"])) <= 1e-11
        assert np.max(np.abs(np.diag(a_st) - g["a_exp_diag"])) <= 1e-11
        assert np.max(np.abs(a_st.sum(axis=1) - g["a_exp_rowsum"])) <= 1e-10
        assert np.max(np.abs(a_st.sum(axis=0) - g["a_exp_colsum"])) <= 1e-10
        assert np.max(np.abs(f_st - g["f_exp"])) <= 1e-11
        assert np.max(np.abs(x0_st - g["i_exp"])) <= 1e-11
        _close(so.st_solve(a_st, f_st, x0_st), g["x_st"], 1e-11)
