"""Generate golden vectors by running the REAL reference (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports ``strom`` from /root/reference/pkg/src (read-only, pure Python), runs
its hot-path functions on seeded inputs and stores inputs + outputs as small
``.npz`` fixtures next to this script.  The fixtures travel with the repo; the
reference does not (it is absent on the GPU box).  The oracle restatement
(oracle/strom_oracle.py) is pinned against these files by
tests/test_oracle_golden.py, and the CUDA path is checked against the oracle.
"""

from __future__ import annotations

import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from strom import basis, linalg, spatial, spacetime, system  # noqa: E402
from strom.problems import ProblemSpec, make_heat1d  # noqa: E402
from strom.verify import random_basis_set, random_stable_system  # noqa: E402

from paper_1910_01260_b200 import workloads as wl  # noqa: E402


def _save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def _state_arrays(prefix, st):
    return {
        f"{prefix}_phi": st.phi, f"{prefix}_sigma": st.sigma, f"{prefix}_v": st.v,
        f"{prefix}_counters": np.array([st.k, st.n_rejected, st.n_dependent,
                                        st.n_truncated, st.n_restarts]),
    }


def gen_linalg():
    rng = np.random.default_rng(100)
    out = {}
    mats = {
        "rand64": rng.standard_normal((6, 4)),
        "rand87": rng.standard_normal((8, 7)),
        "wide": rng.standard_normal((3, 9)),
        "diag": np.diag([3.0, 2.0]),
        "eye": np.eye(2),
    }
    # a bordered iSVD core [[diag(s), ell], [0, p]] like basis.py:141-144
    s = np.sort(rng.uniform(0.1, 2.0, 9))[::-1]
    core = np.zeros((10, 10))
    core[:9, :9] = np.diag(s)
    core[:9, 9] = rng.standard_normal(9) * 0.3
    core[9, 9] = 0.05
    mats["core10"] = core
    for k, m in mats.items():
        w, sg, v = linalg.thin_svd(m)
        out[f"svd_{k}_in"], out[f"svd_{k}_w"], out[f"svd_{k}_s"], out[f"svd_{k}_v"] = m, w, sg, v
    for k, m in {"qr83": rng.standard_normal((8, 3)), "qr34": np.array([[3.0], [4.0]]),
                 "qr_ones": np.ones((4, 2))}.items():
        q, r = linalg.qr(m)
        out[f"{k}_in"], out[f"{k}_q"], out[f"{k}_r"] = m, q, r
    a = rng.standard_normal((10, 10)) + 10.0 * np.eye(10)
    b = rng.standard_normal(10)
    out["solve_a"], out["solve_b"], out["solve_x"] = a, b, linalg.solve_dense(a, b)
    _save("golden_linalg.npz", **out)


def gen_isvd_small():
    out = {}
    # KATs from tests/test_basis.py:10-45
    st = basis.isvd_init(np.array([0.0, 2.0, 0.0]), tol_svd=1e-8)
    out.update(_state_arrays("kat_init", st))
    st = basis.isvd_init(np.array([1.0, 0.0, 0.0]), tol_svd=1e-8)
    st = basis.isvd_update(st, np.array([0.0, 1.0, 0.0]))
    out.update(_state_arrays("kat_e1e2", st))
    e1 = np.array([1.0, 0.0, 0.0])
    st = basis.isvd_update(basis.isvd_init(e1, tol_svd=1e-8), e1)
    out.update(_state_arrays("kat_e1e1", st))
    # random 200 x 50, tol 0 (test_basis.py:47-55)
    m = np.random.default_rng(0).standard_normal((200, 50))
    st = basis.ingest_simulation(basis.isvd_init(m[:, 0], tol_svd=0.0), m[:, 1:])
    out["rand_in"] = m
    out.update(_state_arrays("rand", st))
    # exact duplicates, tol 0 (test_basis.py:57-70)
    x = np.random.default_rng(1).standard_normal(30)
    st = basis.isvd_init(x, tol_svd=0.0)
    for _ in range(5):
        st = basis.isvd_update(st, x)
    out["dup_in"] = x
    out.update(_state_arrays("dup", st))
    # truncate cap (test_basis.py:85-96)
    rng = np.random.default_rng(3)
    cols = [rng.standard_normal(20) for _ in range(13)]
    st = basis.isvd_init(cols[0], tol_svd=1e-10, r_max=5, cap_mode="truncate")
    for c in cols[1:]:
        st = basis.isvd_update(st, c)
    out["trunc_in"] = np.column_stack(cols)
    out.update(_state_arrays("trunc", st))
    # restart cap (test_basis.py:98-105)
    rng = np.random.default_rng(4)
    cols = [rng.standard_normal(10) for _ in range(3)]
    st = basis.isvd_init(cols[0], tol_svd=1e-10, r_max=2)
    st = basis.isvd_update(st, cols[1])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        st = basis.isvd_update(st, cols[2])
    out["restart_in"] = np.column_stack(cols)
    out.update(_state_arrays("restart", st))
    # in-span column (test_basis.py:107-117)
    cols = np.random.default_rng(5).standard_normal((15, 3))
    st = basis.ingest_simulation(basis.isvd_init(cols[:, 0], tol_svd=1e-6), cols[:, 1:])
    st = basis.isvd_update(st, cols @ np.array([0.3, -0.2, 1.1]))
    out["inspan_in"] = np.column_stack([cols, cols @ np.array([0.3, -0.2, 1.1])])
    out.update(_state_arrays("inspan", st))
    # orthogonality stream (test_basis.py:77-83)
    rng = np.random.default_rng(2)
    cols = [rng.standard_normal(40) for _ in range(31)]
    st = basis.ingest_simulation(basis.isvd_init(cols[0], tol_svd=1e-10), np.column_stack(cols[1:]))
    out["orth_in"] = np.column_stack(cols)
    out.update(_state_arrays("orth", st))
    # heat1d, two kappas, tol 0 (test_basis.py:135-151)
    grid = system.TimeGrid.uniform(0.02, 20)
    mats = [system.fom_march(make_heat1d(ProblemSpec(kind="heat1d", nx=12), {"kappa": k}), grid).states
            for k in (0.8, 1.6)]
    u = system.snapshot_matrix(mats)
    st = basis.ingest_simulation(basis.isvd_init(u[:, 0], tol_svd=0.0), u[:, 1:])
    out["heat_in"] = u
    out.update(_state_arrays("heat", st))
    # temporal bases of a 3-sample heat1d stream (test_basis.py:203-254)
    grid = system.TimeGrid.uniform(0.02, 15)
    mats = [system.fom_march(make_heat1d(ProblemSpec(kind="heat1d", nx=10), {"kappa": k}), grid).states
            for k in (0.7, 1.0, 1.9)]
    u = system.snapshot_matrix(mats)
    st = basis.ingest_simulation(basis.isvd_init(u[:, 0], tol_svd=0.0), u[:, 1:])
    bs = basis.build_basis_set(st, 3, 2, 15, 3)
    out["tb_in"] = u
    out.update(_state_arrays("tb", st))
    out["tb_phi_s"], out["tb_temporal"] = bs.phi_s, bs.temporal_stack()
    _save("golden_isvd_small.npz", **out)


def gen_cfg1():
    """Full BASELINE config 1 pipeline (n_t = 4; n_t = 5 raises BasisError)."""
    grid = system.TimeGrid.uniform(wl.CFG1_DT, wl.CFG1_NT)

    def lds(nu):
        d = wl.cfg1_system(nu)
        return system.LinearDynamicalSystem(a=d.a, b=d.b, c=d.c, x0=d.x0,
                                            input_signal=d.inputs, constant_input=True)

    mats = [system.fom_march(lds(nu), grid).states for nu in wl.CFG1_TRAIN_NU]
    u = system.snapshot_matrix(mats)
    st = basis.isvd_init(u[:, 0], wl.CFG1_TOL, tol_sv=wl.CFG1_TOL)
    ranks = [st.rank]
    for col in range(1, u.shape[1]):
        st = basis.isvd_update(st, u[:, col])
        ranks.append(st.rank)
    try:
        basis.build_basis_set(st, wl.CFG1_NS, 5, wl.CFG1_NT, 4)
        raise AssertionError("n_t=5 unexpectedly accepted")
    except basis.BasisError as exc:
        assert "ceiling" in str(exc)
    bs = basis.build_basis_set(st, wl.CFG1_NS, wl.CFG1_NTMODES, wl.CFG1_NT, 4)
    test_sys = lds(wl.CFG1_TEST_NU)
    srom = spatial.build_spatial_rom(test_sys, bs, ref_mode="zero")
    rom = spacetime.build_st_rom(srom, bs, grid, test_sys.input_signal, True)
    x_st = spacetime.solve_st_rom(rom)
    states = spacetime.reconstruct_states(bs, x_st)
    fom = system.fom_march(test_sys, grid).states
    out = dict(
        u_colsum=u.sum(axis=0), u_abssum=np.abs(u).sum(axis=0), u_sample=u[::97, ::7],
        ranks=np.array(ranks), sigma=st.sigma, phi10=st.phi[:, :10], v10=st.v[:, :10],
        counters=np.array([st.k, st.n_rejected, st.n_dependent, st.n_truncated, st.n_restarts]),
        phi_s=bs.phi_s, temporal=bs.temporal_stack(),
        a_hat=srom.a_hat, b_hat=srom.b_hat, x0_hat=srom.x0_hat,
        a_st=rom.a_st_hat, f_st=rom.f_st_hat, x0_st=rom.x0_st_hat, x_st=x_st,
        states_colsum=states.sum(axis=0), fom_colsum=fom.sum(axis=0),
        rel_err=np.linalg.norm(states - fom, axis=0) / np.linalg.norm(fom, axis=0),
    )
    _save("golden_cfg1.npz", **out)


def gen_blocks():
    """verify.suite_block_assembly instances (verify.py:124-158) + linear-scaling KATs."""
    out = {}
    for trial in range(5):
        rng = np.random.default_rng(trial)
        sys_ = random_stable_system(rng, 12, n_inputs=2)
        grid = system.TimeGrid(rng.uniform(0.01, 0.1, 8))
        bs = random_basis_set(rng, 12, 8, 3, 2)
        srom = spatial.build_spatial_rom(sys_, bs, ref_mode="zero")
        phi_st = spacetime.explicit_st_basis(bs)
        a_st, f_st, x0_st = system.assemble_st(sys_, grid)
        p = f"t{trial}_"
        out[p + "a"] = sys_.a.toarray()
        out[p + "b"] = sys_.b.toarray()
        out[p + "c"] = sys_.c
        out[p + "x0"] = sys_.x0
        out[p + "f"] = np.column_stack([sys_.input_signal(k + 1) for k in range(8)])
        out[p + "dt"] = grid.dt
        out[p + "phi"] = bs.phi_s
        out[p + "temporal"] = bs.temporal_stack()
        out[p + "a_hat"] = srom.a_hat
        out[p + "b_hat"] = srom.b_hat
        out[p + "x0_hat"] = srom.x0_hat
        out[p + "a_blk"] = spacetime.build_st_matrix(srom, bs, grid)
        out[p + "f_blk"] = spacetime.build_st_input(srom, bs, grid, sys_.input_signal)
        out[p + "i_blk"] = spacetime.build_st_init(srom, bs)
        out[p + "a_exp"] = phi_st.T @ (a_st @ phi_st)
        out[p + "f_exp"] = phi_st.T @ f_st
        out[p + "i_exp"] = phi_st.T @ x0_st
        rom = spacetime.build_st_rom(srom, bs, grid, sys_.input_signal)
        out[p + "x_st"] = spacetime.solve_st_rom(rom)
    _save("golden_blocks.npz", **out)


def gen_cfg4_small():
    """cfg4 recipe at 10^3 cells, N_t = 20, n_s = 8, n_t = 4, checked vs explicit Kronecker."""
    d = wl.cfg4_inputs(nx=10, n_s=8, n_t=4, n_steps=20, dt=1e-3)
    grid = system.TimeGrid(d.dt)
    sys_ = system.LinearDynamicalSystem(a=d.a, b=d.b, c=d.c, x0=d.x0, input_signal=d.inputs,
                                        constant_input=True)
    bs = basis.BasisSet(phi_s=d.phi_s, temporal=d.temporal, n_mu=4)
    srom = spatial.build_spatial_rom(sys_, bs, ref_mode="zero")
    rom = spacetime.build_st_rom(srom, bs, grid, sys_.input_signal, True)
    phi_st = spacetime.explicit_st_basis(bs)
    a_st, f_st, x0_st = system.assemble_st(sys_, grid)
    out = dict(a_hat=srom.a_hat, b_hat=srom.b_hat, c_hat=srom.c_hat, x0_hat=srom.x0_hat,
               a_st=rom.a_st_hat, f_st=rom.f_st_hat, x0_st=rom.x0_st_hat,
               x_st=spacetime.solve_st_rom(rom),
               a_exp=phi_st.T @ (a_st @ phi_st), f_exp=phi_st.T @ f_st, i_exp=phi_st.T @ x0_st,
               a_nnz=np.array(d.a.nnz), a_datasum=np.array(d.a.data.sum()),
               phi_sum=np.array(d.phi_s.sum()))
    assert np.max(np.abs(out["a_exp"] - out["a_st"])) <= 1e-11
    _save("golden_cfg4_small.npz", **out)


def gen_cfg4_kron():
    """BASELINE configs[3]'s stated check instance: the cfg4 recipe on a 20^3 grid,
    N_t = 50, n_s = 50, n_t = 20, block-assembled (spacetime.py:43-115) and by the
    explicit Kronecker basis (spacetime.py:189-210, system.py:166-194; the
    verify.py:124-158 protocol).  Phi_st is 400,000 x 1,000 (3.2 GB), so the
    1000 x 1000 operators are stored as checksums plus a seeded sample of entries."""
    d = wl.cfg4_inputs(nx=20, n_s=50, n_t=20, n_steps=50, dt=1e-3)
    grid = system.TimeGrid(d.dt)
    sys_ = system.LinearDynamicalSystem(a=d.a, b=d.b, c=d.c, x0=d.x0, input_signal=d.inputs,
                                        constant_input=True)
    bs = basis.BasisSet(phi_s=d.phi_s, temporal=d.temporal, n_mu=20)
    srom = spatial.build_spatial_rom(sys_, bs, ref_mode="zero")
    rom = spacetime.build_st_rom(srom, bs, grid, sys_.input_signal, True)
    cap = d.a.shape[0] * len(d.dt)  # above the reference's verification cap (20,000 rows); SURVEY 8(d)
    phi_st = spacetime.explicit_st_basis(bs, cap=cap)
    a_st, f_st, x0_st = system.assemble_st(sys_, grid, cap=cap)
    a_exp = phi_st.T @ (a_st @ phi_st)
    f_exp = phi_st.T @ f_st
    i_exp = phi_st.T @ x0_st
    del phi_st
    worst = max(np.max(np.abs(a_exp - rom.a_st_hat)), np.max(np.abs(f_exp - rom.f_st_hat)),
                np.max(np.abs(i_exp - rom.x0_st_hat)))
    print(f"cfg4 Kronecker instance: block vs explicit max-abs {worst:.3e}")
    assert worst <= 1e-11
    rng = np.random.default_rng(11)
    m = a_exp.shape[0]
    idx = rng.choice(m * m, size=20000, replace=False)
    out = dict(a_nnz=np.array(d.a.nnz), a_datasum=np.array(d.a.data.sum()), phi_sum=np.array(d.phi_s.sum()),
               a_hat=srom.a_hat, b_hat=srom.b_hat, x0_hat=srom.x0_hat,
               sample_idx=idx.astype(np.int64),
               a_exp_sample=a_exp.ravel()[idx], a_blk_sample=rom.a_st_hat.ravel()[idx],
               a_exp_diag=np.diag(a_exp).copy(), a_exp_rowsum=a_exp.sum(axis=1), a_exp_colsum=a_exp.sum(axis=0),
               a_exp_fro=np.array(np.linalg.norm(a_exp)), a_blk_fro=np.array(np.linalg.norm(rom.a_st_hat)),
               f_exp=f_exp, i_exp=i_exp, f_blk=rom.f_st_hat, i_blk=rom.x0_st_hat,
               x_st=spacetime.solve_st_rom(rom), worst_blk_vs_exp=np.array(worst))
    _save("golden_cfg4_kron.npz", **out)


def gen_persist():
    """A STROMMAT file written by the reference's persist.write_matrix (persist.py:35-48)."""
    from strom import persist

    m = np.random.default_rng(7).standard_normal((5, 3))
    persist.write_matrix(os.path.join(HERE, "golden_ref_5x3.strommat"), m)
    np.save(os.path.join(HERE, "golden_ref_5x3_values.npy"), m)


def gen_bounds():
    """Space-time inverse applies, residuals and the three a-posteriori bounds
    (bounds.py, system.py:195-275) on small heat1d / random systems."""
    from strom import bounds

    out = {}
    rng = np.random.default_rng(31)
    sys_ = random_stable_system(rng, 10)
    grid = system.TimeGrid(rng.uniform(0.02, 0.08, 6))
    v = rng.standard_normal(60)
    out["inv_a"] = sys_.a.toarray()
    out["inv_b"] = sys_.b.toarray()
    out["inv_dt"] = grid.dt
    out["inv_v"] = v
    out["inv_fwd"] = system.st_apply_inverse(sys_, grid, v)
    out["inv_adj"] = system.st_apply_inverse_adjoint(sys_, grid, v)
    for tag, nx, dt, nt in (("small", 12, 1e-3, 10), ("large", 300, 2e-6, 6)):
        heat = make_heat1d(ProblemSpec(kind="heat1d", nx=nx), {"kappa": 1.0})
        grid = system.TimeGrid.uniform(dt, nt)
        fom = system.fom_march(heat, grid).states
        st = basis.isvd_init(fom[:, 0], tol_svd=0.0)
        st = basis.ingest_simulation(st, fom[:, 1:])
        bs = basis.build_basis_set(st, 3, 1, nt, 1)
        srom = spatial.build_spatial_rom(heat, bs, ref_mode="zero")
        approx = spatial.reconstruct_states(srom, bs, spatial.srom_march(srom, grid, heat.input_signal))
        rom = spacetime.build_st_rom(srom, bs, grid, heat.input_signal, True)
        approx_st = spacetime.reconstruct_states(bs, spacetime.solve_st_rom(rom)).T.ravel()
        out[f"{tag}_approx"] = approx
        out[f"{tag}_approx_st"] = approx_st
        out[f"{tag}_st_res"] = system.st_residual(heat, grid, approx_st)
        for name, rep in (("residual", bounds.residual_error_bound(heat, grid, approx)),
                          ("rom", bounds.rom_error_bound(heat, grid, approx)),
                          ("st", bounds.space_time_error_bound(heat, grid, approx_st))):
            out[f"{tag}_{name}_errors"] = rep.step_errors
            out[f"{tag}_{name}_bounds"] = rep.step_bounds
            out[f"{tag}_{name}_constants"] = rep.constants
            out[f"{tag}_{name}_valid"] = np.array([rep.valid])
    _save("golden_bounds.npz", **out)


if __name__ == "__main__":
    if "--only-kron" in sys.argv:
        gen_cfg4_kron()
        sys.exit(0)
    gen_linalg()
    gen_isvd_small()
    gen_cfg1()
    gen_blocks()
    gen_cfg4_small()
    gen_cfg4_kron()
    gen_persist()
    gen_bounds()
