"""CPU oracle for the strom hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy/scipy, the reference algorithm of the
three north-star subsystems so that the CUDA product path can be checked
against it:

  * streaming incremental SVD       reference pkg/src/strom/basis.py:65-194
  * per-mode temporal bases         reference pkg/src/strom/basis.py:215-302
  * spatial + space-time operators  reference pkg/src/strom/spatial.py:45-67,
                                    pkg/src/strom/spacetime.py:37-162
  * dense kernels they lean on      reference pkg/src/strom/linalg.py:31-99

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this file, and only as
the checker (or the timed CPU baseline) -- never as the thing shipped.  The
product package ``paper_1910_01260_b200`` never imports it and has no CPU
fallback.

Parity pin: every function here is checked against golden vectors produced by
running the *real* reference (``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src/strom``) -- see ``tests/test_oracle_golden.py``.
The restatement performs the same numpy operations in the same order, so on
the same numpy/OpenBLAS build it is bit-identical to the reference.

The arithmetic lives in NumPy/SciPy (LAPACK gesdd/geqrf/getrf via OpenBLAS,
SciPy sparsetools, SuperLU); the reference pins only lower bounds
(pkg/pyproject.toml:10-14).  Versions in this image: numpy 2.3.5, scipy 1.18.1.

Beyond the reference, ``update`` returns a decision record (dependent /
truncated / qr / restart flags, the Pythagorean p and the drift value) used by
the lock-step parity harness.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, field, replace

import numpy as np
import scipy.linalg
import scipy.sparse as sp
import scipy.sparse.linalg as spla

EPS = np.finfo(float).eps


class OracleBasisError(Exception):
    """Mirror of strom.basis.BasisError (basis.py:26-27)."""


class OracleSingularMatrixError(Exception):
    """Mirror of strom.linalg.SingularMatrixError (linalg.py:19-20)."""


# --------------------------------------------------------------------------
# dense kernels (reference linalg.py)
# --------------------------------------------------------------------------

def sign_fix(w: np.ndarray, v: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Column j of w gets its largest-|.| entry (first on ties) made >= 0; v follows.

    Restates linalg._fix_svd_signs (linalg.py:31-38).
    """
    for col in range(w.shape[1]):
        at = int(np.argmax(np.abs(w[:, col])))
        if w[at, col] < 0.0:
            w[:, col] *= -1.0
            v[:, col] *= -1.0
    return w, v


def thin_svd(m: np.ndarray) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """gesdd thin SVD, descending sigma, deterministic signs (linalg.py:41-57)."""
    m = np.asarray(m, dtype=float)
    if m.ndim != 2 or min(m.shape) < 1:
        raise ValueError(f"need a non-empty 2-D matrix, got shape {m.shape}")
    if not np.all(np.isfinite(m)):
        raise ValueError("matrix has non-finite entries")
    w, s, vt = np.linalg.svd(m, full_matrices=False)
    w, v = sign_fix(w, vt.T.copy())
    return w, s, v


def qr_pos(m: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Reduced QR with diag(R) >= 0, zero diagonal -> +1 (linalg.py:60-72)."""
    m = np.asarray(m, dtype=float)
    if m.ndim != 2 or m.shape[0] < m.shape[1]:
        raise ValueError(f"need rows >= cols, got shape {m.shape}")
    q, r = np.linalg.qr(m, mode="reduced")
    d = np.sign(np.diag(r))
    d[d == 0.0] = 1.0
    return q * d, d[:, None] * r


def solve_dense(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """LU with partial pivoting + pivot floor 1e-14*||A||_F (linalg.py:75-99)."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError(f"matrix must be square, got shape {a.shape}")
    if b.shape[0] != a.shape[0]:
        raise ValueError(f"dimension mismatch: {a.shape} vs {b.shape}")
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", scipy.linalg.LinAlgWarning)
        lu, piv = scipy.linalg.lu_factor(a)
    piv_abs = np.abs(np.diag(lu))
    floor = 1e-14 * np.linalg.norm(a)
    bad = np.nonzero(piv_abs <= floor)[0]
    if bad.size:
        raise OracleSingularMatrixError(
            f"matrix numerically singular: pivot {bad[0]} is "
            f"{piv_abs[bad[0]]:.3e} (floor {floor:.3e})"
        )
    return scipy.linalg.lu_solve((lu, piv), b)


# --------------------------------------------------------------------------
# incremental SVD (reference basis.py:30-194, PAPER.md Algorithms 1-2)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class OState:
    """Frozen running-SVD state; field meaning as strom.basis.SvdState (basis.py:30-62)."""

    phi: np.ndarray
    sigma: np.ndarray
    v: np.ndarray
    k: int
    tol_svd: float
    tol_sv: float = 0.0
    r_max: int | None = None
    cap_mode: str = "restart"
    n_rejected: int = 0
    n_dependent: int = 0
    n_truncated: int = 0
    n_restarts: int = 0

    @property
    def rank(self) -> int:
        return int(self.sigma.size)


@dataclass
class Decision:
    """What one update decided -- used by the lock-step harness."""

    restart: bool = False
    rejected: bool = False
    dependent: bool = False
    truncated: bool = False
    qr: bool = False
    p: float = 0.0
    p_sq: float = 0.0
    xnorm: float = 0.0
    drift: float = 0.0
    sigma_bar: np.ndarray = field(default_factory=lambda: np.empty(0))


def init(x, tol_svd, k=1, tol_sv=0.0, r_max=None, cap_mode="restart") -> OState:
    """Algorithm 1 (basis.py:65-102): accept iff ||x|| > tol_svd (strict)."""
    if cap_mode not in ("restart", "truncate"):
        raise ValueError(f"unknown cap_mode {cap_mode!r}")
    x = np.asarray(x, dtype=float)
    nrm = float(np.linalg.norm(x))
    if nrm > tol_svd:
        v = np.zeros((k, 1))
        v[k - 1, 0] = 1.0
        return OState((x / nrm)[:, None], np.array([nrm]), v, k, float(tol_svd),
                      float(tol_sv), r_max, cap_mode)
    return OState(np.empty((x.size, 0)), np.empty(0), np.empty((k, 0)), k,
                  float(tol_svd), float(tol_sv), r_max, cap_mode, n_rejected=1)


def update(st: OState, x, log: Decision | None = None) -> OState:
    """Algorithm 2 (basis.py:105-184) with an optional decision record."""
    x = np.asarray(x, dtype=float)
    n = st.phi.shape[0] if st.rank else x.size
    if x.shape != (n,):
        raise ValueError(f"expected column of length {n}, got shape {x.shape}")
    log = log if log is not None else Decision()
    r = st.rank
    k = st.k + 1
    capped = st.r_max is not None and r >= st.r_max
    # restart / first-accept branch (basis.py:115-133)
    if r == 0 or (capped and st.cap_mode == "restart"):
        if capped:
            warnings.warn(f"incremental SVD rank hit r_max={st.r_max}; restarting",
                          RuntimeWarning, stacklevel=2)
        fresh = init(x, st.tol_svd, k, st.tol_sv, st.r_max, st.cap_mode)
        log.restart = bool(capped)
        log.rejected = fresh.rank == 0
        return replace(fresh, n_rejected=st.n_rejected + fresh.n_rejected,
                       n_dependent=st.n_dependent, n_truncated=st.n_truncated,
                       n_restarts=st.n_restarts + (1 if capped else 0))
    # projection and Pythagorean residual norm (basis.py:135-139)
    ell = st.phi.T @ x
    p_sq = float(x @ x - ell @ ell)
    p = np.sqrt(p_sq) if p_sq > 0.0 else 0.0
    dep = p < st.tol_svd or p == 0.0 or r >= n
    log.p, log.p_sq, log.dependent = float(p), p_sq, bool(dep)
    log.xnorm = float(np.sqrt(x @ x))
    # bordered core and its SVD (basis.py:141-145)
    core = np.zeros((r + 1, r + 1))
    core[:r, :r] = np.diag(st.sigma)
    core[:r, r] = ell
    core[r, r] = 0.0 if dep else p
    wb, sb, vb = thin_svd(core)
    log.sigma_bar = sb.copy()
    vbord = np.zeros((k, r + 1))
    vbord[: k - 1, :r] = st.v
    vbord[k - 1, r] = 1.0
    # rotation (basis.py:150-158)
    if dep:
        phi = st.phi @ wb[:r, :r]
        sig = sb[:r]
        v = vbord @ vb[:, :r]
    else:
        j = (x - st.phi @ ell) / p
        phi = np.hstack([st.phi, j[:, None]]) @ wb
        sig = sb
        v = vbord @ vb
    # truncation (basis.py:160-168)
    trunc = 0
    if sig.size and sig[-1] < st.tol_sv:
        phi, sig, v = phi[:, :-1], sig[:-1], v[:, :-1]
        trunc = 1
    if st.r_max is not None and sig.size > st.r_max:
        phi, sig, v = phi[:, : st.r_max], sig[: st.r_max], v[:, : st.r_max]
        trunc = 1
    log.truncated = bool(trunc)
    # drift-triggered re-orthogonalisation (basis.py:170-174)
    if sig.size:
        drift = abs(float(phi[:, 0] @ phi[:, -1])) if sig.size > 1 else 0.0
        log.drift = drift
        if drift > min(st.tol_svd, EPS * n):
            phi, _ = qr_pos(phi)
            log.qr = True
    return replace(st, phi=phi, sigma=sig, v=v, k=k,
                   n_dependent=st.n_dependent + (1 if dep else 0),
                   n_truncated=st.n_truncated + trunc)


def ingest(st: OState, cols, logs: list | None = None) -> OState:
    """Fold columns left to right (basis.py:187-194)."""
    cols = np.asarray(cols, dtype=float)
    if cols.ndim != 2:
        raise ValueError("expected a 2-D state matrix")
    for c in range(cols.shape[1]):
        d = Decision()
        st = update(st, cols[:, c], d)
        if logs is not None:
            logs.append(d)
    return st


def stream(cols, tol_svd, tol_sv=0.0, r_max=None, cap_mode="restart", logs=None):
    """pipeline.train ingestion order (pipeline.py:98-111): init on col 0, update on the rest."""
    cols = np.asarray(cols, dtype=float)
    st = init(cols[:, 0], tol_svd, tol_sv=tol_sv, r_max=r_max, cap_mode=cap_mode)
    return ingest(st, cols[:, 1:], logs)


def batch_pod(u, n_s):
    """Batch POD oracle (basis.py:197-212)."""
    u = np.asarray(u, dtype=float)
    if n_s < 1:
        raise OracleBasisError(f"need n_s >= 1, got {n_s}")
    w, s, v = thin_svd(u)
    lead = s[0] if s.size else 0.0
    rank = int(np.sum(s > max(u.shape) * EPS * lead))
    if n_s > rank:
        raise OracleBasisError(f"requested {n_s} modes but the snapshots have rank {rank}")
    return w[:, :n_s], s, v


# --------------------------------------------------------------------------
# temporal bases (reference basis.py:215-302)
# --------------------------------------------------------------------------

def temporal_snapshots(v, mode, n_steps, n_mu):
    """T_i = v[:, mode] reshaped (n_mu, N_t) and transposed (basis.py:215-228)."""
    v = np.asarray(v, dtype=float)
    if v.shape[0] != n_mu * n_steps:
        raise ValueError(f"right singular matrix has {v.shape[0]} rows, expected {n_mu * n_steps}")
    if not 0 <= mode < v.shape[1]:
        raise IndexError(f"mode {mode} out of range for rank {v.shape[1]}")
    return v[:, mode].reshape(n_mu, n_steps).T


def basis_set(st: OState, n_s, n_t, n_steps, n_mu):
    """build_basis_set (basis.py:275-302) -> (phi_s, temporal tuple, temporal ranks)."""
    if n_s < 1 or n_s > st.rank:
        raise OracleBasisError(f"requested n_s={n_s} but the stream has rank {st.rank}")
    if n_t < 1 or n_t > min(n_steps, n_mu):
        raise OracleBasisError(
            f"requested n_t={n_t} exceeds the temporal ceiling min(N_t={n_steps}, n_mu={n_mu})")
    if st.v.shape[0] != n_mu * n_steps:
        raise OracleBasisError(
            f"stream saw {st.v.shape[0]} columns, expected n_mu*N_t = {n_mu * n_steps}")
    temporal, ranks = [], []
    for i in range(n_s):
        t_i = temporal_snapshots(st.v, i, n_steps, n_mu)
        w_i, s_i, _ = thin_svd(t_i)
        rk = int(np.sum(s_i > max(t_i.shape) * EPS * s_i[0]))
        ranks.append(rk)
        if n_t > rk:
            raise OracleBasisError(
                f"temporal snapshots of mode {i} have rank {rk}, cannot supply n_t={n_t}")
        temporal.append(w_i[:, :n_t])
    return st.phi[:, :n_s].copy(), tuple(temporal), ranks


# --------------------------------------------------------------------------
# spatial ROM (reference spatial.py:45-67)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class OSpatial:
    a_hat: np.ndarray
    b_hat: np.ndarray
    c_hat: np.ndarray
    x_ref: np.ndarray
    x_ref_hat: np.ndarray
    x0_hat: np.ndarray
    y_ref: np.ndarray
    ref_mode: str


def spatial_rom(a, b, c, x0, phi, ref_mode="initial_state") -> OSpatial:
    """Galerkin projection of (A, B, C, x0) onto phi (spatial.py:45-67)."""
    if ref_mode not in ("zero", "initial_state"):
        raise ValueError(f"ref_mode must be one of ('zero', 'initial_state'), got {ref_mode!r}")
    a = sp.csr_array(a)
    b = sp.csr_array(b)
    c = np.atleast_2d(np.asarray(c, dtype=float))
    x0 = np.asarray(x0, dtype=float)
    if phi.shape[0] != a.shape[0]:
        raise ValueError(f"basis has {phi.shape[0]} rows but the system has {a.shape[0]} states")
    x_ref = x0 if ref_mode == "initial_state" else np.zeros(a.shape[0])
    a_phi = a @ phi
    return OSpatial(
        a_hat=phi.T @ a_phi,
        b_hat=phi.T @ b.toarray(),
        c_hat=phi.T @ c,
        x_ref=x_ref,
        x_ref_hat=phi.T @ (a @ x_ref),
        x0_hat=phi.T @ (x0 - x_ref),
        y_ref=c.T @ x_ref,
        ref_mode=ref_mode,
    )


# --------------------------------------------------------------------------
# space-time block assembly (reference spacetime.py:37-162)
# --------------------------------------------------------------------------

def step_factors(temporal) -> np.ndarray:
    """F[j] (N_t x n_s), F[j][k, i] = Psi_i[k, j] (spacetime.py:37-40)."""
    return np.transpose(np.stack(temporal), (2, 1, 0))


def st_matrix(a_hat, temporal, dt) -> np.ndarray:
    """Block (j', j) = -(F_j'^T diag(dt) F_j) o A_hat + diag(same - coupling) (spacetime.py:43-69)."""
    dt = np.asarray(dt, dtype=float)
    f = step_factors(temporal)
    n_t, n_steps, n_s = f.shape
    if n_steps != dt.size:
        raise ValueError(f"basis covers {n_steps} steps but the grid has {dt.size}")
    out = np.empty((n_s * n_t, n_s * n_t))
    for jp in range(n_t):
        fp = f[jp]
        for j in range(n_t):
            fj = f[j]
            same = np.einsum("ki,ki->i", fp, fj)
            coup = np.einsum("ki,ki->i", fp[1:], fj[:-1])
            blk = -(fp.T @ (dt[:, None] * fj)) * a_hat
            blk[np.diag_indices(n_s)] += same - coup
            out[jp * n_s:(jp + 1) * n_s, j * n_s:(j + 1) * n_s] = blk
    return out


def st_input(b_hat, temporal, dt, inputs, constant_input=False) -> np.ndarray:
    """Block j = sum_k dt_k E_k^(j) (B_hat f_k) (spacetime.py:72-99)."""
    dt = np.asarray(dt, dtype=float)
    f = step_factors(temporal)
    n_t, n_steps, n_s = f.shape
    out = np.empty(n_s * n_t)
    if constant_input:
        bf = b_hat @ np.atleast_1d(inputs(1))
        for j in range(n_t):
            out[j * n_s:(j + 1) * n_s] = (dt[:, None] * f[j]).sum(axis=0) * bf
    else:
        g = np.column_stack([b_hat @ np.atleast_1d(inputs(k + 1)) for k in range(n_steps)]).T
        for j in range(n_t):
            out[j * n_s:(j + 1) * n_s] = (dt[:, None] * f[j] * g).sum(axis=0)
    return out


def st_init(x0_hat, temporal) -> np.ndarray:
    """Every block j = E_1^(j) x0_hat -- the code, not the paper (spacetime.py:102-115)."""
    f = step_factors(temporal)
    n_t, _, n_s = f.shape
    out = np.empty(n_s * n_t)
    for j in range(n_t):
        out[j * n_s:(j + 1) * n_s] = f[j, 0, :] * x0_hat
    return out


def st_solve(a_st, f_st, x0_st) -> np.ndarray:
    """solve_st_rom (spacetime.py:154-162)."""
    return solve_dense(a_st, f_st + x0_st)


def st_reconstruct(phi_s, temporal, x_hat_st) -> np.ndarray:
    """Lift the ST solution to N_s x N_t (spacetime.py:180-186)."""
    f = step_factors(temporal)
    n_t, _, n_s = f.shape
    blocks = np.asarray(x_hat_st).reshape(n_t, n_s)
    return phi_s @ np.einsum("jki,ji->ik", f, blocks)


def explicit_st_basis(phi_s, temporal) -> np.ndarray:
    """Kronecker columns psi_i^j (x) phi_i, column i + n_s j (spacetime.py:189-210)."""
    n_s = phi_s.shape[1]
    n_t = temporal[0].shape[1]
    cols = [np.kron(temporal[i][:, j][:, None], phi_s[:, i][:, None]).ravel()
            for j in range(n_t) for i in range(n_s)]
    return np.column_stack(cols)


def assemble_st(a, b, x0, dt, inputs):
    """Explicit block-bidiagonal space-time system (system.py:166-194)."""
    a = sp.csr_array(a)
    b = sp.csr_array(b)
    n, nt = a.shape[0], len(dt)
    eye = sp.eye_array(n, format="csr")
    blocks = [[None] * nt for _ in range(nt)]
    for k in range(nt):
        blocks[k][k] = eye - dt[k] * a
        if k > 0:
            blocks[k][k - 1] = -eye
    a_st = sp.csr_array(sp.bmat(blocks, format="csr"))
    f_st = np.concatenate([dt[k] * (b @ np.atleast_1d(inputs(k + 1))) for k in range(nt)])
    x0_st = np.zeros(n * nt)
    x0_st[:n] = x0
    return a_st, f_st, x0_st


# --------------------------------------------------------------------------
# full-order snapshot producer (reference system.py:106-163) -- input generation
# --------------------------------------------------------------------------

def fom_march(a, b, x0, dt, inputs) -> np.ndarray:
    """Backward Euler with one SuperLU factor per distinct dt (system.py:106-163)."""
    a = sp.csr_array(a)
    b = sp.csr_array(b)
    n, nt = a.shape[0], len(dt)
    eye = sp.eye_array(n, format="csc")
    facs = {}
    out = np.empty((n, nt))
    fs = [np.atleast_1d(inputs(k)) for k in range(1, nt + 1)]
    x = np.asarray(x0, dtype=float)
    for k in range(nt):
        h = float(dt[k])
        lu = facs.get(h)
        if lu is None:
            lu = spla.splu(sp.csc_array(eye - h * a))
            facs[h] = lu
        x = lu.solve(x + dt[k] * (b @ fs[k]))
        out[:, k] = x
    return out
