"""NumPy model of the DEVICE incremental-SVD algorithm (test infrastructure).

Mirrors csrc/isvd_kernels.cuh step for step -- append-only U, small-space W,
Cholesky factor L of G = U^T U, folding of in-span residuals, drift test via
L^T w, small-space QR of L^T W, host-scheduled compaction -- so the
representation's numerics can be studied on the CPU.  Not bit-identical to the
kernels (different reduction orders, LAPACK core SVD instead of Jacobi).
"""

from __future__ import annotations

import numpy as np

from oracle import strom_oracle as so

EPS = np.finfo(float).eps
FOLD_TAU = 1e-3


class LocalSums:
    """Sums over rows, all rows in this process (the unsharded device)."""

    def total(self, partial):
        return partial


class BlockSums:
    """Sums over rows as the row-sharded device forms them (csrc/shard.cuh): a
    partial per row block, exchanged, added in BLOCK (rank) order on every rank.
    `exchange(partial) -> list of every rank's partial in rank order`."""

    def __init__(self, exchange):
        self.exchange = exchange

    def total(self, partial):
        parts = self.exchange(np.asarray(partial, dtype=float))
        out = np.zeros_like(parts[0])
        for q in parts:  # rank order: identical bits on every rank
            out = out + q
        return out


class DevState:
    """n is the matrix's (global) row count; U holds this process's rows."""

    def __init__(self, n, tol_svd, tol_sv=0.0, r_max=None, ccap=None, sums=None):
        self.n = n
        self.sums = sums or LocalSums()
        self.U = np.zeros((n, 0))
        self.W = np.zeros((0, 0))
        self.L = np.zeros((0, 0))
        self.sigma = np.zeros(0)
        self.V = np.zeros((0, 0))
        self.k = 0
        self.tol_svd, self.tol_sv, self.r_max = tol_svd, tol_sv, r_max
        self.ccap = ccap
        self.flags = {}

    @property
    def r(self):
        return self.sigma.size

    @property
    def phi(self):
        return self.U @ self.W


def init(x, tol_svd, k=1, n=None, **kw):
    s = DevState(x.size if n is None else n, tol_svd, **kw)
    s.k = k
    xx = float(s.sums.total(x @ x))
    nrm = np.sqrt(xx)
    if nrm > tol_svd:
        s.U = x[:, None].copy()
        s.W = np.array([[1.0 / nrm]])
        s.L = np.array([[np.sqrt(xx)]])
        s.sigma = np.array([nrm])
        s.V = np.zeros((k, 1))
        s.V[k - 1, 0] = 1.0
    else:
        s.V = np.zeros((k, 0))
    return s


def compact(s):
    c, r = s.W.shape
    if r == 0:
        s.U = np.zeros((s.U.shape[0], 0)); s.W = np.zeros((0, 0)); s.L = np.zeros((0, 0))
        return
    m = s.L.T @ s.W
    q, rr = np.linalg.qr(m)
    t = np.linalg.solve(s.L.T, q)
    s.U = s.U @ t
    s.W = rr
    # the device measures the Gram of the stored U_new (one more exchange when sharded)
    s.L = np.linalg.cholesky(s.sums.total(s.U.T @ s.U))


def update(s, x):
    r, c = s.r, s.U.shape[1]
    k = s.k + 1
    if s.ccap is not None and c + 1 > s.ccap:
        compact(s)
        c = s.U.shape[1]
    if r == 0:
        t = init(x, s.tol_svd, k, n=s.n, tol_sv=s.tol_sv, r_max=s.r_max, ccap=s.ccap, sums=s.sums)
        return t
    # one exchange per pass: [U^T x | x.x], then [U^T r | r.r] (the k_pass partial layout)
    gx = s.sums.total(np.concatenate([s.U.T @ x, [x @ x]]))
    g, xx = gx[:-1], gx[-1]
    ell = s.W.T @ g
    p_sq = xx - ell @ ell
    p = np.sqrt(p_sq) if p_sq > 0 else 0.0
    dep = p < s.tol_svd or p == 0.0 or r >= s.n
    y = s.W @ ell
    cn = c
    Ln = s.L.copy()
    h = np.zeros(c)
    if not dep:
        gt = np.linalg.solve(s.L.T, np.linalg.solve(s.L, g))
        r1 = x - s.U @ gt
        er = s.sums.total(np.concatenate([s.U.T @ r1, [r1 @ r1]]))
        e, rho2 = er[:-1], er[-1]
        lv = np.linalg.solve(s.L, e) if c else np.zeros(0)
        lam2 = rho2 - lv @ lv
        app = lam2 > FOLD_TAU ** 2 * rho2 and rho2 > 0
        if not app and c < s.n:
            # DGKS: second classical Gram-Schmidt pass on r1 (in place)
            h = np.linalg.solve(s.L.T, lv)
            r1 = r1 - s.U @ h
            er = s.sums.total(np.concatenate([s.U.T @ r1, [r1 @ r1]]))
            e, rho2 = er[:-1], er[-1]
            lv = np.linalg.solve(s.L, e) if c else np.zeros(0)
            lam2 = rho2 - lv @ lv
            app = lam2 > 0.25 * rho2 and rho2 > 0
        if app:
            cn = c + 1
            Ln = np.zeros((cn, cn))
            Ln[:c, :c] = s.L
            Ln[c, :c] = lv
            Ln[c, c] = np.sqrt(lam2)
            wj = np.concatenate([(gt + h - y) / p, [1.0 / p]])
            Un = np.hstack([s.U, r1[:, None]])
        elif c >= r + 1:
            wj = (gt + h - y + np.linalg.solve(s.L.T, lv)) / p
            Un = s.U
        else:
            dep = True  # x lies in span(U) to working precision and U has no spare direction
            Un = s.U
    else:
        Un = s.U
    q = np.zeros((r + 1, r + 1))
    q[:r, :r] = np.diag(s.sigma)
    q[:r, r] = ell
    q[r, r] = 0.0 if dep else p
    wb, sb, vb = so.thin_svd(q)
    vbord = np.zeros((k, r + 1))
    vbord[: k - 1, :r] = s.V
    vbord[k - 1, r] = 1.0
    if dep:
        W = s.W @ wb[:r, :r]
        sig = sb[:r]
        V = vbord @ vb[:, :r]
    else:
        Wb = np.zeros((cn, r + 1))
        Wb[:c, :r] = s.W
        Wb[:, r] = wj
        W = Wb @ wb
        sig = sb
        V = vbord @ vb
    trunc = False
    if sig.size and sig[-1] < s.tol_sv:
        W, sig, V = W[:, :-1], sig[:-1], V[:, :-1]
        trunc = True
    if s.r_max is not None and sig.size > s.r_max:
        W, sig, V = W[:, : s.r_max], sig[: s.r_max], V[:, : s.r_max]
        trunc = True
    did_qr = False
    drift = 0.0
    if sig.size > 1:
        a0 = Ln.T @ W[:, 0]
        a1 = Ln.T @ W[:, -1]
        drift = abs(a0 @ a1)
        if drift > min(s.tol_svd, EPS * s.n):
            m = Ln.T @ W
            qs, rs = np.linalg.qr(m)
            d = np.sign(np.diag(rs)); d[d == 0] = 1
            qs = qs * d
            W = np.linalg.solve(Ln.T, qs)
            did_qr = True
    t = DevState(s.n, s.tol_svd, s.tol_sv, s.r_max, s.ccap, s.sums)
    t.U, t.W, t.L, t.sigma, t.V, t.k = Un, W, Ln, sig, V, k
    t.flags = dict(dep=dep, trunc=trunc, qr=did_qr, drift=drift, p=p, appended=cn > c)
    return t


def stream(cols, tol, **kw):
    s = init(cols[:, 0], tol, **kw)
    for j in range(1, cols.shape[1]):
        s = update(s, cols[:, j])
    return s
