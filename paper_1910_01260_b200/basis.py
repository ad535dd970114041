"""Streaming incremental SVD and spatial/temporal bases on the B200.

Drop-in mirror of the reference module ``strom.basis`` (pkg/src/strom/basis.py):
same names, signatures, defaults, functional semantics and exception types.
Arrays live on the GPU as float64 torch tensors; every numerical step runs in
the sm_100a kernels of ``libstrom_b200.so`` (no CPU fallback).

Asynchrony: ``isvd_update``/``ingest_simulation`` only enqueue work; reading a
state attribute (``rank``, ``phi``, counters, ...) synchronises the stream.  A
non-finite snapshot poisons the state and the ValueError the reference raises
inside ``thin_svd`` (linalg.py:50-51) is raised when the state is inspected.
"""

from __future__ import annotations

import ctypes as C
import warnings

import numpy as np
import torch

from . import _capi as capi
from ._tensors import F64, colmajor, device, to_dev
from .errors import BasisError

EPS = float(np.finfo(float).eps)

__all__ = [
    "BasisError", "SvdState", "isvd_init", "isvd_update", "ingest_simulation",
    "temporal_snapshots", "BasisSet", "build_basis_set", "batch_pod", "basis_set_from_pod",
]

_CAP_MODES = ("restart", "truncate")


class SvdState:
    """Running thin SVD of every column ingested so far (basis.py:30-62).

    Fields as the reference: ``phi`` (n x r), ``sigma`` (r, non-increasing),
    ``v`` (k x r), ``k``, ``tol_svd``, ``tol_sv``, ``r_max``, ``cap_mode`` and
    the stream counters.  The state is immutable; it owns a handle to the
    device representation phi = U W.
    """

    __slots__ = ("_h", "n", "k", "tol_svd", "tol_sv", "r_max", "cap_mode", "_r_ub", "_info", "_cache",
                 "__weakref__")

    def __init__(self, phi, sigma, v, k, tol_svd, tol_sv=0.0, r_max=None, cap_mode="restart",
                 n_rejected=0, n_dependent=0, n_truncated=0, n_restarts=0):
        if cap_mode not in _CAP_MODES:
            raise ValueError(f"unknown cap_mode {cap_mode!r}")
        phi = to_dev(phi)
        if phi.dim() != 2:
            raise ValueError("phi must be 2-D")
        n, r = phi.shape
        sigma = to_dev(sigma).reshape(-1)
        v = to_dev(v).reshape(int(k), r) if r else None
        cnt = (C.c_int32 * 4)(n_rejected, n_dependent, n_truncated, n_restarts)
        out = C.c_void_p()
        capi.call("strom_isvd_load", n, int(k), r, phi.data_ptr() if r else None,
                  sigma.data_ptr() if r else None, v.data_ptr() if r else None,
                  float(tol_svd), float(tol_sv), -1 if r_max is None else int(r_max),
                  _CAP_MODES.index(cap_mode), cnt, capi.stream_ptr(), C.byref(out))
        self._setup(out.value, n, int(k), tol_svd, tol_sv, r_max, cap_mode, r)

    @classmethod
    def from_factors(cls, u, w, sigma, v, k, tol_svd, tol_sv=0.0, r_max=None, cap_mode="restart",
                     counters=(0, 0, 0, 0), chol=None):
        """State with phi = u @ w given in factored form (u: n x c, w: c x r).

        ``chol`` is the lower Cholesky factor of u^T u; omit it when u has
        orthonormal columns.  Used to resume a stream from an explicit,
        possibly ill-conditioned basis (the lock-step parity harness).
        """
        if cap_mode not in _CAP_MODES:
            raise ValueError(f"unknown cap_mode {cap_mode!r}")
        u = to_dev(u)
        w = to_dev(w)
        n, c = u.shape
        r = w.shape[1]
        ucm, ldu = colmajor(u)
        wcm, ldw = colmajor(w) if r else (w, max(c, 1))
        lcm, ldl = (colmajor(to_dev(chol)) if chol is not None else (None, 0))
        sigma = to_dev(sigma).reshape(-1)
        v = to_dev(v).reshape(int(k), r) if r else None
        cnt = (C.c_int32 * 4)(*[int(x) for x in counters])
        out = C.c_void_p()
        capi.call("strom_isvd_load_factored", n, int(k), c, r, ucm.data_ptr() if c else None, ldu,
                  wcm.data_ptr() if r else None, ldw, None if lcm is None else lcm.data_ptr(), ldl,
                  sigma.data_ptr() if r else None, v.data_ptr() if r else None, float(tol_svd),
                  float(tol_sv), -1 if r_max is None else int(r_max), _CAP_MODES.index(cap_mode), cnt,
                  capi.stream_ptr(), C.byref(out))
        torch.cuda.current_stream().synchronize()
        return cls._wrap(out.value, n, int(k), tol_svd, tol_sv, r_max, cap_mode, r)

    # -- construction from a device handle -------------------------------
    @classmethod
    def _wrap(cls, handle, n, k, tol_svd, tol_sv, r_max, cap_mode, r_ub):
        obj = cls.__new__(cls)
        obj._setup(handle, n, k, tol_svd, tol_sv, r_max, cap_mode, r_ub)
        return obj

    def _setup(self, handle, n, k, tol_svd, tol_sv, r_max, cap_mode, r_ub):
        self._h = handle
        self.n = int(n)
        self.k = int(k)
        self.tol_svd = float(tol_svd)
        self.tol_sv = float(tol_sv)
        self.r_max = r_max
        self.cap_mode = cap_mode
        self._r_ub = int(r_ub)
        self._info = None
        self._cache = {}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                capi.lib.strom_isvd_free(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    # -- device header -----------------------------------------------------
    def info(self) -> capi.IsvdInfo:
        if self._info is None:
            inf = capi.IsvdInfo()
            capi.call("strom_isvd_query", self._h, capi.stream_ptr(), C.byref(inf))
            if inf.status:
                raise ValueError("matrix has non-finite entries (a non-finite snapshot reached the "
                                 "incremental SVD)")
            self._info = inf
            self._r_ub = inf.rank
        return self._info

    @property
    def rank(self) -> int:
        return int(self.info().rank)

    @property
    def n_rejected(self) -> int:
        return int(self.info().n_rejected)

    @property
    def n_dependent(self) -> int:
        return int(self.info().n_dependent)

    @property
    def n_truncated(self) -> int:
        return int(self.info().n_truncated)

    @property
    def n_restarts(self) -> int:
        return int(self.info().n_restarts)

    @property
    def last_flags(self) -> int:
        """Decision bits (STROM_F_*) of the update that produced this state."""
        return int(self.info().flags)

    def _export(self, want: str):
        """Materialise one of the reference's arrays on first use.  phi = U W is a tall GEMM
        and n x r doubles (50 GiB at n = 2^26, r = 100): reading sigma or v must not cost it."""
        if want not in self._cache:
            r = self.rank
            dev = device()
            shape = {"phi": (self.n, r), "sigma": (r,), "v": (self.k, r)}[want]
            if want == "phi":
                capi.lib.strom_trim_cache()  # the spare compaction block must not starve this allocation
            out = torch.empty(shape, dtype=F64, device=dev)
            if r:
                ptr = {k: (out.data_ptr() if k == want else None) for k in ("phi", "sigma", "v")}
                capi.call("strom_isvd_export", self._h, ptr["phi"], ptr["sigma"], ptr["v"], capi.stream_ptr())
            self._cache[want] = out
        return self._cache[want]

    def factors(self):
        """(U, W, L) of the device representation phi = U W, L = chol(U^T U) (diagnostics)."""
        inf = self.info()
        dev = device()
        c, r = inf.ncols_u, inf.rank
        u = torch.empty((c, self.n), dtype=F64, device=dev)
        w = torch.empty((r, c), dtype=F64, device=dev)
        lm = torch.empty((c, c), dtype=F64, device=dev)
        capi.call("strom_isvd_factors", self._h, u.data_ptr() if c else None, w.data_ptr() if c and r else None,
                  lm.data_ptr() if c else None, capi.stream_ptr())
        return u.t(), w.t(), lm.t()

    @property
    def phi(self) -> torch.Tensor:
        return self._export("phi")

    @property
    def sigma(self) -> torch.Tensor:
        return self._export("sigma")

    @property
    def v(self) -> torch.Tensor:
        return self._export("v")

    def __repr__(self):
        return f"SvdState(n={self.n}, k={self.k}, rank={self.rank})"


def _column(x, n=None) -> torch.Tensor:
    x = to_dev(x)
    if n is not None and tuple(x.shape) != (n,):
        raise ValueError(f"expected column of length {n}, got shape {tuple(x.shape)}")
    if x.dim() != 1:
        raise ValueError(f"expected a 1-D column, got shape {tuple(x.shape)}")
    return x


def isvd_init(x, tol_svd: float, k: int = 1, tol_sv: float = 0.0, r_max: int | None = None,
              cap_mode: str = "restart") -> SvdState:
    """Start (or restart) the stream from its k-th column (basis.py:65-102)."""
    if cap_mode not in _CAP_MODES:
        raise ValueError(f"unknown cap_mode {cap_mode!r}")
    x = _column(x)
    out = C.c_void_p()
    capi.call("strom_isvd_init", x.numel(), x.data_ptr(), int(k), float(tol_svd), float(tol_sv),
              -1 if r_max is None else int(r_max), _CAP_MODES.index(cap_mode), capi.stream_ptr(),
              C.byref(out))
    return SvdState._wrap(out.value, x.numel(), int(k), tol_svd, tol_sv, r_max, cap_mode, 1)


def _warn_if_cap_restart(state: SvdState) -> None:
    # basis.py:114-123: the reference warns when the cap forces a restart.
    if state.r_max is not None and state.cap_mode == "restart" and state._r_ub >= state.r_max:
        if state.rank >= state.r_max:
            warnings.warn(
                f"incremental SVD rank hit r_max={state.r_max}; restarting from the incoming column "
                "and discarding the accumulated basis (set cap_mode='truncate' to keep it)",
                RuntimeWarning, stacklevel=3)


def _next_bound(state: SvdState) -> int:
    b = state._r_ub + 1
    return b if state.r_max is None else min(b, max(int(state.r_max), 1))


def isvd_update(state: SvdState, x) -> SvdState:
    """Fold one more column into the running SVD and return the new state (basis.py:105-184)."""
    x = _column(x, state.n)
    _warn_if_cap_restart(state)
    out = C.c_void_p()
    capi.call("strom_isvd_update", state._h, x.data_ptr(), capi.stream_ptr(), C.byref(out))
    return SvdState._wrap(out.value, state.n, state.k + 1, state.tol_svd, state.tol_sv, state.r_max,
                          state.cap_mode, _next_bound(state))


def ingest_simulation(state: SvdState, states) -> SvdState:
    """Fold the columns of one simulation's state matrix, left to right (basis.py:187-194).

    ``states`` may be a CUDA tensor (used in place when its columns are
    contiguous), a host torch tensor or a numpy array (streamed to the device
    in chunks overlapped with the updates).
    """
    on_host = not (isinstance(states, torch.Tensor) and states.is_cuda)
    if on_host:
        if isinstance(states, torch.Tensor):
            st = states.detach().to(F64)
        else:
            st = torch.from_numpy(np.asarray(states, dtype=np.float64))
    else:
        st = states.to(F64)
    if st.dim() != 2:
        raise ValueError("expected a 2-D state matrix")
    if st.shape[0] != state.n:
        raise ValueError(f"expected columns of length {state.n}, got shape {tuple(st.shape)}")
    ncols = st.shape[1]
    if state.cap_mode == "restart" and state.r_max is not None:
        # keep the reference's per-column warning semantics: step one by one
        for j in range(ncols):
            state = isvd_update(state, st[:, j])
        return state
    cm, ld = colmajor(st)
    out = C.c_void_p()
    capi.call("strom_isvd_ingest", state._h, cm.data_ptr(), ld, ncols, 1 if on_host else 0,
              capi.stream_ptr(), C.byref(out))
    rb = state._r_ub + ncols
    if state.r_max is not None:
        rb = min(rb, max(int(state.r_max), 1))
    res = SvdState._wrap(out.value, state.n, state.k + ncols, state.tol_svd, state.tol_sv, state.r_max,
                         state.cap_mode, rb)
    if on_host:
        torch.cuda.current_stream().synchronize()  # host buffer must outlive the async copies
    return res


def temporal_snapshots(v, mode: int, n_steps: int, n_mu: int) -> torch.Tensor:
    """Column p = rows p*N_t:(p+1)*N_t of v[:, mode] (basis.py:215-228); a view."""
    v = to_dev(v)
    if v.shape[0] != n_mu * n_steps:
        raise ValueError(f"right singular matrix has {v.shape[0]} rows, expected {n_mu * n_steps}")
    if not 0 <= mode < v.shape[1]:
        raise IndexError(f"mode {mode} out of range for rank {v.shape[1]}")
    return v[:, mode].reshape(n_mu, n_steps).T


class BasisSet:
    """Spatial basis plus one temporal basis per spatial mode (basis.py:231-272)."""

    __slots__ = ("phi_s", "temporal", "n_mu", "_stack")

    def __init__(self, phi_s, temporal, n_mu):
        # stored column-major (each spatial mode contiguous): the operator build's
        # CSR gather then reads 32 consecutive rows of one mode per load
        self.phi_s = colmajor(to_dev(phi_s, contiguous=False))[0]
        if isinstance(temporal, torch.Tensor) and temporal.dim() == 3:
            stack = to_dev(temporal)
            self.temporal = tuple(stack[i] for i in range(stack.shape[0]))
        else:
            self.temporal = tuple(to_dev(t) for t in temporal)
            stack = None
        self.n_mu = n_mu
        if len(self.temporal) != self.phi_s.shape[1]:
            raise ValueError("need one temporal basis per spatial mode")
        shapes = {tuple(t.shape) for t in self.temporal}
        if len(shapes) > 1:
            raise ValueError(f"temporal bases disagree on shape: {shapes}")
        self._stack = stack

    @property
    def n_s(self) -> int:
        return self.phi_s.shape[1]

    @property
    def n_t(self) -> int:
        return self.temporal[0].shape[1]

    @property
    def n_steps(self) -> int:
        return self.temporal[0].shape[0]

    def temporal_stack(self) -> torch.Tensor:
        """All temporal bases as one (n_s, N_t, n_t) tensor."""
        if self._stack is None:
            self._stack = torch.stack(self.temporal).contiguous()
        return self._stack

    def orthonormality_defect(self) -> float:
        eye_s = torch.eye(self.n_s, dtype=F64, device=self.phi_s.device)
        d = (self.phi_s.T @ self.phi_s - eye_s).abs().max()
        st = self.temporal_stack()
        eye_t = torch.eye(self.n_t, dtype=F64, device=st.device)
        d2 = (st.transpose(1, 2) @ st - eye_t).abs().amax()
        return float(torch.maximum(d, d2))


def build_basis_set(state: SvdState, n_s: int, n_t: int, n_steps: int, n_mu: int) -> BasisSet:
    """Spatial basis and per-mode temporal bases from a final state (basis.py:275-302).

    The n_s temporal SVDs run as one batched device kernel (one CTA per mode).
    """
    if n_s < 1 or n_s > state.rank:
        raise BasisError(f"requested n_s={n_s} but the stream has rank {state.rank}")
    if n_t < 1 or n_t > min(n_steps, n_mu):
        raise BasisError(
            f"requested n_t={n_t} exceeds the temporal ceiling min(N_t={n_steps}, n_mu={n_mu})")
    if state.k != n_mu * n_steps:
        raise BasisError(f"stream saw {state.k} columns, expected n_mu*N_t = {n_mu * n_steps}")
    from .linalg import _temporal_batch

    v_cm = state.v.t().contiguous()  # column-major k x r
    psi, ranks, _ = _temporal_batch(v_cm, state.k, state.rank, n_steps, n_mu, n_s, n_t)
    bad = [i for i in range(n_s) if n_t > int(ranks[i])]
    if bad:
        i = bad[0]
        raise BasisError(
            f"temporal snapshots of mode {i} have rank {int(ranks[i])}, cannot supply n_t={n_t}")
    return BasisSet(phi_s=state.phi[:, :n_s].clone(), temporal=psi, n_mu=n_mu)


def batch_pod(u, n_s: int):
    """One-shot POD of a snapshot matrix (basis.py:197-212): ``(phi_s, sigma, v)``
    with phi_s the leading n_s left singular vectors, by the device thin SVD.
    The oracle the streaming path is checked against."""
    from . import linalg

    u = to_dev(u)
    if n_s < 1:
        raise BasisError(f"need n_s >= 1, got {n_s}")
    w, sigma, v = linalg.thin_svd(u)
    smax = float(sigma[0]) if sigma.numel() else 0.0
    rank = int((sigma > max(u.shape) * EPS * smax).sum())
    if n_s > rank:
        raise BasisError(f"requested {n_s} modes but the snapshots have rank {rank}")
    return w[:, :n_s], sigma, v


def basis_set_from_pod(u, n_s: int, n_t: int, n_steps: int, n_mu: int) -> BasisSet:
    """Batch-POD twin of :func:`build_basis_set` (basis.py:305-315)."""
    from . import linalg

    phi_s, _, v = batch_pod(u, n_s)
    temporal = []
    for i in range(n_s):
        w_i, _, _ = linalg.thin_svd(temporal_snapshots(v, i, n_steps, n_mu))
        temporal.append(w_i[:, :n_t])
    return BasisSet(phi_s=phi_s, temporal=tuple(temporal), n_mu=n_mu)
