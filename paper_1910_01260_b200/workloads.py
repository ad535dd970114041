"""Seeded synthetic inputs for the BASELINE.json configurations.

The paper's ARDRA transport runs are not available; BASELINE.json defines
synthetic stand-ins and these generators build them deterministically (numpy
``default_rng`` seeds, draw order as SURVEY.md section 8(d) lists).  Nothing
here is on the timed path: they produce the snapshot streams, sparse operators
and bases that the device kernels consume.

* cfg1 -- 1D periodic upwind advection + central diffusion, N = 1024 cells.
* cfg2 -- low-rank-plus-noise stream X = Q diag(sigma) W^T + E, n_s = 2^20.
* cfg4 -- 3D 7-point advection-diffusion on a 100^3 grid with random
  per-cell diffusivity, plus a Haar spatial basis and Haar temporal blocks.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp


def haar(rng: np.random.Generator, rows: int, cols: int) -> np.ndarray:
    """Haar-random orthonormal columns: Q of QR(Gaussian) with diag(R) >= 0.

    Same recipe as the reference's ``verify._random_orthonormal``
    (pkg/src/strom/verify.py:52-54 -> linalg.qr, linalg.py:60-72).
    """
    q, r = np.linalg.qr(rng.standard_normal((rows, cols)), mode="reduced")
    d = np.sign(np.diag(r))
    d[d == 0.0] = 1.0
    return q * d


# --------------------------------------------------------------------------
# cfg1: periodic advection-diffusion (BASELINE.json configs[0])
# --------------------------------------------------------------------------

CFG1_N = 1024
CFG1_TRAIN_NU = (0.01, 0.02, 0.03, 0.04)
CFG1_TEST_NU = 0.025
CFG1_DT = 1e-3
CFG1_NT = 100
CFG1_TOL = 1e-8
CFG1_NS = 10
CFG1_NTMODES = 4  # n_t = 5 is infeasible with 4 training nu (SURVEY Finding 3)


@dataclass
class LinearSystemData:
    """Plain operator data of one parameter instance: x' = A x + B f, y = C^T x."""

    a: sp.csr_array
    b: sp.csr_array
    c: np.ndarray
    x0: np.ndarray
    f_const: np.ndarray  # constant input vector

    def inputs(self, k: int) -> np.ndarray:
        return self.f_const


def cfg1_system(nu: float, n: int = CFG1_N, speed: float = 1.0) -> LinearSystemData:
    """A = -c D1_upwind + nu D2_central on a periodic grid, x_i = (i + 1/2)/n.

    B = 0 (one input column), f = 0, x0 = Gaussian bump at 0.3 (width 0.05),
    output C = cell mean.
    """
    dx = 1.0 / n
    idx = np.arange(n)
    left = (idx - 1) % n
    right = (idx + 1) % n
    diag = np.full(n, -speed / dx - 2.0 * nu / dx**2)
    lo = np.full(n, speed / dx + nu / dx**2)
    hi = np.full(n, nu / dx**2)
    rows = np.concatenate([idx, idx, idx])
    cols = np.concatenate([idx, left, right])
    vals = np.concatenate([diag, lo, hi])
    a = sp.csr_array((vals, (rows, cols)), shape=(n, n))
    a.sum_duplicates()
    a.sort_indices()
    x = (idx + 0.5) * dx
    x0 = np.exp(-(((x - 0.3) / 0.05) ** 2))
    b = sp.csr_array((n, 1))
    c = np.full((n, 1), 1.0 / n)
    return LinearSystemData(a=a, b=b, c=c, x0=x0, f_const=np.zeros(1))


def cfg1_dt() -> np.ndarray:
    return np.full(CFG1_NT, CFG1_DT)


# --------------------------------------------------------------------------
# cfg2: synthetic low-rank stream (BASELINE.json configs[1])
# --------------------------------------------------------------------------

CFG2_N = 1 << 20
CFG2_COLS = 500
CFG2_RANK = 64
CFG2_TOL = 1e-9
CFG2_RMAX = 64


def cfg2_sigma(rank: int = CFG2_RANK, decades_per: float = 8.0) -> np.ndarray:
    return 10.0 ** (-np.arange(rank) / decades_per)


def cfg2_stream_numpy(n: int = CFG2_N, cols: int = CFG2_COLS, rank: int = CFG2_RANK,
                      seed: int = 0, noise: float = 1e-12, decades_per: float = 8.0):
    """X = Q diag(sigma) W^T + noise * N(0,1); draw order Q, W, E.

    Returns (X (n x cols, Fortran order so columns are contiguous), Q, W, sigma).
    """
    rng = np.random.default_rng(seed)
    q = haar(rng, n, rank)
    w = haar(rng, cols, rank)
    s = cfg2_sigma(rank, decades_per)
    e = rng.standard_normal((n, cols))
    x = np.asfortranarray((q * s) @ w.T + noise * e)
    return x, q, w, s


def cfg2_stream_torch(n: int = CFG2_N, cols: int = CFG2_COLS, rank: int = CFG2_RANK,
                      seed: int = 0, noise: float = 1e-12, decades_per: float = 8.0,
                      device: str = "cuda"):
    """Device-side generator of the same construction (torch RNG, for the bench).

    Statistically identical to :func:`cfg2_stream_numpy` (different draws).
    Returns X as a (cols, n) contiguous tensor, i.e. column t is X[t].
    """
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)

    def _haar(rows, c):
        a = torch.randn(rows, c, generator=g, device=device, dtype=torch.float64)
        q, r = torch.linalg.qr(a, mode="reduced")
        d = torch.sign(torch.diagonal(r))
        d[d == 0] = 1.0
        return q * d

    q = _haar(n, rank)
    w = _haar(cols, rank)
    s = torch.tensor(cfg2_sigma(rank, decades_per), device=device, dtype=torch.float64)
    xt = (w * s) @ q.T  # (cols, n)
    xt += noise * torch.randn(cols, n, generator=g, device=device, dtype=torch.float64)
    return xt, q, w, s


# --------------------------------------------------------------------------
# cfg4: 3D 7-point advection-diffusion operator build (BASELINE.json configs[3])
# --------------------------------------------------------------------------

CFG4_NX = 100
CFG4_NS = 50
CFG4_NT_MODES = 20
CFG4_NSTEPS = 500
CFG4_DT = 1e-3
CFG4_VELOCITY = (1.0, 0.5, 0.25)


def cfg4_operator(nx: int = CFG4_NX, seed: int = 1,
                  velocity=CFG4_VELOCITY) -> sp.csr_array:
    """7-point operator on nx^3 interior cells of the unit cube, h = 1/(nx+1).

    (A u)_i = kappa_i sum_nb (u_nb - u_i)/h^2 - sum_d v_d (u_i - u_{i-e_d})/h,
    kappa_i ~ U[0.5, 1.5] per cell (seed), Dirichlet-zero (missing neighbours
    drop out), x fastest.  int32 indices; nnz = 7 nx^3 - 6 nx^2.
    """
    rng = np.random.default_rng(seed)
    n = nx ** 3
    h = 1.0 / (nx + 1)
    kappa = rng.uniform(0.5, 1.5, n)
    vx, vy, vz = velocity
    idx = np.arange(n)
    ix = idx % nx
    iy = (idx // nx) % nx
    iz = idx // (nx * nx)
    diag = -6.0 * kappa / h**2 - (vx + vy + vz) / h
    rows, cols, vals = [idx], [idx], [diag]
    for (coord, stride, v) in ((ix, 1, vx), (iy, nx, vy), (iz, nx * nx, vz)):
        m = coord > 0  # lower neighbour: diffusion + upwind inflow (v > 0)
        rows.append(idx[m]); cols.append(idx[m] - stride)
        vals.append(kappa[m] / h**2 + v / h)
        m = coord < nx - 1  # upper neighbour: diffusion only
        rows.append(idx[m]); cols.append(idx[m] + stride)
        vals.append(kappa[m] / h**2)
    a = sp.csr_array((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                     shape=(n, n))
    a.sum_duplicates()
    a.sort_indices()
    a.indices = a.indices.astype(np.int32)
    a.indptr = a.indptr.astype(np.int32)
    return a


@dataclass
class Cfg4Inputs:
    a: sp.csr_array
    phi_s: np.ndarray          # N x n_s
    temporal: tuple            # n_s arrays of N_t x n_t
    dt: np.ndarray
    b: sp.csr_array            # N x 1
    x0: np.ndarray
    c: np.ndarray              # N x 1
    f_const: np.ndarray

    def inputs(self, k: int) -> np.ndarray:
        return self.f_const


def cfg4_inputs(nx: int = CFG4_NX, n_s: int = CFG4_NS, n_t: int = CFG4_NT_MODES,
                n_steps: int = CFG4_NSTEPS, dt: float = CFG4_DT) -> Cfg4Inputs:
    """Operator (seed 1), Haar Phi_s (seed 2), Haar temporal blocks (seed 3),
    dense B column (seed 4), x0 (seed 5); f = 1 constant."""
    a = cfg4_operator(nx, seed=1)
    n = a.shape[0]
    phi = haar(np.random.default_rng(2), n, n_s)
    rng3 = np.random.default_rng(3)
    temporal = tuple(haar(rng3, n_steps, n_t) for _ in range(n_s))
    bcol = np.random.default_rng(4).standard_normal((n, 1))
    x0 = np.random.default_rng(5).standard_normal(n)
    c = np.full((n, 1), 1.0 / n)
    return Cfg4Inputs(a=a, phi_s=phi, temporal=temporal, dt=np.full(n_steps, dt),
                      b=sp.csr_array(bcol), x0=x0, c=c, f_const=np.ones(1))


# --------------------------------------------------------------------------
# small random instances (same recipes as the reference's verify.py:52-82)
# --------------------------------------------------------------------------

def random_basis(rng, n_states, n_steps, n_s, n_t):
    phi = haar(rng, n_states, n_s)
    temporal = tuple(haar(rng, n_steps, n_t) for _ in range(n_s))
    return phi, temporal


def random_stable_system(rng, n_states, n_inputs=1):
    """Dense diagonally-shifted Gaussian A, Gaussian B/C/x0; per-step random inputs."""
    a = rng.standard_normal((n_states, n_states))
    a -= (np.abs(a).sum(axis=1).max() + 0.5) * np.eye(n_states)
    sig_rng = np.random.default_rng(rng.integers(2**63))
    cache = {}

    def signal(k):
        if k not in cache:
            cache[k] = np.asarray(sig_rng.standard_normal(n_inputs))
        return cache[k]

    return dict(a=sp.csr_array(a), b=sp.csr_array(rng.standard_normal((n_states, n_inputs))),
                c=rng.standard_normal((n_states, 1)), x0=rng.standard_normal(n_states),
                inputs=signal)


# --------------------------------------------------------------------------
# cfg5: capacity stream on the device (BASELINE.json configs[4])
# --------------------------------------------------------------------------

class HadamardStream:
    """Low-rank-plus-noise stream X = Q diag(sigma) W^T + E generated on the device.

    The capacity configuration (2^26 rows, 1000 snapshots, rank 100) does not
    fit on the host (537 GB) and its Haar Q (54 GB) would not fit next to the
    iSVD store, so Q is an implicit randomized Hadamard matrix
    Q[i, c] = s_i (-1)^popcount(i & p_c) / sqrt(n) with orthonormal columns,
    never stored (C ABI ``strom_gen_lowrank_batch``).  W is Haar (device QR),
    sigma_c = 10^(-c / decades_per), E = noise * N(0, 1) from a counter hash, so
    any column can be regenerated bit-identically.
    """

    def __init__(self, n: int, cols: int, rank: int, decades_per: float = 12.0, seed: int = 0,
                 noise: float = 1e-12, device: str = "cuda"):
        import torch

        if n < 2 or n & (n - 1):
            raise ValueError("HadamardStream needs n = 2^m")
        self.n, self.cols, self.rank, self.seed, self.noise = n, cols, rank, seed, noise
        g = torch.Generator(device=device)
        g.manual_seed(seed)
        a = torch.randn(cols, rank, generator=g, device=device, dtype=torch.float64)
        q, r = torch.linalg.qr(a, mode="reduced")
        d = torch.sign(torch.diagonal(r))
        d[d == 0] = 1.0
        self.w = (q * d).contiguous()                                   # cols x rank
        self.sigma = torch.tensor(cfg2_sigma(rank, decades_per), device=device, dtype=torch.float64)
        self.prow = torch.tensor([((c + 1) * 0x9E3779B1) % n for c in range(rank)], device=device,
                                 dtype=torch.int64)
        self.device = device

    def _gen(self, coef, t0: int, nb: int, noise: float, out=None):
        import torch

        from paper_1910_01260_b200 import _capi as capi  # absolute: bench.py loads this file by path

        if out is None:
            out = torch.empty((nb, self.n), dtype=torch.float64, device=self.device)
        capi.call("strom_gen_lowrank_batch", self.n, self.rank, nb, coef.data_ptr(), self.prow.data_ptr(),
                  self.seed, t0, noise, out.data_ptr(), self.n, capi.stream_ptr())
        return out.T  # n x nb, column-major

    def batch(self, t0: int, nb: int, out=None):
        """Columns t0 .. t0+nb-1 of X as an (n, nb) column-major CUDA tensor."""
        coef = (self.w[t0:t0 + nb] * self.sigma).T.contiguous()        # rank x nb, row-major
        return self._gen(coef, t0, nb, self.noise, out)

    def q_columns(self, c0: int, nc: int, out=None):
        """Columns c0 .. c0+nc-1 of the implicit Q (noise-free), (n, nc) column-major."""
        import torch

        coef = torch.zeros((self.rank, nc), dtype=torch.float64, device=self.device)
        coef[torch.arange(c0, c0 + nc), torch.arange(nc)] = 1.0
        return self._gen(coef, 0, nc, 0.0, out)


# --------------------------------------------------------------------------
# cfg3: 3D discrete-ordinates transport proxy (BASELINE.json configs[2])
# --------------------------------------------------------------------------

CFG3_NC = 64
CFG3_DT = 0.01
CFG3_NT = 100
CFG3_AMPLITUDES = (0.5, 1.0, 1.5, 2.0)
CFG3_TOL = 1e-8
CFG3_DIRECTIONS = np.array([[1.0, 1.0, 1.0], [-1.0, -1.0, -1.0], [1.0, -1.0, 1.0], [-1.0, 1.0, -1.0]]) / np.sqrt(3.0)


def cfg3_source(nc: int = CFG3_NC, seed: int = 6, n_gauss: int = 8, width: float = 0.1) -> np.ndarray:
    """Sum of 8 Gaussians (width 0.1, centres U[0,1]^3, seed 6) at the cell centres, x fastest."""
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0.0, 1.0, (n_gauss, 3))
    xc = (np.arange(nc) + 0.5) / nc
    z, y, x = np.meshgrid(xc, xc, xc, indexing="ij")  # cell (iz, iy, ix) at index (iz*nc + iy)*nc + ix
    g = np.zeros((nc, nc, nc))
    for c in centres:
        g += np.exp(-((x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2) / (2.0 * width**2))
    return g.ravel()


def cfg3_operator(nc: int = CFG3_NC, sigma_t: float = 1.0, sigma_s: float = 0.5, speed: float = 1.0):
    """dx/dt = nu (scatter - H) x on nc^3 cells x 4 directions, direction-major.

    The 3D analogue of the reference's transport1d (problems.py:196-247): per
    direction H_d = first-order upwind streaming Omega_d . grad with vacuum
    inflow plus sigma_t; isotropic scattering with equal weights 1/4 couples
    the directions of a cell.  Unknown (d, iz, iy, ix) at d * nc^3 +
    (iz * nc + iy) * nc + ix."""
    nd = CFG3_DIRECTIONS.shape[0]
    ncell = nc**3
    h = 1.0 / nc
    iz, iy, ix = np.meshgrid(np.arange(nc), np.arange(nc), np.arange(nc), indexing="ij")
    iz, iy, ix = iz.ravel(), iy.ravel(), ix.ravel()
    cell = np.arange(ncell)
    rows, cols, vals = [], [], []
    w = 1.0 / nd
    for d, om in enumerate(CFG3_DIRECTIONS):
        base = d * ncell
        diag = np.full(ncell, -speed * (np.sum(np.abs(om)) / h + sigma_t) + speed * sigma_s * w)
        rows.append(base + cell)
        cols.append(base + cell)
        vals.append(diag)
        for axis, (coord, stride) in enumerate(((ix, 1), (iy, nc), (iz, nc * nc))):
            o = om[axis]
            up = coord - 1 if o > 0 else coord + 1  # upstream neighbour along this axis
            ok = (up >= 0) & (up < nc)               # vacuum inflow: no entry at the boundary
            shift = -stride if o > 0 else stride
            rows.append(base + cell[ok])
            cols.append(base + cell[ok] + shift)
            vals.append(np.full(int(ok.sum()), speed * abs(o) / h))
        for d2 in range(nd):
            if d2 != d:
                rows.append(base + cell)
                cols.append(d2 * ncell + cell)
                vals.append(np.full(ncell, speed * sigma_s * w))
    n = nd * ncell
    a = sp.csr_array((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))
    a.sort_indices()
    return a


@dataclass
class Cfg3Inputs:
    a: sp.csr_array
    b: np.ndarray
    c: np.ndarray
    x0: np.ndarray
    amplitude: float

    def inputs(self, k):
        return np.array([self.amplitude])


def cfg3_system(amplitude: float, nc: int = CFG3_NC, seed: int = 6, a=None) -> Cfg3Inputs:
    """Transport proxy at one training amplitude: x0 = the smooth source in every
    direction, B = the same field, constant input f = amplitude; output = the
    scalar flux integral (weights 1/4 x cell volume, as transport1d's c_out)."""
    g = cfg3_source(nc, seed)
    nd = CFG3_DIRECTIONS.shape[0]
    if a is None:
        a = cfg3_operator(nc)
    field = np.tile(g, nd)
    c = np.full((nd * nc**3, 1), (1.0 / nd) / nc**3)
    return Cfg3Inputs(a=a, b=field[:, None].copy(), c=c, x0=field.copy(), amplitude=float(amplitude))
