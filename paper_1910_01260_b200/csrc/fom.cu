// Full-order backward-Euler march on the device (reference system.py:150-163
// fom_march, system.py:106-147 StepSolver / backward_euler_step): the snapshot
// producer that feeds the incremental SVD without a host round trip.
//
//   (I - dt_k A) x_k = x_{k-1} + dt_k B f_k ,   k = 1 .. N_t
//
// The reference factors I - dt A with SuperLU; at the transport-proxy size
// (2^20 dofs in 3D) that is infeasible, so each step is
// solved by BiCGSTAB on the left-Jacobi-preconditioned system D^-1 M x =
// D^-1 b (M = I - dt A, D = diag M; the scaling is applied row by row inside
// the SpMV, so no preconditioned copies of the iterates exist), started from
// x_{k-1}, to a relative preconditioned residual tol (default 1e-13), over the
// tiled-ELL operator of the spatial reduction (diagonal kept apart).
//
// One cooperative persistent kernel marches every step: grid-wide syncs
// separate the phases; dot products are per-CTA partials summed by every CTA
// in CTA order (deterministic, identical on every CTA).  Systems of up to 8192
// rows march in one 512-thread CTA instead: a grid barrier costs microseconds,
// a CTA barrier tens of nanoseconds; up to 2560 rows the vectors (the iterate
// included) live in shared memory, above that in L1.
#include <cooperative_groups.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/strom_b200.h"
#include "common.cuh"
#include "runtime.cuh"

using namespace strom;
namespace cg = cooperative_groups;

namespace {

constexpr int kFomThreads = 256;
constexpr int kFomOneThreads = 512;
constexpr int64_t kFomOneMax = 8192;   // single-CTA march up to this many rows
constexpr int64_t kFomSmemMax = 2560;  // ... with its vectors in shared memory (180 KB)
// BiCGSTAB restarts from the true residual every kFomRestart iterations: near
// a 1e-13 relative residual the shadow residual loses its grip ((r^, r) at
// rounding level) and the recursion can wander for hundreds of iterations
// (the cfg1 test system shows it at step 92); a fresh start converges in a few.
constexpr int kFomRestart = 100;
constexpr int kEllRows = 64;  // tile height of the ELL layout (spatial.cu)

struct FomArgs {
  int64_t n;
  int K;
  const uint32_t* eidx;  // per 64-row tile: [K][64] off-diagonal columns
  const double* eval;    // per tile: [K][64] off-diagonal values, then [64] diagonal
  const double* b;       // n x m column-major (ldb = n)
  int m;
  const double* x0;
  const double* dt;      // N_t
  const double* f;       // N_t x m row-major (row k = input of step k+1)
  const double* v;       // or: n x N_t column-major right-hand-side blocks (rhs_k = x_{k-1} + v_k), x0 = 0
  int nt;
  double tol;
  int maxit;
  double* states;        // n x N_t column-major (ld = n)
  double* w;             // 7 work vectors of n: r, rh, p, v, s, t, b
  double* part;          // 2 x 3 x gridDim partial sums
  int* iters;            // N_t iteration counts (-1: not converged)
};

// Row i of the left-Jacobi-preconditioned step operator D^-1 (I - dt A), D =
// diag(I - dt A):  y_i = z_i - (dt / d_i) sum_k a_ik z_{c_ik}  (off-diagonal
// slots only; the scaled diagonal is 1).
// ONE passes the precomputed row scale sc = -dt / d_i (one fp64 division per
// row and step instead of per SpMV); the HBM-bound grid mode recomputes it.
template <int K, bool ONE>
__device__ __forceinline__ double mrow(const FomArgs& a, int64_t i, double dt, const double* __restrict__ z,
                                       const double* __restrict__ sc) {
  const int64_t tile = i / kEllRows;
  const int li = (int)(i % kEllRows);
  const uint32_t* ti = a.eidx + tile * K * kEllRows + li;
  const double* tv = a.eval + tile * (K + 1) * kEllRows + li;
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < K; ++k) acc = fma(tv[k * kEllRows], z[ti[k * kEllRows]], acc);
  if constexpr (ONE) return fma(sc[i], acc, z[i]);
  else return fma(-dt / (1.0 - dt * tv[K * kEllRows]), acc, z[i]);
}

template <int K>
__device__ __forceinline__ double mdiag(const FomArgs& a, int64_t i, double dt) {
  return 1.0 - dt * a.eval[(i / kEllRows) * (K + 1) * kEllRows + K * kEllRows + i % kEllRows];
}

// deterministic reduction of NV <= 3 values: every CTA returns the same sums.
// Grid mode: per-CTA partials summed by every CTA in CTA order; consecutive
// reductions alternate between two partial buffers, so a CTA writing
// reduction R+1 never races a CTA still reading reduction R.  Single-CTA mode
// (small n): warp partials summed in warp order, no grid barrier.
template <bool ONE, int NT, int NV>
__device__ __forceinline__ void reduce3(cg::grid_group& grid, double* part_base, int& nred, double v0, double v1,
                                        double v2, double* out, double* sred) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double vv[3] = {v0, v1, v2};
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double s = warp_sum(vv[q]);
    if (lane == 0) sred[q * NW + w] = s;
  }
  __syncthreads();
  if constexpr (ONE) {
    static_assert(NW <= 32, "single-CTA mode reduces one partial per lane");
    if (w < NV) {
      const double s = warp_sum(lane < NW ? sred[w * NW + lane] : 0.0);  // fixed shuffle tree
      if (lane == 0) sred[3 * NW + w] = s;
    }
  } else {
    double* part = part_base + (int64_t)(nred++ & 1) * 3 * gridDim.x;
    if (threadIdx.x < NV) {
      double s = 0.0;
      for (int k = 0; k < NW; ++k) s += sred[threadIdx.x * NW + k];
      part[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = s;
    }
    grid.sync();
    if (w < NV) {
      double s = 0.0;
      for (int c = lane; c < (int)gridDim.x; c += 32) s += part[(int64_t)w * gridDim.x + c];
      s = warp_sum(s);  // fixed shuffle tree: the same on every CTA
      if (lane == 0) sred[3 * NW + w] = s;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) out[q] = sred[3 * NW + q];
  __syncthreads();
}

template <bool ONE>
__device__ __forceinline__ void sync_all(cg::grid_group& grid) {
  if constexpr (ONE) __syncthreads();
  else grid.sync();
}

// ONE: a single 512-thread CTA marches a small system (n <= kFomOneMax); the
// vectors stay in L1 and every barrier is a CTA barrier.  Otherwise one
// cooperative grid of kFomThreads-thread CTAs.
// SMEM (single-CTA only, n <= kFomSmemMax): the eight vectors, x included,
// live in shared memory; x is copied out to the states column after each step.
template <int K, bool ONE, bool SMEM>
__global__ void __launch_bounds__(ONE ? kFomOneThreads : kFomThreads) k_fom_march(FomArgs a) {
  constexpr int NT = ONE ? kFomOneThreads : kFomThreads;
  static_assert(ONE || !SMEM, "shared-memory vectors need the single-CTA mode");
  cg::grid_group grid = cg::this_grid();
  __shared__ double sred[3 * (NT / 32) + 3];
  extern __shared__ double svec[];
  const int64_t n = a.n;
  const int64_t g0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gs = (int64_t)gridDim.x * blockDim.x;
  // BiCGSTAB on the left-preconditioned system D^-1 M x = D^-1 b (M = I - dt A)
  double* wv = SMEM ? svec : a.w;
  double* r = wv;
  double* rh = wv + n;
  double* p = wv + 2 * n;
  double* v = wv + 3 * n;
  double* s = wv + 4 * n;
  double* t = wv + 5 * n;
  double* bb = wv + 6 * n;
  double* xs = wv + 7 * n;  // SMEM: the iterate
  double* sc = wv + 8 * n;  // ONE: row scales -dt / d_i of the current step
  double red[3];
  int nred = 0;
  for (int k = 0; k < a.nt; ++k) {
    const double dt = a.dt[k];
    // x0 may be null (zero); SMEM marches x in place from x_{k-1}
    const double* xp = k == 0 ? a.x0 : SMEM ? xs : a.states + (int64_t)(k - 1) * n;
    double* x = SMEM ? xs : a.states + (int64_t)k * n;
    // preconditioned rhs D^-1 (x_{k-1} + dt B f_k); initial guess x = x_{k-1}
    for (int64_t i = g0; i < n; i += gs) {
      const double xpi = xp ? xp[i] : 0.0;
      double bi = xpi;
      if (a.v) bi += a.v[(int64_t)k * n + i];
      else
        for (int q = 0; q < a.m; ++q) bi = fma(dt * a.b[(int64_t)q * n + i], a.f[(int64_t)k * a.m + q], bi);
      const double di = mdiag<K>(a, i, dt);
      bb[i] = bi / di;
      if constexpr (ONE) sc[i] = -dt / di;
      x[i] = xpi;
    }
    sync_all<ONE>(grid);
    double rho = 0.0, stop2 = 0.0;
    int it = 0;
    bool ok = false, fresh = true;
    for (;;) {
      if (fresh) {
        // (re)start from the true residual of the current iterate; restarts
        // recover from breakdowns and from the stagnation BiCGSTAB shows once
        // the recursive residual nears rounding level (see kFomRestart)
        fresh = false;
        double pr = 0.0, pb = 0.0;
        for (int64_t i = g0; i < n; i += gs) {
          const double ri = bb[i] - mrow<K, ONE>(a, i, dt, x, sc);
          r[i] = ri;
          rh[i] = ri;
          p[i] = ri;
          pr = fma(ri, ri, pr);
          pb = fma(bb[i], bb[i], pb);
        }
        reduce3<ONE, NT, 2>(grid, a.part, nred, pr, pb, 0.0, red, sred);
        rho = red[0];
        stop2 = a.tol * a.tol * red[1];
        if (red[0] <= stop2) {
          ok = true;
          break;
        }
      }
      if (it >= a.maxit) break;
      ++it;
      // v = M' p ; (rh, v)
      double prv = 0.0;
      for (int64_t i = g0; i < n; i += gs) {
        const double vi = mrow<K, ONE>(a, i, dt, p, sc);
        v[i] = vi;
        prv = fma(rh[i], vi, prv);
      }
      reduce3<ONE, NT, 1>(grid, a.part, nred, prv, 0.0, 0.0, red, sred);
      if (red[0] == 0.0) {  // breakdown
        fresh = true;
        continue;
      }
      const double alpha = rho / red[0];
      for (int64_t i = g0; i < n; i += gs) s[i] = fma(-alpha, v[i], r[i]);
      sync_all<ONE>(grid);
      // t = M' s ; (t, s), (t, t), (s, s)
      double pts = 0.0, ptt = 0.0, pss = 0.0;
      for (int64_t i = g0; i < n; i += gs) {
        const double ti = mrow<K, ONE>(a, i, dt, s, sc);
        const double si = s[i];
        t[i] = ti;
        pts = fma(ti, si, pts);
        ptt = fma(ti, ti, ptt);
        pss = fma(si, si, pss);
      }
      reduce3<ONE, NT, 3>(grid, a.part, nred, pts, ptt, pss, red, sred);
      if (red[2] <= stop2) {  // converged on s: x + alpha p
        for (int64_t i = g0; i < n; i += gs) x[i] = fma(alpha, p[i], x[i]);
        ok = true;
        break;
      }
      if (red[1] == 0.0) break;  // t = M s = 0 with s != 0: M is singular
      const double omega = red[0] / red[1];
      double prr = 0.0, prh = 0.0;
      for (int64_t i = g0; i < n; i += gs) {
        x[i] = fma(omega, s[i], fma(alpha, p[i], x[i]));
        const double ri = fma(-omega, t[i], s[i]);
        r[i] = ri;
        prr = fma(ri, ri, prr);
        prh = fma(rh[i], ri, prh);
      }
      reduce3<ONE, NT, 2>(grid, a.part, nred, prr, prh, 0.0, red, sred);
      if (red[0] <= stop2) {
        ok = true;
        break;
      }
      if (omega == 0.0 || red[1] == 0.0 || it % kFomRestart == 0) {
        fresh = true;
        continue;
      }
      const double beta = (red[1] / rho) * (alpha / omega);
      rho = red[1];
      for (int64_t i = g0; i < n; i += gs) p[i] = r[i] + beta * fma(-omega, v[i], p[i]);
      sync_all<ONE>(grid);
    }
    if constexpr (SMEM)
      for (int64_t i = g0; i < n; i += gs) a.states[(int64_t)k * n + i] = x[i];
    if (blockIdx.x == 0 && threadIdx.x == 0) a.iters[k] = ok ? it : -1;
    sync_all<ONE>(grid);
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// Direct march for (periodic) tridiagonal operators: 1-D problems (cfg1: periodic
// advection-diffusion, n = 1024) are latency work for a Krylov solver (33
// BiCGSTAB iterations of 3.6 us per step) and a trivial direct solve, which is
// what the reference does (SuperLU factor once per dt, system.py:106-125).
// Parallel cyclic reduction in ONE CTA: level s combines equation i with
// equations i -+ 2^s,
//   alpha = -l_i / d_{i-s},  gamma = -u_i / d_{i+s},
//   l_i' = alpha l_{i-s},  u_i' = gamma u_{i+s},  d_i' = d_i + alpha u_{i-s} + gamma l_{i+s},
//   r_i' = r_i + alpha r_{i-s} + gamma r_{i+s},
// and after ceil(log2 n) levels x_i = r_i / d_i (non-periodic) or
// r_i / (l_i + d_i + u_i) (periodic, n a power of two: the neighbours are i itself).
// The multipliers depend on dt only: they are tabulated per distinct dt
// (levels x n alpha / gamma and the final reciprocal, in global memory and then
// L1), so a step is the right-hand side's levels: two fused multiply-adds per
// row and level.  No pivoting: the host checks strict diagonal dominance of
// I - dt A before taking this path (otherwise the Krylov march runs).
// ---------------------------------------------------------------------------
namespace {
constexpr int kTriThreads = 1024;
constexpr int kTriMaxN = 4096;
constexpr int kTriRows = kTriMaxN / kTriThreads;

struct TriArgs {
  int n, nt, m, periodic, levels;
  const double* lo;   // A(i, i-1)  (periodic: lo[0] = A(0, n-1))
  const double* di;   // A(i, i)
  const double* up;   // A(i, i+1)  (periodic: up[n-1] = A(n-1, 0))
  const double* b;    // m x n (B column-major)
  const double* x0;
  const double* dt;
  const double* f;    // nt x m row-major, or null
  const double* v;    // n x nt column-major right-hand-side blocks (st_apply_inverse), or null
  double* states;     // n x nt column-major
  double* tab;        // (2 levels + 1) x n: alpha, gamma per level, then the final reciprocal
};

__global__ void __launch_bounds__(kTriThreads, 1) k_fom_tridiag(TriArgs a) {
  extern __shared__ double sm[];  // 6 n: l, d, u ping-pong during the set-up; 2 n: r ping-pong afterwards
  const int n = a.n, L = a.levels;
  const int tid = threadIdx.x;
  double* alpha = a.tab;
  double* gamma = a.tab + (size_t)L * n;
  double* rinv = a.tab + (size_t)2 * L * n;
  double dt_tab = -1.0;  // the dt the tables hold
  auto nb = [&](int i, int s, bool& ok) {  // neighbour index of i at distance s (s may be negative)
    int j = i + s;
    if (a.periodic) {
      ok = true;
      j %= n;
      if (j < 0) j += n;
    } else {
      ok = j >= 0 && j < n;
      if (!ok) j = i;
    }
    return j;
  };
  for (int k = 0; k < a.nt; ++k) {
    const double h = a.dt[k];
    if (h != dt_tab) {
      // ---- tables of M = I - h A
      double* l0 = sm; double* d0 = sm + n; double* u0 = sm + 2 * n;
      double* l1 = sm + 3 * n; double* d1 = sm + 4 * n; double* u1 = sm + 5 * n;
      __syncthreads();
      for (int i = tid; i < n; i += kTriThreads) {
        l0[i] = (a.periodic || i > 0) ? -h * a.lo[i] : 0.0;
        d0[i] = 1.0 - h * a.di[i];
        u0[i] = (a.periodic || i < n - 1) ? -h * a.up[i] : 0.0;
      }
      __syncthreads();
      for (int lev = 0, s = 1; lev < L; ++lev, s <<= 1) {
        for (int i = tid; i < n; i += kTriThreads) {
          bool okm, okp;
          const int im = nb(i, -s, okm), ip = nb(i, s, okp);
          const double al = okm ? -l0[i] / d0[im] : 0.0;
          const double ga = okp ? -u0[i] / d0[ip] : 0.0;
          alpha[(size_t)lev * n + i] = al;
          gamma[(size_t)lev * n + i] = ga;
          l1[i] = okm ? al * l0[im] : 0.0;
          u1[i] = okp ? ga * u0[ip] : 0.0;
          d1[i] = d0[i] + (okm ? al * u0[im] : 0.0) + (okp ? ga * l0[ip] : 0.0);
        }
        __syncthreads();
        double* t;
        t = l0; l0 = l1; l1 = t;
        t = d0; d0 = d1; d1 = t;
        t = u0; u0 = u1; u1 = t;
      }
      for (int i = tid; i < n; i += kTriThreads)
        rinv[i] = 1.0 / (a.periodic ? (l0[i] + d0[i] + u0[i]) : d0[i]);
      __threadfence_block();
      __syncthreads();
      dt_tab = h;
    }
    // ---- right-hand side: x_{k-1} + h B f_k  (or x_{k-1} + v_k)
    double* r0 = sm; double* r1 = sm + n;
    const double* xp = k ? a.states + (size_t)(k - 1) * n : a.x0;
    for (int i = tid; i < n; i += kTriThreads) {
      double r = (k || a.x0) ? xp[i] : 0.0;
      if (a.v) r += a.v[(size_t)k * n + i];
      if (a.f) {
        double bf = 0.0;
        for (int q = 0; q < a.m; ++q) bf = fma(a.b[(size_t)q * n + i], a.f[(size_t)k * a.m + q], bf);
        r = fma(h, bf, r);
      }
      r0[i] = r;
    }
    __syncthreads();
    for (int lev = 0, s = 1; lev < L; ++lev, s <<= 1) {
      for (int i = tid; i < n; i += kTriThreads) {
        bool okm, okp;
        const int im = nb(i, -s, okm), ip = nb(i, s, okp);
        r1[i] = fma(alpha[(size_t)lev * n + i], r0[im], fma(gamma[(size_t)lev * n + i], r0[ip], r0[i]));
      }
      __syncthreads();
      double* t = r0; r0 = r1; r1 = t;
    }
    double* xk = a.states + (size_t)k * n;
    for (int i = tid; i < n; i += kTriThreads) xk[i] = r0[i] * rinv[i];
    __threadfence_block();
    __syncthreads();
  }
}
}  // namespace

extern "C" {

// fom_march (system.py:150-163) on the device: states (n x N_t, column-major)
// column k-1 = x_k.  The operator is the tiled ELL form of A
// (strom_csr_to_ell, K in {4, 6, 8, 16}); b_dev n x m column-major; f_dev
// N_t x m row-major (row k = input of step k+1); dt_dev N_t.  iters_out
// (host, N_t ints, may be NULL): BiCGSTAB iterations per step, -1 where the
// relative residual did not reach tol within maxit (the call then returns a
// numerical error).
static int fom_march_impl(int64_t n, int32_t K, const uint32_t* eidx_dev, const double* eval_dev,
                          const double* b_dev, int64_t m, const double* x0_dev, const double* dt_dev,
                          const double* f_dev, const double* v_dev, int64_t nt, double tol, int32_t maxit,
                          double* states_dev, int32_t* iters_out, void* stream);

int strom_fom_march(int64_t n, int32_t K, const uint32_t* eidx_dev, const double* eval_dev, const double* b_dev,
                    int64_t m, const double* x0_dev, const double* dt_dev, const double* f_dev, int64_t nt, double tol,
                    int32_t maxit, double* states_dev, int32_t* iters_out, void* stream) {
  return fom_march_impl(n, K, eidx_dev, eval_dev, b_dev, m, x0_dev, dt_dev, f_dev, nullptr, nt, tol, maxit, states_dev,
                        iters_out, stream);
}

// fom_march for a tridiagonal or periodic tridiagonal A (diagonals lo, di, up; see k_fom_tridiag).
// v_dev non-null: the forward block substitution of st_apply_inverse instead (b, f, x0 null).
int strom_fom_march_tridiag(int64_t n, const double* lo_dev, const double* di_dev, const double* up_dev,
                            int32_t periodic, const double* b_dev, int64_t m, const double* x0_dev,
                            const double* dt_dev, const double* f_dev, const double* v_dev, int64_t nt,
                            double* states_dev, void* stream) {
  return guarded([&] {
    STROM_REQUIRE(n >= 2 && n <= kTriMaxN && nt >= 1 && m >= 0, "bad tridiagonal march shape");
    STROM_REQUIRE(lo_dev && di_dev && up_dev && dt_dev && states_dev, "null argument");
    STROM_REQUIRE(!periodic || (n & (n - 1)) == 0, "the periodic tridiagonal march needs n = 2^k");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int levels = 0;
    while (((int64_t)1 << levels) < n) ++levels;
    auto tab = dev_alloc((size_t)(2 * levels + 1) * n * 8, s, false);
    TriArgs a{};
    a.n = (int)n; a.nt = (int)nt; a.m = (int)m; a.periodic = periodic ? 1 : 0; a.levels = levels;
    a.lo = lo_dev; a.di = di_dev; a.up = up_dev; a.b = b_dev; a.x0 = x0_dev; a.dt = dt_dev; a.f = f_dev; a.v = v_dev;
    a.states = states_dev; a.tab = tab->as<double>();
    const size_t smem = (size_t)6 * n * 8;
    STROM_CUDA(cudaFuncSetAttribute(k_fom_tridiag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_fom_tridiag<<<1, kTriThreads, smem, s>>>(a);
    STROM_LAUNCH_CHECK();
  });
}

// (A_st)^{-1} v by forward block substitution (system.py:195-213 st_apply_inverse):
// x_k solves (I - dt_k A) x_k = x_{k-1} + v_k, x_0 = 0; v_dev and out_dev n x N_t
// column-major.  The adjoint (system.py:216-233) is the same march over the
// transposed operator's ELL form with the blocks and steps in reverse order.
int strom_st_apply_inverse(int64_t n, int32_t K, const uint32_t* eidx_dev, const double* eval_dev, const double* dt_dev,
                           const double* v_dev, int64_t nt, double tol, int32_t maxit, double* out_dev,
                           int32_t* iters_out, void* stream) {
  return fom_march_impl(n, K, eidx_dev, eval_dev, nullptr, 0, nullptr, dt_dev, nullptr, v_dev, nt, tol, maxit,
                        out_dev, iters_out, stream);
}

static int fom_march_impl(int64_t n, int32_t K, const uint32_t* eidx_dev, const double* eval_dev,
                          const double* b_dev, int64_t m, const double* x0_dev, const double* dt_dev,
                          const double* f_dev, const double* v_dev, int64_t nt, double tol, int32_t maxit,
                          double* states_dev, int32_t* iters_out, void* stream) {
  return guarded([&] {
    STROM_REQUIRE(n >= 1 && nt >= 1 && m >= 0, "bad fom_march shape");
    STROM_REQUIRE(K == 4 || K == 6 || K == 8 || K == 16, "ELL width must be 4, 6, 8 or 16");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const bool one = n <= kFomOneMax, smem = n <= kFomSmemMax;
#define STROM_FOM_K(O, S) (K == 4 ? k_fom_march<4, O, S> : K == 6 ? k_fom_march<6, O, S> \
                           : K == 8 ? k_fom_march<8, O, S> : k_fom_march<16, O, S>)
    auto kern = smem ? STROM_FOM_K(true, true) : one ? STROM_FOM_K(true, false) : STROM_FOM_K(false, false);
#undef STROM_FOM_K
    const int threads = one ? kFomOneThreads : kFomThreads;
    const size_t dsmem = smem ? (size_t)9 * n * sizeof(double) : 0;
    if (smem) STROM_CUDA(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsmem));
    int occ = 0;
    STROM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, dsmem));
    STROM_REQUIRE(occ >= 1, "fom_march kernel cannot be resident");
    const int64_t want = ceil_div(n, kFomThreads);
    const int grid = one ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count() * std::min(occ, 4)));
    auto work = dev_alloc((size_t)9 * n * 8, s, false);
    auto part = dev_alloc((size_t)6 * grid * 8, s, true);
    auto its = dev_alloc((size_t)nt * 4, s, true);
    FomArgs a{};
    a.n = n;
    a.K = K;
    a.eidx = eidx_dev;
    a.eval = eval_dev;
    a.b = b_dev;
    a.m = (int)m;
    a.x0 = x0_dev;
    a.dt = dt_dev;
    a.f = f_dev;
    a.v = v_dev;
    a.nt = (int)nt;
    a.tol = tol;
    a.maxit = maxit;
    a.states = states_dev;
    a.w = work->as<double>();
    a.part = part->as<double>();
    a.iters = its->as<int>();
    void* args[] = {&a};
    STROM_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(threads), args, dsmem, s));
    STROM_LAUNCH_CHECK();
    std::vector<int> h((size_t)nt);
    STROM_CUDA(cudaMemcpyAsync(h.data(), its->ptr, (size_t)nt * 4, cudaMemcpyDeviceToHost, s));
    STROM_CUDA(cudaStreamSynchronize(s));
    if (iters_out)
      for (int64_t k = 0; k < nt; ++k) iters_out[k] = h[k];
    for (int64_t k = 0; k < nt; ++k)
      if (h[k] < 0)
        throw Error(kNumericalError, "fom_march: step " + std::to_string(k + 1) +
                                         " did not reach the residual tolerance (BiCGSTAB)");
  });
}

}  // extern "C"
