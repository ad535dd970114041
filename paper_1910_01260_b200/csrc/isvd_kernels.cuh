// Device kernels of the streaming incremental SVD (reference basis.py:105-184).
//
// Representation: the reference keeps the
// n x r left basis Phi explicitly and rewrites it every snapshot
// (Phi' = [Phi j] W_bar, basis.py:155-156).  Here Phi = Q_U N with
//   U    n x c_cap  append-only column store in HBM (column-major, ld = ldu),
//                   columns nearly orthogonal; G = U^T U = L L^T tracked exactly
//   Q_U  = U L^{-T} (never formed): an orthonormal basis of span(U)
//   N    c x r      Phi's coordinates in Q_U (small, read by one CTA); Phi^T Phi = N^T N
// (U-coordinates, needed by the passes and the export, are W = L^{-T} N).
// so one snapshot costs one projection pass (g = U^T x) and, when the column is
// independent, one residual pass that appends r1 = x - U G^{-1} g and measures
// e = U^T r1, |r1|^2.  Everything else -- the bordered core SVD, the W and V
// rotations, truncation, drift test, re-orthogonalisation -- is small-space
// work on one CTA.  The reference's tall QR (basis.py:174) becomes a QR of the
// (c x r) matrix L^T W; its Q is the same unique positive-diagonal Q.
#pragma once

#include "common.cuh"
#include "core_svd.cuh"
#include "small_dense.cuh"

namespace strom {

// -------- per-state header (lives in the state's small block) --------------
struct IsvdHdr {
  int32_t r;       // rank = sigma.size
  int32_t c;       // logical columns of U in use
  int32_t base;    // physical column of logical column 0
  int32_t status;  // 0 ok, 1 non-finite input
  int32_t n_rejected, n_dependent, n_truncated, n_restarts;
  int32_t flags;   // decision bits of the update that produced this state
  int32_t pad0;
  double p;        // Pythagorean residual norm of that update
  double drift;    // |phi_0 . phi_last| of that update
  double xnorm;    // ||x|| of that update
  double p_sq;     // unclamped x.x - ell.ell of that update
};

enum : int32_t {
  F_DEPENDENT = 1, F_TRUNCATED = 2, F_QR = 4, F_RESTART = 8, F_REJECTED = 16,
  F_APPENDED = 32, F_FOLDED = 64, F_ERROR = 128,
};

enum : int32_t { M_NORMAL_DEP = 0, M_NORMAL_INDEP = 1, M_RESTART_ACCEPT = 2, M_REJECT = 3, M_ERROR = 4 };

// -------- transient per-update scalars (scratch) ---------------------------
struct IsvdStep {
  int32_t mode, write_slot, c_dot, restart;
  int32_t m, mkeep, append, reorth;
  double xx, rho2, p, norm;
  int32_t pad_status, pad2;
  double p_sq;
};

struct StateView {
  IsvdHdr* hdr;
  double* N;      // c_cap x (r_cap + 1), ld = ldn   (Phi = U L^{-T} N)
  double* L;      // c_cap x c_cap lower, ld = ldl   (Cholesky factor of G = U^T U)
  double* Li;     // c_cap x c_cap lower, ld = ldl   (L^{-1}, kept explicitly)
  double* sigma;  // r_cap + 1
  double* V;      // k_cap x (r_cap + 1), ld = ldv
  int32_t ldn, ldl;
  int64_t ldv;
};

struct Scratch {
  double* g;      // c_cap   U^T x
  double* gt;     // c_cap   G^{-1} g
  double* y;      // c_cap   t - N ell  (t = L^{-1} g: x's coordinates in Q_U)
  double* ell;    // r_cap+1 Phi^T x
  double* e;      // c_cap   U^T r1
  double* h;      // c_cap   G^{-1} e of the first residual (DGKS correction), else 0
  double* lvec;   // c_cap   L^{-1} e
  double* l1;     // c_cap   L^{-1} e of the first residual (kept across the DGKS pass)
  double* tmp;    // c_cap   scratch vector
  double* vbar;   // (r_cap+2)^2 sorted, sign-fixed V_bar of the core
  double* work;   // large fallback workspace (global) for the one-CTA kernels
  double* T;      // c_cap x (r_cap+1) compaction transform
  double* part;   // per-CTA partial sums
  unsigned* counter;
  IsvdStep* step;
};

struct IsvdParams {
  int64_t n, ldu;
  int32_t ccap, rcap;
  double tol_svd, tol_sv;
  int32_t r_max;     // -1: no cap
  int32_t cap_mode;  // 0 restart, 1 truncate
  int64_t k_new;     // column counter after this update
  int32_t pstride;   // stride of one CTA's partial row
  int32_t work_stride;
  unsigned long long* prof;  // device byte counters (runtime.cuh ProfKind) or null
  long long* tprobe;         // phase timestamps of step B (diagnostics) or null
};

#define STROM_TPROBE(P, k)                                  \
  do {                                                      \
    if ((P).tprobe && threadIdx.x == 0) (P).tprobe[k] = clock64(); \
  } while (0)

constexpr int kTileRows = 64;
constexpr int kPassThreads = 256;
constexpr int kSmallThreads = 512;  // one-CTA kernels: 128 registers per thread (no spills)

// Deterministic grid finish: the last CTA to arrive sums the per-CTA partials
// in CTA order.  Returns true in that CTA (after the counter is reset).
__device__ inline bool last_cta_arrives(unsigned* counter, int* s_is_last) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(counter, 1u);
    *s_is_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (*s_is_last) {
    __threadfence();
    if (threadIdx.x == 0) *counter = 0u;
    return true;
  }
  return false;
}

// ---------------------------------------------------------------------------
// Projection pass: g = U[:, base:base+c]^T x and xx = x.x  (basis.py:135-136)
// Warp w owns columns w, w+8, ...; lane l owns rows 2l, 2l+1 of each 64-row
// tile (128-bit loads of U).  Contiguous tile ranges per CTA.
// ---------------------------------------------------------------------------
template <int MAXJ>
__global__ void __launch_bounds__(kPassThreads) k_proj(const double* __restrict__ U,
                                                        const double* __restrict__ x,
                                                        StateView src, Scratch sc, IsvdParams P) {
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int c = src.hdr->c, base = src.hdr->base;
  if (P.prof && blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd(P.prof + 0, 8ull * (unsigned long long)P.n * (unsigned long long)(c + 1));  // U cols + x
  const int64_t ntiles = P.ldu / kTileRows;
  const int64_t per = ceil_div(ntiles, gridDim.x);
  const int64_t t0 = blockIdx.x * per;
  const int64_t t1 = min(ntiles, t0 + per);
  double acc[MAXJ];
#pragma unroll
  for (int q = 0; q < MAXJ; ++q) acc[q] = 0.0;
  double xx = 0.0;
  for (int64_t t = t0; t < t1; ++t) {
    const int64_t row = t * kTileRows + 2 * lane;
    const double x0 = (row < P.n) ? __ldg(x + row) : 0.0;
    const double x1 = (row + 1 < P.n) ? __ldg(x + row + 1) : 0.0;
    if (wid == 0) xx = fma(x1, x1, fma(x0, x0, xx));
#pragma unroll
    for (int q = 0; q < MAXJ; ++q) {
      const int j = wid + 8 * q;
      if (j < c) {
        const double2 u = __ldg(reinterpret_cast<const double2*>(U + (int64_t)(base + j) * P.ldu + row));
        acc[q] = fma(u.y, x1, fma(u.x, x0, acc[q]));
      }
    }
  }
  double* mypart = sc.part + (int64_t)blockIdx.x * P.pstride;
#pragma unroll
  for (int q = 0; q < MAXJ; ++q) {
    const int j = wid + 8 * q;
    const double v = warp_sum(acc[q]);
    if (lane == 0 && j < c) mypart[j] = v;
  }
  if (wid == 0) {
    const double v = warp_sum(xx);
    if (lane == 0) mypart[P.ccap] = v;
  }
  if (!last_cta_arrives(sc.counter, &s_last)) return;
  // one warp per output, lanes stride over the CTA partials, fixed tree: deterministic
  for (int j = wid; j <= c; j += 8) {
    const int col = (j == c) ? P.ccap : j;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int b = lane;
    for (; b + 96 < (int)gridDim.x; b += 128) {
      s0 += sc.part[(int64_t)b * P.pstride + col];
      s1 += sc.part[(int64_t)(b + 32) * P.pstride + col];
      s2 += sc.part[(int64_t)(b + 64) * P.pstride + col];
      s3 += sc.part[(int64_t)(b + 96) * P.pstride + col];
    }
    for (; b < (int)gridDim.x; b += 32) s0 += sc.part[(int64_t)b * P.pstride + col];
    double s = warp_sum((s0 + s1) + (s2 + s3));
    if (lane == 0) {
      if (j == c) sc.step->xx = s;
      else sc.g[j] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// Step A (one CTA): t = L^{-1} g, ell = N^T t (= Phi^T x), Pythagorean p,
// dependent test, restart / reject branch (basis.py:112-139); y = t - N ell and
// gt = G^{-1} g = L^{-T} t for the residual pass.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_step_a(StateView src, Scratch sc, IsvdParams P) {
  __shared__ double red[32];
  __shared__ int s_mode;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const IsvdHdr h = *src.hdr;
  IsvdStep* st = sc.step;
  const double xx = st->xx;
  if (threadIdx.x == 0) {
    int mode;
    st->restart = 0;
    st->write_slot = -1;
    st->c_dot = 0;
    st->norm = sqrt(xx);
    if (h.status != 0 || !isfinite(xx)) {
      mode = M_ERROR;
    } else {
      const bool at_cap = P.r_max >= 0 && h.r >= P.r_max;
      if (h.r == 0 || (at_cap && P.cap_mode == 0)) {
        st->restart = at_cap ? 1 : 0;
        if (sqrt(xx) > P.tol_svd) {
          mode = M_RESTART_ACCEPT;
          st->write_slot = h.base + h.c;
          st->c_dot = 0;
        } else {
          mode = M_REJECT;
        }
      } else {
        mode = -1;  // decided below
      }
    }
    s_mode = mode;
  }
  __syncthreads();
  if (s_mode != -1) {
    if (threadIdx.x == 0) st->mode = s_mode;
    return;
  }
  const int r = h.r, c = h.c;
  double* t = sc.tmp;
  cta_lower_mv(src.Li, src.ldl, c, sc.g, t);  // t = L^{-1} g
  __syncthreads();
  // ell_i = sum_j N[j, i] t[j]
  for (int i = wid; i < r; i += nw) {
    const double* ni = src.N + (int64_t)i * src.ldn;
    double s = 0.0;
    for (int j = lane; j < c; j += 32) s = fma(ni[j], t[j], s);
    s = warp_sum(s);
    if (lane == 0) sc.ell[i] = s;
  }
  __syncthreads();
  double part = 0.0;
  for (int i = threadIdx.x; i < r; i += blockDim.x) part = fma(sc.ell[i], sc.ell[i], part);
  const double ll = block_sum(part, red);
  const double p_sq = xx - ll;
  const double p = (p_sq > 0.0) ? sqrt(p_sq) : 0.0;
  const bool dep = (p < P.tol_svd) || (p == 0.0) || ((int64_t)r >= P.n);
  if (threadIdx.x == 0) {
    st->p = p;
    st->p_sq = p_sq;
    st->mode = dep ? M_NORMAL_DEP : M_NORMAL_INDEP;
    if (!dep) {
      st->write_slot = h.base + c;
      st->c_dot = c;
    }
  }
  if (!dep) {
    // y = t - N ell: the in-span part of x - Phi ell in Q_U coordinates
    for (int j = threadIdx.x; j < c; j += blockDim.x) {
      double s = t[j];
      for (int i = 0; i < r; ++i) s = fma(-src.N[(int64_t)i * src.ldn + j], sc.ell[i], s);
      sc.y[j] = s;
    }
    cta_lower_t_mv(src.Li, src.ldl, c, t, sc.gt);  // gt = L^{-T} t = G^{-1} g
  }
}

// ---------------------------------------------------------------------------
// Residual pass: r1 = x - U[:, base:base+c_dot] gt written to U[:, slot];
// e = U[:, ...]^T r1 and rho2 = r1.r1.  Two phases per 64-row tile through
// shared memory (row dots, then column dots against the fresh residual).
// ---------------------------------------------------------------------------
// phase 0: r1 = x - U gt (gt = G^{-1} U^T x);  phase 1 (DGKS re-orthogonalisation,
// only when step B1 asked for it): r2 = r1 - U h in place on the slot column.
template <int MAXJ>
__global__ void __launch_bounds__(kPassThreads) k_resid(double* U, const double* xin,
                                                         StateView src, Scratch sc, IsvdParams P, int phase) {
  extern __shared__ double smem[];
  __shared__ int s_last;
  __shared__ double red[8];
  const IsvdStep* st = sc.step;
  const int mode = st->mode;
  if (phase == 0 && mode != M_NORMAL_INDEP && mode != M_RESTART_ACCEPT) return;
  if (phase == 1 && !(mode == M_NORMAL_INDEP && st->reorth)) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int cd = st->c_dot, slot = st->write_slot, base = src.hdr->base;
  const double* x = (phase == 0) ? xin : U + (int64_t)slot * P.ldu;
  const double* coef = (phase == 0) ? sc.gt : sc.h;
  if (P.prof && blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd(P.prof + 1, 8ull * (unsigned long long)P.n * (unsigned long long)(cd + 2));  // U, x; r1 out
  double* tile = smem;                            // cd x 64 (column-major, 64 rows)
  double* gts = tile + (int64_t)P.ccap * kTileRows;  // ccap (rounded to even: keeps rs 16B-aligned)
  double* xs = gts + ((P.ccap + 1) & ~1);         // 64
  double* rs = xs + kTileRows;                    // 64
  double* pp = rs + kTileRows;                    // 4 x 64 partial row dots
  for (int j = threadIdx.x; j < cd; j += blockDim.x) gts[j] = coef[j];
  const int64_t ntiles = P.ldu / kTileRows;
  const int64_t per = ceil_div(ntiles, gridDim.x);
  const int64_t t0 = blockIdx.x * per;
  const int64_t t1 = min(ntiles, t0 + per);
  double acc[MAXJ];
#pragma unroll
  for (int q = 0; q < MAXJ; ++q) acc[q] = 0.0;
  double rr = 0.0;
  for (int64_t t = t0; t < t1; ++t) {
    const int64_t row0 = t * kTileRows;
    __syncthreads();  // previous tile fully consumed
#pragma unroll
    for (int q = 0; q < MAXJ; ++q) {
      const int j = wid + 8 * q;
      if (j < cd) {
        const double2 u = __ldg(reinterpret_cast<const double2*>(U + (int64_t)(base + j) * P.ldu + row0 + 2 * lane));
        reinterpret_cast<double2*>(tile + (int64_t)j * kTileRows)[lane] = u;
      }
    }
    if (threadIdx.x < kTileRows) {
      const int64_t row = row0 + threadIdx.x;
      xs[threadIdx.x] = (row < P.n) ? x[row] : 0.0;
    }
    __syncthreads();
    {
      const int rrow = threadIdx.x & (kTileRows - 1), quarter = threadIdx.x >> 6;
      double s = 0.0;
      for (int j = quarter; j < cd; j += 4) s = fma(tile[(int64_t)j * kTileRows + rrow], gts[j], s);
      pp[quarter * kTileRows + rrow] = s;
    }
    __syncthreads();
    if (threadIdx.x < kTileRows) {
      const int i = threadIdx.x;
      const double dot = (pp[i] + pp[kTileRows + i]) + (pp[2 * kTileRows + i] + pp[3 * kTileRows + i]);
      const double r1 = (row0 + i < P.n) ? xs[i] - dot : 0.0;
      rs[i] = r1;
      U[(int64_t)slot * P.ldu + row0 + i] = r1;
      rr = fma(r1, r1, rr);
    }
    __syncthreads();
    const double2 r2 = reinterpret_cast<const double2*>(rs)[lane];
#pragma unroll
    for (int q = 0; q < MAXJ; ++q) {
      const int j = wid + 8 * q;
      if (j < cd) {
        const double2 u = reinterpret_cast<const double2*>(tile + (int64_t)j * kTileRows)[lane];
        acc[q] = fma(u.y, r2.y, fma(u.x, r2.x, acc[q]));
      }
    }
  }
  double* mypart = sc.part + (int64_t)blockIdx.x * P.pstride;
#pragma unroll
  for (int q = 0; q < MAXJ; ++q) {
    const int j = wid + 8 * q;
    const double v = warp_sum(acc[q]);
    if (lane == 0 && j < cd) mypart[j] = v;
  }
  const double rtot = block_sum(rr, red);
  if (threadIdx.x == 0) mypart[P.ccap] = rtot;
  if (!last_cta_arrives(sc.counter, &s_last)) return;
  for (int j = wid; j <= cd; j += 8) {
    const int col = (j == cd) ? P.ccap : j;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int b = lane;
    for (; b + 96 < (int)gridDim.x; b += 128) {
      s0 += sc.part[(int64_t)b * P.pstride + col];
      s1 += sc.part[(int64_t)(b + 32) * P.pstride + col];
      s2 += sc.part[(int64_t)(b + 64) * P.pstride + col];
      s3 += sc.part[(int64_t)(b + 96) * P.pstride + col];
    }
    for (; b < (int)gridDim.x; b += 32) s0 += sc.part[(int64_t)b * P.pstride + col];
    double s = warp_sum((s0 + s1) + (s2 + s3));
    if (lane == 0) {
      if (j == cd) sc.step->rho2 = s;
      else sc.e[j] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// Step B (one CTA, 1024 threads): everything in small space.
//   * extend the Cholesky factor of G with the appended column (or fold an
//     in-span residual back into U's existing columns)
//   * bordered core Q = [[diag(sigma), ell], [0, p]] (basis.py:141-144) and its
//     SVD by one-sided Jacobi on Q^T (accumulated rotations give W_bar)
//   * sort descending + sign rule (linalg.py:31-38, 53)
//   * W' = [W w_j] W_bar  (basis.py:150-158), truncation (basis.py:160-168)
//   * drift |phi_0 . phi_last| = |(L^T w_0) . (L^T w_last)|, and on drift the
//     small-space QR replacing linalg.qr(phi) (basis.py:170-174)
// ---------------------------------------------------------------------------
constexpr double kFoldTau = 1e-3;  // append r1 only if its out-of-span part is >= tau |r1|

// ---------------------------------------------------------------------------
// Step B1 (one CTA): decide how the new direction enters U.  l = L^{-1} e,
// lambda^2 = |r1|^2 - |l|^2 is the squared out-of-span part of r1 in the
// G-metric.  Append r1 if lambda >= tau |r1|; otherwise (r1 is mostly
// rounding noise inside span(U)) request one more classical Gram-Schmidt pass
// (DGKS) when U does not yet span R^n.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_step_b1(StateView src, Scratch sc, IsvdParams P) {
  __shared__ double red[32];
  IsvdStep* st = sc.step;
  const int wid = threadIdx.x >> 5;
  const int c = src.hdr->c;
  for (int j = threadIdx.x; j < c; j += blockDim.x) sc.h[j] = 0.0;
  if (st->mode != M_NORMAL_INDEP) {
    if (threadIdx.x == 0) { st->reorth = 0; st->append = 0; }
    return;
  }
  cta_lower_mv(src.Li, src.ldl, c, sc.e, sc.lvec);
  __syncthreads();
  for (int j = threadIdx.x; j < c; j += blockDim.x) sc.l1[j] = sc.lvec[j];
  double part = 0.0;
  for (int j = threadIdx.x; j < c; j += blockDim.x) part = fma(sc.lvec[j], sc.lvec[j], part);
  const double ll = block_sum(part, red);
  const double rho2 = st->rho2;
  const double lam2 = rho2 - ll;
  const bool app = (lam2 > kFoldTau * kFoldTau * rho2) && (rho2 > 0.0);
  const bool reorth = !app && ((int64_t)c < P.n) && (st->write_slot < P.ccap);
  __syncthreads();
  if (reorth) cta_lower_t_mv(src.Li, src.ldl, c, sc.lvec, sc.h);
  if (threadIdx.x == 0) {
    st->append = app ? 1 : 0;
    st->reorth = reorth ? 1 : 0;
  }
}

__global__ void __launch_bounds__(kSmallThreads) k_step_b(StateView src, StateView dst, Scratch sc, IsvdParams P,
                                                 int use_smem) {
  extern __shared__ double smem[];
  __shared__ double red[32];
  __shared__ double s_misc[4];
  __shared__ int s_int[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const IsvdHdr h = *src.hdr;
  IsvdStep* st = sc.step;
  const int mode = st->mode;
  IsvdHdr o = h;
  o.flags = 0;
  o.p = 0.0;
  o.drift = 0.0;
  o.xnorm = st->norm;
  if (mode == M_ERROR) {
    if (threadIdx.x == 0) {
      o.status = 1;
      o.flags = F_ERROR;
      *dst.hdr = o;
      st->m = 0;
      st->mkeep = -1;
    }
    return;
  }
  if (mode == M_REJECT || mode == M_RESTART_ACCEPT) {
    if (threadIdx.x == 0) {
      if (st->restart) { o.n_restarts += 1; o.flags |= F_RESTART; }
      if (mode == M_REJECT) {
        o.r = 0;
        o.c = 0;
        o.base = h.base + h.c;
        o.n_rejected += 1;
        o.flags |= F_REJECTED;
        st->mkeep = 0;
      } else {
        o.r = 1;
        o.c = 1;
        o.base = st->write_slot;
        dst.L[0] = sqrt(st->rho2);
        dst.Li[0] = 1.0 / dst.L[0];
        dst.N[0] = dst.L[0] / st->norm;  // Phi = x / ||x|| = U W, W = 1/||x||, N = L W
        dst.sigma[0] = st->norm;
        st->mkeep = 1;
      }
      st->m = 0;
      *dst.hdr = o;
    }
    return;
  }
  STROM_TPROBE(P, 0);
  bool dep = (mode == M_NORMAL_DEP);
  const int r = h.r, c = h.c, m = r + 1;
  const double p = st->p;
  o.p = p;
  o.p_sq = st->p_sq;
  // ---- 1. how the new direction enters U (see k_step_b1) --------------------
  //   append: U' = [U r], L' = [[L, 0], [l^T, lambda]]
  //   fold:   r is (numerically) in span(U) and U has a spare direction
  //   demote: r is in span(U) to working precision and U has none -> dependent
  int cn = c;
  int action = 0;  // 0 none (dependent), 1 append, 2 fold
  double* lvec = sc.lvec;
  if (!dep) {
    if (st->reorth) {  // second pass done: recompute l, lambda from (e2, |r2|^2)
      cta_lower_mv(src.Li, src.ldl, c, sc.e, lvec);
      __syncthreads();
    }
    double part = 0.0;
    for (int j = threadIdx.x; j < c; j += blockDim.x) part = fma(lvec[j], lvec[j], part);
    const double ll = block_sum(part, red);
    const double rho2 = st->rho2;
    const double lam2 = rho2 - ll;
    bool app;
    // after the second pass r2 is kept whenever it carries a genuine out-of-span
    // direction, however small: the reference appends j = (x - Phi ell)/p even
    // when it is pure rounding noise (basis.py:155-156)
    if (st->reorth) app = (lam2 > 0.25 * rho2) && (rho2 > 0.0);
    else app = st->append != 0;
    app = app && (st->write_slot < P.ccap) && ((int64_t)c < P.n);
    if (threadIdx.x == 0) s_misc[0] = app ? sqrt(lam2) : 0.0;
    if (app) action = 1;
    else if (c >= r + 1) action = 2;
    else { action = 0; dep = true; }
    __syncthreads();
    // append: u = L^{-T} l for the new row of L^{-1}
    if (action == 1) cta_lower_t_mv(src.Li, src.ldl, c, lvec, sc.tmp);
    __syncthreads();
    if (action == 1) cn = c + 1;
  }
  const bool appended = (action == 1);
  // copy L and L^{-1} (lower) into dst, extended by the new row when appended
  for (int j = wid; j < cn; j += nw) {
    const double* ls = src.L + (int64_t)j * src.ldl;
    const double* lis = src.Li + (int64_t)j * src.ldl;
    double* ld_ = dst.L + (int64_t)j * dst.ldl;
    double* lid = dst.Li + (int64_t)j * dst.ldl;
    for (int i = lane; i < cn; i += 32) {
      double v = 0.0, vi = 0.0;
      if (i < c && j < c) {
        if (i >= j) { v = ls[i]; vi = lis[i]; }
      } else if (i == c && j < c) {
        v = lvec[j];
        vi = -sc.tmp[j] / s_misc[0];
      } else if (i == c && j == c) {
        v = s_misc[0];
        vi = 1.0 / s_misc[0];
      }
      ld_[i] = v;
      lid[i] = vi;
    }
  }
  // new N column for j = (x - Phi ell)/p in Q_U coordinates (length cn):
  //   x - Phi ell = Q_U (t - N ell + l_1 [+ l_2]) + lambda q   (q the appended direction)
  // (the fold drops the rounding-level out-of-span part; l_2 only after the DGKS pass)
  double* wj = sc.work + 3 * (int64_t)P.work_stride;
  if (!dep) {
    const bool two = st->reorth != 0;
    for (int a = threadIdx.x; a < cn; a += blockDim.x) {
      double v;
      if (a < c) {
        v = sc.y[a] + sc.l1[a];
        if (two) v += lvec[a];
        v /= p;
      } else {
        v = s_misc[0] / p;
      }
      wj[a] = v;
    }
  }
  STROM_TPROBE(P, 1);
  // ---- shared-memory plan (global fallback when it does not fit) ----------
  //   WS m^2 | Wt m^2 | Vt m^2 | core work 16 ms | WB ccap x m (staged N_b, later QR's M)
  const int64_t ms = P.work_stride;
  double* base = use_smem ? smem : sc.work + 4 * ms;
  double* WS = base;                      // sorted, signed W_bar (m x m)
  double* Wt = WS + (int64_t)m * m;       // vectors by slot, later W^T W
  double* Vt = Wt + (int64_t)m * m;       // vectors by slot, later the polished W_bar
  double* cb = Vt + (int64_t)m * m;
  double* WB = cb + 16 * ms;              // N_b = [[N, n_j]] (cn x m, ld ccap)
  double* svs = cb + 14 * ms;             // m sorted singular values
  CoreSvdWork cw;
  cw.d = cb; cw.z = cb + ms; cw.zh = cb + 2 * ms; cw.mu = cb + 3 * ms; cw.sv = cb + 4 * ms;
  cw.rc = cb + 5 * ms; cw.rs = cb + 6 * ms;
  {
    int* ib = reinterpret_cast<int*>(cb + 7 * ms);
    cw.org = ib; cw.kset = ib + ms; cw.defl = ib + 2 * ms; cw.ra = ib + 3 * ms; cw.rb = ib + 4 * ms;
    cw.perm = ib + 5 * ms; cw.cnt = ib + 6 * ms;
  }
  // stage N_b: columns 0..r-1 = N (c rows; the appended row is 0), column r = n_j
  __syncthreads();  // w_j complete
  if (P.tprobe && threadIdx.x == 0) P.tprobe[7] = use_smem;
  for (int b = wid; b < m; b += nw) {
    const double* ns = src.N + (int64_t)b * src.ldn;
    double* wb = WB + b * P.ccap;
    for (int a = lane; a < cn; a += 32) {
      double v;
      if (b < r) v = (a < c) ? ns[a] : 0.0;
      else v = dep ? 0.0 : wj[a];
      wb[a] = v;
    }
  }
  // ---- 2. the bordered core and its SVD (rank-one secular solver) ----------
  core_svd_secular(src.sigma, sc.ell, dep ? 0.0 : p, r, cw, Wt, Vt, svs, WS, sc.vbar, red,
                   P.tprobe ? P.tprobe + 8 : nullptr, P.tprobe ? P.tprobe + 300 : nullptr);
  STROM_TPROBE(P, 2);
  // (no orthogonality polish needed: the Gu-Eisenstat vectors are orthogonal to
  // working precision, unlike accumulated Jacobi rotations)
  STROM_TPROBE(P, 3);
  // ---- 3. truncation (basis.py:160-168) ------------------------------------
  int mk = dep ? r : m;
  bool trunc = false;
  if (mk > 0 && svs[mk - 1] < P.tol_sv) { mk -= 1; trunc = true; }
  if (P.r_max >= 0 && mk > P.r_max) { mk = P.r_max; trunc = true; }
  // ---- 4. N' = N_b W_bar[:, :mk]  (basis.py:150-158 in Q_U coordinates) ---
  {
    const int kdim = dep ? r : m;
    cta_gemm_dmma(cn, mk, kdim, WB, 1, P.ccap, WS, 1, m,
                  [&](int a, int k, double v) { dst.N[(int64_t)k * dst.ldn + a] = v; });
  }
  for (int k = threadIdx.x; k < mk; k += blockDim.x) dst.sigma[k] = svs[k];
  __syncthreads();
  STROM_TPROBE(P, 4);
  // ---- 5. drift test and small-space QR (basis.py:170-174) -----------------
  bool did_qr = false;
  double drift = 0.0;
  if (mk > 1) {
    // phi_0 . phi_last = N_0 . N_last (Q_U is orthonormal)
    double part = 0.0;
    for (int a = threadIdx.x; a < cn; a += blockDim.x)
      part = fma(dst.N[a], dst.N[(int64_t)(mk - 1) * dst.ldn + a], part);
    drift = fabs(block_sum(part, red));
    const double thr = fmin(P.tol_svd, 2.220446049250313e-16 * (double)P.n);
    STROM_TPROBE(P, 5);
    if (drift > thr) {
      did_qr = true;
      // linalg.qr(phi) (basis.py:174): Phi' = Q_U N' and Q_U is orthonormal, so
      // the positive-diagonal QR of Phi' is Q_U times that of N'.  CholeskyQR2 on
      // the shared-memory N' (two passes: orthonormal to working precision);
      // an ill-conditioned N' (the reference's non-unit j columns can make it so)
      // takes the Householder path.
      double* M = WB;   // cn x mk, ld cn  (N_b is dead)
      double* Bm = Wt;  // mk x mk Gram, then its Cholesky factor
      bool chol_ok = true;
      for (int k = wid; k < mk; k += nw)
        for (int a = lane; a < cn; a += 32) M[k * cn + a] = dst.N[(int64_t)k * dst.ldn + a];
      __syncthreads();
      for (int pass = 0; pass < 2 && chol_ok; ++pass) {
        cta_gemm_dmma(mk, mk, cn, M, cn, 1, M, 1, cn, [&](int i, int k, double v) { Bm[k * mk + i] = v; });
        __syncthreads();
        const double ratio = cta_cholesky(Bm, mk, mk, nullptr);
        // CholeskyQR loses ~eps cond^2 in the triangular factor: only for
        // well-conditioned N' (Householder otherwise, like the reference)
        if (!(ratio > 1e-2)) { chol_ok = false; break; }
        cta_lower_inverse(Bm, mk, mk, Vt, mk);
        __syncthreads();
        // M <- M R^{-1} = M L_B^{-T}:  (L_B^{-T})(j, k) = Vt(k, j); DMMA into WS
        cta_gemm_dmma(cn, mk, mk, M, 1, cn, Vt, mk, 1,
                      [&](int a, int k, double v) { dst.N[(int64_t)k * dst.ldn + a] = v; });
        __syncthreads();
        for (int k = wid; k < mk; k += nw)
          for (int a = lane; a < cn; a += 32) M[k * cn + a] = dst.N[(int64_t)k * dst.ldn + a];
        __syncthreads();
      }
      if (!chol_ok) {
        for (int k = wid; k < mk; k += nw)
          for (int a = lane; a < cn; a += 32) M[k * cn + a] = dst.N[(int64_t)k * dst.ldn + a];
        __syncthreads();
        cta_householder_qr(M, cn, cn, mk, nullptr, 0, sc.work, sc.work + P.work_stride, red);
      }
      if (P.tprobe && threadIdx.x == 0) P.tprobe[6 + 1] = chol_ok ? 1 : 2;
      for (int k = wid; k < mk; k += nw)
        for (int a = lane; a < cn; a += 32) dst.N[(int64_t)k * dst.ldn + a] = M[k * cn + a];
      __syncthreads();
    }
  }
  STROM_TPROBE(P, 6);
  if (threadIdx.x == 0) {
    o.r = mk;
    o.c = cn;
    o.drift = drift;
    o.n_dependent += dep ? 1 : 0;
    o.n_truncated += trunc ? 1 : 0;
    o.flags = (dep ? F_DEPENDENT : 0) | (trunc ? F_TRUNCATED : 0) | (did_qr ? F_QR : 0) |
              (appended ? F_APPENDED : 0) | ((mode == M_NORMAL_INDEP && !appended) ? F_FOLDED : 0);
    *dst.hdr = o;
    st->m = m;
    st->mkeep = mk;
  }
}

// ---------------------------------------------------------------------------
// V' = [[V, 0], [0, 1]] V_bar[:, :mkeep]  (basis.py:147-158); restart/reject
// produce the fresh e_k column (basis.py:83-91).  Thread per row of V'.
// ---------------------------------------------------------------------------
constexpr int kVCols = 16;
constexpr int kVRows = 64;
__global__ void __launch_bounds__(kVRows) k_vupdate(StateView src, StateView dst, Scratch sc, IsvdParams P) {
  extern __shared__ double vbs[];  // (r+1) x kVCols slice of V_bar
  const IsvdStep* st = sc.step;
  const int mode = st->mode;
  const int64_t k = P.k_new;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int col0 = blockIdx.y * kVCols;
  if (mode == M_ERROR || mode == M_REJECT) return;
  if (mode == M_RESTART_ACCEPT) {
    if (col0 == 0 && i < k) dst.V[i] = (i == k - 1) ? 1.0 : 0.0;
    return;
  }
  const int m = st->m, mk = st->mkeep, r = m - 1;
  if (col0 >= mk) return;
  const double* vb = sc.vbar;
  for (int idx = threadIdx.x; idx < m * kVCols; idx += blockDim.x) {
    const int b = idx % m, q = idx / m, col = col0 + q;
    vbs[q * m + b] = (col < mk) ? vb[(int64_t)col * m + b] : 0.0;
  }
  __syncthreads();
  if (i >= k) return;
  double acc[kVCols];
#pragma unroll
  for (int q = 0; q < kVCols; ++q) acc[q] = 0.0;
  if (i < k - 1) {
    for (int b = 0; b < r; ++b) {
      const double v = src.V[(int64_t)b * src.ldv + i];
#pragma unroll
      for (int q = 0; q < kVCols; ++q) acc[q] = fma(v, vbs[q * m + b], acc[q]);
    }
  } else {
#pragma unroll
    for (int q = 0; q < kVCols; ++q) acc[q] = vbs[q * m + r];
  }
#pragma unroll
  for (int q = 0; q < kVCols; ++q) {
    const int col = col0 + q;
    if (col < mk) dst.V[(int64_t)col * dst.ldv + i] = acc[q];
  }
}

// ---------------------------------------------------------------------------
// Compaction prep (one CTA): L^T W = Q_c R_c;  T = L^{-T} Q_c;  new W = R_c,
// new L = I, c = r, base = 0.  Phi = U W = (U T) R_c exactly.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSmallThreads) k_compact_prep(StateView src, StateView dst, Scratch sc, IsvdParams P,
                                                       int use_smem) {
  extern __shared__ double smem[];
  __shared__ double red[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const IsvdHdr h = *src.hdr;
  const int r = h.r, c = h.c;
  IsvdHdr o = h;
  if (h.status != 0 || r == 0) {
    if (threadIdx.x == 0) {
      if (h.status == 0) { o.c = 0; o.base = 0; }
      *dst.hdr = o;
      sc.step->m = 0;
    }
    return;
  }
  // N = Q_c R_c; U_new = U L^{-T} Q_c (orthonormal), and with L_new = chol of
  // the measured U_new Gram the new coordinates are N_new = L_new^T R_c
  // (k_compact_finish, after the Gram); R_c waits in dst.N.
  double* M = use_smem ? smem : sc.work + 4 * (int64_t)P.work_stride;  // c x r
  for (int64_t idx = threadIdx.x; idx < (int64_t)c * r; idx += blockDim.x) {
    const int i = idx % c, k = idx / c;
    M[idx] = src.N[(int64_t)k * src.ldn + i];
  }
  __syncthreads();
  cta_householder_qr(M, c, c, r, dst.N, dst.ldn, sc.work, sc.work + P.work_stride, red);
  cta_gemm_dmma(c, r, c, src.Li, src.ldl, 1, M, 1, c,
                [&](int a, int k, double v) { sc.T[(int64_t)k * P.ccap + a] = v; });
  for (int64_t idx = threadIdx.x; idx < (int64_t)r * r; idx += blockDim.x) {
    const int i = idx % r, j = idx / r;
    dst.L[(int64_t)j * dst.ldl + i] = (i == j) ? 1.0 : 0.0;
    dst.Li[(int64_t)j * dst.ldl + i] = (i == j) ? 1.0 : 0.0;
  }
  for (int k = threadIdx.x; k < r; k += blockDim.x) dst.sigma[k] = src.sigma[k];
  if (threadIdx.x == 0) {
    o.c = r;
    o.base = 0;
    *dst.hdr = o;
    sc.step->m = c;  // number of source columns for the GEMM
    sc.step->mkeep = r;
  }
}

// After the compaction Gram: N_new = L_new^T R_c (R_c parked in dst.N).
__global__ void __launch_bounds__(256) k_compact_finish(StateView dst, double* tmp, int ldt) {
  const int r = dst.hdr->r;
  if (dst.hdr->status != 0 || r == 0) return;
  // upper-triangular (L_new^T) times upper-triangular R_c
  for (int64_t idx = threadIdx.x; idx < (int64_t)r * r; idx += blockDim.x) {
    const int i = idx % r, k = idx / r;
    const double* lcol = dst.L + (int64_t)i * dst.ldl;  // column i of L = row i of L^T
    double s = 0.0;
    for (int j = i; j <= k; ++j) s = fma(lcol[j], dst.N[(int64_t)k * dst.ldn + j], s);
    tmp[(int64_t)k * ldt + i] = s;
  }
  __syncthreads();
  for (int64_t idx = threadIdx.x; idx < (int64_t)r * r; idx += blockDim.x) {
    const int i = idx % r, k = idx / r;
    dst.N[(int64_t)k * dst.ldn + i] = tmp[(int64_t)k * ldt + i];
  }
}

// U-coordinates W = L^{-T} N (c x r, ld c) for the export / materialisation.
__global__ void __launch_bounds__(256) k_n_to_w(StateView v, double* w) {
  const int r = v.hdr->r, c = v.hdr->c;
  for (int64_t idx = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; idx < (int64_t)c * r;
       idx += (int64_t)blockDim.x * gridDim.x) {
    const int a = idx % c, k = idx / c;
    const double* lcol = v.Li + (int64_t)a * v.ldl;
    double s = 0.0;
    for (int i = a; i < c; ++i) s = fma(lcol[i], v.N[(int64_t)k * v.ldn + i], s);
    w[(int64_t)k * c + a] = s;
  }
}

// N = L^T W for a state loaded in U-coordinates (W parked in dst.N).
__global__ void __launch_bounds__(256) k_w_to_n(StateView v, double* tmp) {
  const int r = v.hdr->r, c = v.hdr->c;
  for (int64_t idx = threadIdx.x; idx < (int64_t)c * r; idx += blockDim.x) {
    const int i = idx % c, k = idx / c;
    const double* lcol = v.L + (int64_t)i * v.ldl;
    double s = 0.0;
    for (int j = i; j < c; ++j) s = fma(lcol[j], v.N[(int64_t)k * v.ldn + j], s);
    tmp[(int64_t)k * c + i] = s;
  }
  __syncthreads();
  for (int64_t idx = threadIdx.x; idx < (int64_t)c * r; idx += blockDim.x) {
    const int i = idx % c, k = idx / c;
    v.N[(int64_t)k * v.ldn + i] = tmp[(int64_t)k * c + i];
  }
}

// ---------------------------------------------------------------------------
// Tall-skinny GEMM:  out(n x q) = A(n x p) * T(p x q)   (fp64 FMA, register
// blocked 4 rows x 8 cols per thread, T staged through shared memory).
// A column-major (lda, first column a_col0); out column-major (ldo) or
// row-major (ldo = row stride) when out_row_major.  p, q read from device.
// ---------------------------------------------------------------------------
constexpr int kGemmRows = 128;  // rows per CTA tile
constexpr int kGemmKc = 32;     // T chunk (rows of T) per smem stage

__global__ void __launch_bounds__(256) k_tall_gemm(const double* __restrict__ A, int64_t lda,
                                                   const int32_t* a_col0_dev, int a_col0_add,
                                                   const double* __restrict__ T, int64_t ldt,
                                                   const int32_t* p_dev, const int32_t* q_dev,
                                                   int q_max, double* __restrict__ out, int64_t ldo,
                                                   int out_row_major, int64_t n, int64_t nrows_pad) {
  extern __shared__ double ts[];  // kGemmKc x q_max
  const int p = *p_dev, q = *q_dev;
  const int col0 = (a_col0_dev ? *a_col0_dev : 0) + a_col0_add;
  if (q <= 0) return;
  const int tx = threadIdx.x & 31;   // row lane: rows tx, tx+32, tx+64, tx+96
  const int ty = threadIdx.x >> 5;   // column group: cols ty*8 .. ty*8+7 (+64 per pass)
  for (int64_t rt = blockIdx.x; rt * kGemmRows < nrows_pad; rt += gridDim.x) {
    const int64_t r0 = rt * kGemmRows;
    for (int cb = 0; cb < q; cb += 64) {
      double acc[4][8];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
      for (int k0 = 0; k0 < p; k0 += kGemmKc) {
        const int kc = min(kGemmKc, p - k0);
        __syncthreads();
        for (int idx = threadIdx.x; idx < kGemmKc * 64; idx += blockDim.x) {
          const int kk = idx % kGemmKc, cc = idx / kGemmKc;
          const int col = cb + cc;
          ts[cc * kGemmKc + kk] = (kk < kc && col < q) ? T[(int64_t)col * ldt + k0 + kk] : 0.0;
        }
        __syncthreads();
        for (int kk = 0; kk < kc; ++kk) {
          const double* acol = A + (int64_t)(col0 + k0 + kk) * lda + r0;
          double av[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) av[a] = __ldg(acol + tx + 32 * a);
#pragma unroll
          for (int b = 0; b < 8; ++b) {
            const double t = ts[(ty * 8 + b) * kGemmKc + kk];
#pragma unroll
            for (int a = 0; a < 4; ++a) acc[a][b] = fma(av[a], t, acc[a][b]);
          }
        }
      }
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const int col = cb + ty * 8 + b;
        if (col >= q) continue;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const int64_t row = r0 + tx + 32 * a;
          if (out_row_major) {
            if (row < n) out[row * ldo + col] = acc[a][b];
          } else if (row < nrows_pad) {
            out[(int64_t)col * ldo + row] = acc[a][b];
          }
        }
      }
    }
  }
}

}  // namespace strom
