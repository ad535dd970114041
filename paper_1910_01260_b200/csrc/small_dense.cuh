// Single-CTA dense fp64 routines for the small matrices of the hot path:
// the bordered (r+1)^2 iSVD core, the temporal snapshot blocks, the small-space
// QR that replaces the reference's tall Householder QR, triangular solves.
//
// Every routine is called by ALL threads of the CTA (they contain
// __syncthreads) and works on column-major arrays in shared or global memory.
#pragma once

#include "common.cuh"
#include "dmma.cuh"

namespace strom {

// ---------------------------------------------------------------------------
// One-sided (Hestenes) Jacobi on the columns of A (rows x cols, col-major):
// A <- A J, V <- V J until all column pairs are orthogonal to eps*sqrt(rows).
// Parallel round-robin ordering: each round has ceil(cols/2) disjoint pairs,
// one warp per pair (warps loop over pairs).  V may be nullptr.
// `flag` is a shared int used for the convergence vote.
// Returns the number of sweeps performed.
// ---------------------------------------------------------------------------
__device__ inline int cta_jacobi(double* A, int lda, int rows, int cols, double* V, int ldv,
                                 int vrows, int* flag, int max_sweeps = 40) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (cols < 2) return 0;
  const int ne = cols + (cols & 1);  // even number of players (one dummy if odd)
  const int npairs = ne / 2;
  const double tol = 2.220446049250313e-16 * sqrt((double)rows);
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int rnd = 0; rnd < ne - 1; ++rnd) {
      for (int pk = wid; pk < npairs; pk += nw) {
        int a, b;
        if (pk == 0) {
          a = rnd;
          b = ne - 1;
        } else {
          a = (rnd + pk) % (ne - 1);
          b = (rnd - pk + (ne - 1)) % (ne - 1);
        }
        if (a > b) { int t = a; a = b; b = t; }
        if (b >= cols) continue;  // dummy player
        double* ca = A + (int64_t)a * lda;
        double* cb = A + (int64_t)b * lda;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < rows; i += 32) {
          const double x = ca[i], y = cb[i];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga = fma(x, y, ga);
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (al == 0.0 || be == 0.0) continue;
        if (fabs(ga) <= tol * sqrt(al) * sqrt(be)) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
        const double c = 1.0 / sqrt(fma(t, t, 1.0));
        const double s = c * t;
        for (int i = lane; i < rows; i += 32) {
          const double x = ca[i], y = cb[i];
          ca[i] = c * x - s * y;
          cb[i] = s * x + c * y;
        }
        if (V) {
          double* va = V + (int64_t)a * ldv;
          double* vb = V + (int64_t)b * ldv;
          for (int i = lane; i < vrows; i += 32) {
            const double x = va[i], y = vb[i];
            va[i] = c * x - s * y;
            vb[i] = s * x + c * y;
          }
        }
        if (lane == 0) *flag = 1;
      }
      __syncthreads();
    }
    const int any = *flag;
    __syncthreads();
    if (!any) break;
  }
  return sweep;
}

// Column norms of A into out[cols] (one warp per column).
__device__ inline void cta_col_norms(const double* A, int lda, int rows, int cols, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = wid; j < cols; j += nw) {
    const double* cj = A + (int64_t)j * lda;
    double s = 0.0;
    for (int i = lane; i < rows; i += 32) s = fma(cj[i], cj[i], s);
    s = warp_sum(s);
    if (lane == 0) out[j] = sqrt(s);
  }
  __syncthreads();
}

// Stable descending argsort of vals[0..n) into perm (n <= blockDim.x).
// Ties keep the lower index first (rank = #greater + #equal-with-lower-index).
__device__ inline void cta_argsort_desc(const double* vals, int n, int* perm) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = vals[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double u = vals[j];
      rank += (u > v) || (u == v && j < i);
    }
    perm[rank] = i;
  }
  __syncthreads();
}

// Index of the largest |w[i]| (first on ties), computed by one warp.
__device__ inline int warp_argmax_abs(const double* w, int n) {
  const int lane = threadIdx.x & 31;
  double best = -1.0;
  int bi = 0x7fffffff;
  for (int i = lane; i < n; i += 32) {
    const double a = fabs(w[i]);
    if (a > best) { best = a; bi = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
  return bi;
}

// ---------------------------------------------------------------------------
// Householder QR of M (rows x cols, rows >= cols, col-major, ld), overwritten
// by the explicit thin Q with diag(R) >= 0 (zero pivots count as +1), as
// linalg.qr does (linalg.py:60-72).  If R != nullptr the upper triangle of R
// (ldr) receives the matching R.  tau/beta: shared scratch of `cols` doubles.
// ---------------------------------------------------------------------------
__device__ inline void cta_householder_qr(double* M, int ld, int rows, int cols, double* R, int ldr,
                                          double* tau, double* beta, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = 0; j < cols; ++j) {
    double* x = M + (int64_t)j * ld;
    double s = 0.0;
    for (int i = j + 1 + threadIdx.x; i < rows; i += blockDim.x) s = fma(x[i], x[i], s);
    s = block_sum(s, red);
    const double x0 = x[j];
    __syncthreads();
    const double nrm = sqrt(fma(x0, x0, s));
    double bt, tj, scal;
    if (s == 0.0) {  // already upper-triangular in this column: H = I
      bt = x0;
      tj = 0.0;
      scal = 0.0;
    } else {
      bt = (x0 >= 0.0) ? -nrm : nrm;
      tj = (bt - x0) / bt;
      scal = 1.0 / (x0 - bt);
    }
    for (int i = j + 1 + threadIdx.x; i < rows; i += blockDim.x) x[i] *= scal;
    if (threadIdx.x == 0) {
      tau[j] = tj;
      beta[j] = bt;
      x[j] = 1.0;  // implicit unit head of v
    }
    __syncthreads();
    if (tj != 0.0) {
      for (int k = j + 1 + wid; k < cols; k += nw) {
        double* y = M + (int64_t)k * ld;
        double d = 0.0;
        for (int i = j + lane; i < rows; i += 32) d = fma(x[i], y[i], d);
        d = warp_sum(d) * tj;
        for (int i = j + lane; i < rows; i += 32) y[i] = fma(-d, x[i], y[i]);
      }
    }
    __syncthreads();
  }
  // R (before sign fix) lives in the strict upper triangle of M plus beta.
  if (R) {
    for (int idx = threadIdx.x; idx < cols * cols; idx += blockDim.x) {
      const int i = idx % cols, k = idx / cols;
      double v = 0.0;
      if (i < k) v = M[(int64_t)k * ld + i];
      else if (i == k) v = beta[k];
      R[(int64_t)k * ldr + i] = v;
    }
  }
  __syncthreads();
  // Form Q = H_0 ... H_{cols-1} [I; 0] by backward accumulation, in place:
  // column j's Householder vector is consumed before column j becomes Q's.
  for (int j = cols - 1; j >= 0; --j) {
    double* v = M + (int64_t)j * ld;  // v[j] == 1, v[j+1..] stored, v[<j] = R part
    const double tj = tau[j];
    // columns k > j already hold Q entries (rows >= j+1 ... ), apply H_j to them
    for (int k = j + 1 + wid; k < cols; k += nw) {
      double* y = M + (int64_t)k * ld;
      double d = 0.0;
      for (int i = j + 1 + lane; i < rows; i += 32) d = fma(v[i], y[i], d);
      // y[j] is 0 in [I;0] history (row j of columns k>j before applying H_j)
      d = warp_sum(d) * tj;
      for (int i = j + 1 + lane; i < rows; i += 32) y[i] = fma(-d, v[i], y[i]);
      if (lane == 0) y[j] = -d;
    }
    __syncthreads();
    // column j itself: H_j e_j = e_j - tau v  (v_j = 1)
    for (int i = threadIdx.x; i < rows; i += blockDim.x) {
      if (i < j) v[i] = 0.0;
      else if (i == j) v[i] = 1.0 - tj;
      else v[i] = -tj * v[i];
    }
    __syncthreads();
  }
  // diag(R) >= 0: flip Q column j (and R row j) where beta_j < 0.
  for (int idx = threadIdx.x; idx < rows * cols; idx += blockDim.x) {
    const int i = idx % rows, j = idx / rows;
    if (beta[j] < 0.0) M[(int64_t)j * ld + i] = -M[(int64_t)j * ld + i];
  }
  if (R) {
    for (int idx = threadIdx.x; idx < cols * cols; idx += blockDim.x) {
      const int i = idx % cols, k = idx / cols;
      if (beta[i] < 0.0) R[(int64_t)k * ldr + i] = -R[(int64_t)k * ldr + i];
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Warp-level triangular solves with a lower-triangular L (n x n, col-major).
// x holds b on entry and the solution on exit (global or shared); executed by
// ONE warp.  n is small (<= a few hundred).
// ---------------------------------------------------------------------------
__device__ inline void warp_lower_solve(const double* L, int ld, int n, double* x) {
  const int lane = threadIdx.x & 31;
  for (int j = 0; j < n; ++j) {
    double xj = 0.0;
    if (lane == 0) xj = x[j] / L[(int64_t)j * ld + j];
    xj = __shfl_sync(0xffffffffu, xj, 0);
    if (lane == 0) x[j] = xj;
    for (int i = j + 1 + lane; i < n; i += 32) x[i] = fma(-L[(int64_t)j * ld + i], xj, x[i]);
    __syncwarp();
  }
}

// Solve L^T x = b (backward), one warp.
__device__ inline void warp_lower_t_solve(const double* L, int ld, int n, double* x) {
  const int lane = threadIdx.x & 31;
  for (int j = n - 1; j >= 0; --j) {
    // x_j = (b_j - sum_{i>j} L[i,j] x_i) / L[j,j]
    double s = 0.0;
    for (int i = j + 1 + lane; i < n; i += 32) s = fma(L[(int64_t)j * ld + i], x[i], s);
    s = warp_sum(s);
    if (lane == 0) x[j] = (x[j] - s) / L[(int64_t)j * ld + j];
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Register-blocked block-wide GEMM for the small operands (shared or global):
//   C(i, j) = sum_k A(i, k) B(k, j),  A(i, k) = A[i*asi + k*ask],  B(k, j) = B[k*bsk + j*bsj]
// each thread owns a 4 x 4 tile (0.5 operand loads per FMA).  `store(i, j, v)`
// receives the results.  No synchronisation inside.
// ---------------------------------------------------------------------------
template <class Store>
__device__ inline void cta_gemm44(int M, int N, int K, const double* A, int64_t asi, int64_t ask, const double* B,
                                  int64_t bsk, int64_t bsj, Store store) {
  const int nbm = (M + 3) >> 2, nbn = (N + 3) >> 2;
  for (int blk = threadIdx.x; blk < nbm * nbn; blk += blockDim.x) {
    const int i0 = (blk % nbm) << 2, j0 = (blk / nbm) << 2;
    const double* ap[4];
    const double* bp[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      ap[q] = A + (int64_t)min(i0 + q, M - 1) * asi;
      bp[q] = B + (int64_t)min(j0 + q, N - 1) * bsj;
    }
    double acc[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int t = 0; t < 4; ++t) acc[q][t] = 0.0;
#pragma unroll 2
    for (int k = 0; k < K; ++k) {
      double a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = ap[q][(int64_t)k * ask];
        b[q] = bp[q][(int64_t)k * bsk];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int t = 0; t < 4; ++t) acc[q][t] = fma(a[q], b[t], acc[q][t]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (i0 + q < M && j0 + t < N) store(i0 + q, j0 + t, acc[q][t]);
  }
}

// ---------------------------------------------------------------------------
// Block-wide GEMM on the fp64 tensor cores (DMMA m8n8k4), same contract as
// cta_gemm44: C(i, j) = sum_k A(i, k) B(k, j) with strided operands (shared or
// global memory), results handed to store(i, j, v).  Each warp owns 8 x 8
// output tiles; operands beyond M/N/K read as zero.  No synchronisation.
// ---------------------------------------------------------------------------
template <class Store>
__device__ inline void cta_gemm_dmma(int M, int N, int K, const double* A, int64_t asi, int64_t ask,
                                     const double* B, int64_t bsk, int64_t bsj, Store store) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int tm = (M + 7) >> 3, tn = (N + 7) >> 3, ks = (K + 3) >> 2;
  for (int tile = wid; tile < tm * tn; tile += nw) {
    const int i0 = (tile % tm) << 3, j0 = (tile / tm) << 3;
    const int ia = i0 + g, jb = j0 + g;
    const bool va = ia < M, vb = jb < N;
    const double* ap = A + (int64_t)(va ? ia : 0) * asi;
    const double* bp = B + (int64_t)(vb ? jb : 0) * bsj;
    double c0 = 0.0, c1 = 0.0;
    for (int kk = 0; kk < ks; ++kk) {
      const int k = (kk << 2) + t;
      const bool vk = k < K;
      const double av = (va && vk) ? ap[(int64_t)k * ask] : 0.0;
      const double bv = (vb && vk) ? bp[(int64_t)k * bsk] : 0.0;
      dmma884(c0, c1, av, bv);
    }
    const int r = i0 + g, c = j0 + 2 * t;
    if (r < M) {
      if (c < N) store(r, c, c0);
      if (c + 1 < N) store(r, c + 1, c1);
    }
  }
}

// The same product with two accumulator tiles per warp (an 8 x 16 output block:
// one A fragment feeds two independent DMMA chains, the k-steps unrolled so the
// fragment loads run ahead).  B200's fp64 tensor rate equals its vector rate
// (~64 FMA/clk/SM), so a one-CTA product is latency work: what matters is
// independent chains in flight.  Every output sums its k-steps in the same
// order as cta_gemm_dmma: identical results.
template <class Store>
__device__ inline void cta_gemm_dmma_n2(int M, int N, int K, const double* A, int64_t asi, int64_t ask,
                                        const double* B, int64_t bsk, int64_t bsj, Store store) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int tm = (M + 7) >> 3, tn = (N + 15) >> 4, ks = (K + 3) >> 2;
  for (int tile = wid; tile < tm * tn; tile += nw) {
    const int i0 = (tile % tm) << 3, j0 = (tile / tm) << 4;
    const int ia = i0 + g, jb0 = j0 + g, jb1 = j0 + 8 + g;
    const bool va = ia < M, vb0 = jb0 < N, vb1 = jb1 < N;
    const double* ap = A + (int64_t)(va ? ia : 0) * asi;
    const double* bp0 = B + (int64_t)(vb0 ? jb0 : 0) * bsj;
    const double* bp1 = B + (int64_t)(vb1 ? jb1 : 0) * bsj;
    double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
#pragma unroll 4
    for (int kk = 0; kk < ks; ++kk) {
      const int k = (kk << 2) + t;
      const bool vk = k < K;
      const double av = (va && vk) ? ap[(int64_t)k * ask] : 0.0;
      const double b0 = (vb0 && vk) ? bp0[(int64_t)k * bsk] : 0.0;
      const double b1 = (vb1 && vk) ? bp1[(int64_t)k * bsk] : 0.0;
      dmma884(c00, c01, av, b0);
      dmma884(c10, c11, av, b1);
    }
    const int r = i0 + g, c = j0 + 2 * t;
    if (r < M) {
      if (c < N) store(r, c, c00);
      if (c + 1 < N) store(r, c + 1, c01);
      if (c + 8 < N) store(r, c + 8, c10);
      if (c + 9 < N) store(r, c + 9, c11);
    }
  }
}

// The same product with an MT x NT block of accumulator tiles per warp (8 MT x 8 NT outputs:
// MT + NT fragment loads feed MT * NT independent DMMA chains per k-step), blocks dealt to
// the warps round-robin.  For the core step's N update (c x r times r x r, c ~ 90, r = 64):
// 4 x 2 tiles per warp make 12-16 blocks, one per warp, eight chains each -- enough to keep
// the fp64 pipe (one DMMA per 16 cycles per sub-partition) busy.  Same k order per output:
// identical results.
template <int MT, int NT, class Store>
__device__ inline void cta_gemm_dmma_blk(int M, int N, int K, const double* A, int64_t asi, int64_t ask,
                                         const double* B, int64_t bsk, int64_t bsj, Store store) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int bm = (M + 8 * MT - 1) / (8 * MT), bn = (N + 8 * NT - 1) / (8 * NT), ks = (K + 3) >> 2;
  for (int blk = wid; blk < bm * bn; blk += nw) {
    const int i0 = (blk % bm) * 8 * MT, j0 = (blk / bm) * 8 * NT;
    const double* ap[MT];
    const double* bp[NT];
    bool va[MT], vb[NT];
#pragma unroll
    for (int x = 0; x < MT; ++x) {
      va[x] = i0 + 8 * x + g < M;
      ap[x] = A + (int64_t)(va[x] ? i0 + 8 * x + g : 0) * asi;
    }
#pragma unroll
    for (int y = 0; y < NT; ++y) {
      vb[y] = j0 + 8 * y + g < N;
      bp[y] = B + (int64_t)(vb[y] ? j0 + 8 * y + g : 0) * bsj;
    }
    double c[MT][NT][2];
#pragma unroll
    for (int x = 0; x < MT; ++x)
#pragma unroll
      for (int y = 0; y < NT; ++y) c[x][y][0] = c[x][y][1] = 0.0;
#pragma unroll 2
    for (int kk = 0; kk < ks; ++kk) {
      const int k = (kk << 2) + t;
      const bool vk = k < K;
      double av[MT], bv[NT];
#pragma unroll
      for (int x = 0; x < MT; ++x) av[x] = (va[x] && vk) ? ap[x][(int64_t)k * ask] : 0.0;
#pragma unroll
      for (int y = 0; y < NT; ++y) bv[y] = (vb[y] && vk) ? bp[y][(int64_t)k * bsk] : 0.0;
#pragma unroll
      for (int x = 0; x < MT; ++x)
#pragma unroll
        for (int y = 0; y < NT; ++y) dmma884(c[x][y][0], c[x][y][1], av[x], bv[y]);
    }
#pragma unroll
    for (int x = 0; x < MT; ++x)
#pragma unroll
      for (int y = 0; y < NT; ++y) {
        const int r = i0 + 8 * x + g, cc = j0 + 8 * y + 2 * t;
        if (r < M) {
          if (cc < N) store(r, cc, c[x][y][0]);
          if (cc + 1 < N) store(r, cc + 1, c[x][y][1]);
        }
      }
  }
}

// ---------------------------------------------------------------------------
// In-place lower Cholesky B = L L^T (n x n, column-major, ld), right-looking,
// block-parallel, two barriers per column.  Returns min/max pivot ratio, or -1
// if a pivot is not positive (uniform across the block).  Zeroes the strict
// upper triangle.
// ---------------------------------------------------------------------------
__device__ inline double cta_cholesky(double* B, int ld, int n, double* /*unused*/) {
  // right-looking with ONE barrier per column: column j's rank-1 update uses the
  // unscaled column (B(i,j) B(k,j) / B(j,j)), and column j is scaled in the
  // next column's phase, when nobody reads it any more
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double pmin = INFINITY, pmax = 0.0;
  double prev_inv = 0.0;
  for (int j = 0; j < n; ++j) {
    __syncthreads();  // column j is final (updated by all earlier columns)
    const double* cj = B + j * ld;
    const double d2 = cj[j];
    if (!(d2 > 0.0)) {
      __syncthreads();
      return -1.0;
    }
    const double rd2 = 1.0 / d2;
    const double inv = rsqrt(d2);
    pmin = fmin(pmin, d2 * inv);
    pmax = fmax(pmax, d2 * inv);
    if (j > 0) {  // scale the previous column (nobody reads it in this phase)
      double* cp = B + (j - 1) * ld;
      for (int i = j - 1 + threadIdx.x; i < n; i += blockDim.x) cp[i] = (i == j - 1) ? 1.0 / prev_inv : cp[i] * prev_inv;
    }
    for (int k = j + 1 + wid; k < n; k += nw) {
      const double ck = cj[k] * rd2;
      double* colk = B + k * ld;
      for (int i = k + lane; i < n; i += 32) colk[i] = fma(-cj[i], ck, colk[i]);
    }
    prev_inv = inv;
  }
  __syncthreads();
  if (n > 0) {
    double* cp = B + (n - 1) * ld;
    if (threadIdx.x == 0) cp[n - 1] = 1.0 / prev_inv;
  }
  for (int k = wid; k < n; k += nw)
    for (int i = lane; i < k; i += 32) B[k * ld + i] = 0.0;
  __syncthreads();
  return pmin / pmax;
}

// ---------------------------------------------------------------------------
// X <- X L^{-T} in place (X: rows x n, column-major ld; L: n x n lower, ld l),
// i.e. X_new R = X with R = L^T upper: forward substitution along each row,
// one thread per row.  The caller synchronises afterwards.
// ---------------------------------------------------------------------------
__device__ inline void cta_rows_times_inv_lt(double* X, int ldx, int rows, const double* L, int ldl, int n,
                                             const double* dinv) {
  // dinv[k] = 1 / L(k, k) (precomputed: no division on the dependency chain)
  for (int a = threadIdx.x; a < rows; a += blockDim.x) {
    for (int k = 0; k < n; ++k) {
      const double* lrow = L + k;  // L(k, j) = L[j * ldl + k]
      double s0 = X[(int64_t)k * ldx + a], s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int j = 0;
      for (; j + 3 < k; j += 4) {
        s0 = fma(-X[(int64_t)j * ldx + a], lrow[(int64_t)j * ldl], s0);
        s1 = fma(-X[(int64_t)(j + 1) * ldx + a], lrow[(int64_t)(j + 1) * ldl], s1);
        s2 = fma(-X[(int64_t)(j + 2) * ldx + a], lrow[(int64_t)(j + 2) * ldl], s2);
        s3 = fma(-X[(int64_t)(j + 3) * ldx + a], lrow[(int64_t)(j + 3) * ldl], s3);
      }
      for (; j < k; ++j) s0 = fma(-X[(int64_t)j * ldx + a], lrow[(int64_t)j * ldl], s0);
      X[(int64_t)k * ldx + a] = ((s0 + s1) + (s2 + s3)) * dinv[k];
    }
  }
}

// ---------------------------------------------------------------------------
// In-place lower Cholesky B = L L^T (n x n, column-major, ld) by ONE warp
// (right-looking; no block barriers).  Returns min/max pivot ratio, or -1 if a
// pivot is not positive.  The strict upper triangle is zeroed.
// ---------------------------------------------------------------------------
__device__ inline double warp_cholesky(double* B, int ld, int n) {
  const int lane = threadIdx.x & 31;
  double pmin = INFINITY, pmax = 0.0;
  bool bad = false;
  for (int j = 0; j < n; ++j) {
    double* cj = B + (int64_t)j * ld;
    const double d2 = cj[j];
    if (!(d2 > 0.0)) { bad = true; break; }
    const double d = sqrt(d2);
    pmin = fmin(pmin, d);
    pmax = fmax(pmax, d);
    const double inv = 1.0 / d;
    __syncwarp();
    if (lane == 0) cj[j] = d;
    for (int i = j + 1 + lane; i < n; i += 32) cj[i] *= inv;
    __syncwarp();
    // trailing update: columns k > j, rows i >= k
    for (int k = j + 1; k < n; ++k) {
      const double ck = cj[k];
      double* colk = B + (int64_t)k * ld;
      for (int i = k + lane; i < n; i += 32) colk[i] = fma(-cj[i], ck, colk[i]);
    }
    __syncwarp();
  }
  for (int j = 0; j < n; ++j)
    for (int i = lane; i < j; i += 32) B[(int64_t)j * ld + i] = 0.0;
  __syncwarp();
  return bad ? -1.0 : pmin / pmax;
}

// ---------------------------------------------------------------------------
// Triangular matrix-vector products with an explicitly stored inverse factor
// (the iSVD keeps L^{-1} next to L so every "solve" on the per-snapshot
// critical path is a parallel matvec instead of a serial substitution).
// Li lower-triangular, column-major (ld).  y must not alias x.  Block-wide;
// the caller synchronises before using y.
// ---------------------------------------------------------------------------
// y[i] = (base ? base[i] : 0) + sgn * sum_j A(i, j) x[j] for i < rows, j < cols
// (A column-major, ld; lower: only j <= i).  Warp w takes columns j = w mod nw,
// lanes take rows (coalesced), and the per-warp partials are reduced in a fixed
// order through `part` (nw * rows doubles of shared memory): deterministic, and
// every load of A is independent (no serial dependence chain through memory).
// rows <= 32 * K.  x must not alias y.  Ends with __syncthreads.
template <int K>
__device__ inline void cta_gemv_cm(const double* A, int ld, int rows, int cols, const double* x, double sgn,
                                   const double* base, double* y, double* part, bool lower) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
#pragma unroll 2
  for (int j = wid; j < cols; j += nw) {  // unrolled: two columns' loads in flight (L2-latency bound)
    const double xj = x[j];
    const double* col = A + (int64_t)j * ld;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int i = lane + 32 * k;
      if (i < rows && (!lower || i >= j)) acc[k] = fma(col[i], xj, acc[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int i = lane + 32 * k;
    if (i < rows) part[wid * rows + i] = acc[k];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < rows; i += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += part[w * rows + i];
    y[i] = (base ? base[i] : 0.0) + sgn * s;
  }
  __syncthreads();
}

// y[j] = sum_i A(i, j) x[i] over i < rows (lower: i >= j), j < cols: one warp
// per column, lanes over rows.  Ends with __syncthreads.
__device__ inline void cta_gemv_t_cm(const double* A, int ld, int rows, int cols, const double* x, double* y,
                                     bool lower) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll 2
  for (int j = wid; j < cols; j += nw) {
    const double* col = A + (int64_t)j * ld;
    double s = 0.0;
#pragma unroll 4
    for (int i = (lower ? j : 0) + lane; i < rows; i += 32) s = fma(col[i], x[i], s);
    s = warp_sum(s);
    if (lane == 0) y[j] = s;
  }
  __syncthreads();
}

// Two right-hand sides at once: y1 = A x1, y2 = A x2 (same contract as
// cta_gemv_cm with sgn = 1, no base; `part` holds 2 * nw * rows doubles).
// x2 may be null (then y2 is not written).
template <int K>
__device__ inline void cta_gemv2_cm(const double* A, int ld, int rows, int cols, const double* x1, const double* x2,
                                    double* y1, double* y2, double* part, bool lower) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double a1[K], a2[K];
#pragma unroll
  for (int k = 0; k < K; ++k) { a1[k] = 0.0; a2[k] = 0.0; }
#pragma unroll 2
  for (int j = wid; j < cols; j += nw) {
    const double u1 = x1[j], u2 = x2 ? x2[j] : 0.0;
    const double* col = A + (int64_t)j * ld;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int i = lane + 32 * k;
      if (i < rows && (!lower || i >= j)) {
        const double v = col[i];
        a1[k] = fma(v, u1, a1[k]);
        a2[k] = fma(v, u2, a2[k]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int i = lane + 32 * k;
    if (i < rows) {
      part[wid * rows + i] = a1[k];
      part[(nw + wid) * rows + i] = a2[k];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < rows; i += blockDim.x) {
    double s1 = 0.0, s2 = 0.0;
    for (int w = 0; w < nw; ++w) {
      s1 += part[w * rows + i];
      s2 += part[(nw + w) * rows + i];
    }
    y1[i] = s1;
    if (y2) y2[i] = s2;
  }
  __syncthreads();
}

// y1[j] = sum_i A(i, j) x1[i], y2[j] = sum_i A(i, j) x2[i] (lower: i >= j); warp per column.
__device__ inline void cta_gemv2_t_cm(const double* A, int ld, int rows, int cols, const double* x1, const double* x2,
                                      double* y1, double* y2, bool lower) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll 2
  for (int j = wid; j < cols; j += nw) {
    const double* col = A + (int64_t)j * ld;
    double s1 = 0.0, s2 = 0.0;
#pragma unroll 4
    for (int i = (lower ? j : 0) + lane; i < rows; i += 32) {
      const double v = col[i];
      s1 = fma(v, x1[i], s1);
      s2 = fma(v, x2[i], s2);
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
      y1[j] = s1;
      y2[j] = s2;
    }
  }
  __syncthreads();
}

// Copy a rows x cols column-major block (lower: only i >= j) from global memory into the
// work area: a warp per column, 4 x 4 loads per thread in flight, so a block of up to
// 64 columns x 128 rows costs one memory latency instead of one per element row.  The
// small state is usually cold (every pass over U sweeps L2).  No synchronisation.
__device__ inline void cta_stage_block(double* dst, int ldd, const double* src, int64_t lds, int rows, int cols,
                                       bool lower) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int b0 = 0; b0 < cols; b0 += 4 * nw)
    for (int a0 = 0; a0 < rows; a0 += 128) {
      double v[4][4];
#pragma unroll
      for (int q1 = 0; q1 < 4; ++q1)
#pragma unroll
        for (int q2 = 0; q2 < 4; ++q2) {
          const int b = b0 + wid + nw * q1, a = a0 + lane + 32 * q2;
          v[q1][q2] = (b < cols && a < rows && (!lower || a >= b)) ? __ldcg(src + (int64_t)b * lds + a) : 0.0;
        }
#pragma unroll
      for (int q1 = 0; q1 < 4; ++q1)
#pragma unroll
        for (int q2 = 0; q2 < 4; ++q2) {
          const int b = b0 + wid + nw * q1, a = a0 + lane + 32 * q2;
          if (b < cols && a < rows) dst[b * ldd + a] = v[q1][q2];
        }
    }
}

// Three block-wide sums at once (fixed tree, deterministic); `red` >= 3 * 32 doubles.
__device__ inline void block_sum3(double& a, double& b, double& c, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  c = warp_sum(c);
  __syncthreads();
  if (lane == 0) {
    red[wid] = a;
    red[32 + wid] = b;
    red[64 + wid] = c;
  }
  __syncthreads();
  a = warp_sum(lane < nw ? red[lane] : 0.0);
  b = warp_sum(lane < nw ? red[32 + lane] : 0.0);
  c = warp_sum(lane < nw ? red[64 + lane] : 0.0);
}

__device__ inline void cta_lower_mv(const double* Li, int ld, int n, const double* x, double* y) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double s = 0.0;
#pragma unroll 4
    for (int j = 0; j <= i; ++j) s = fma(Li[(int64_t)j * ld + i], x[j], s);
    y[i] = s;
  }
}

__device__ inline void cta_lower_t_mv(const double* Li, int ld, int n, const double* x, double* y) {
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double* col = Li + (int64_t)j * ld;
    double s = 0.0;
#pragma unroll 4
    for (int i = j; i < n; ++i) s = fma(col[i], x[i], s);
    y[j] = s;
  }
}

// Li = L^{-1} for a lower-triangular L (n x n): one warp per column of the
// inverse, lanes hold the right-hand side; n <= 256.
template <int Q>
__device__ inline void cta_lower_inverse_q(const double* L, int ld, int n, double* Li, int ldi) {
  // warp per column of the inverse: forward substitution L x = e_j with the
  // right-hand side distributed over the lanes (rows lane + 32 q); the
  // reciprocal pivots are taken from Li's diagonal (precomputed below), so the
  // serial chain per step is one shuffle and one multiply
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = wid; j < n; j += nw) {
    double x[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) x[q] = (lane + 32 * q == j) ? 1.0 : 0.0;
    for (int k = j; k < n; ++k) {
      const int owner = k & 31, slot = k >> 5;
      double xk = 0.0;
#pragma unroll
      for (int q = 0; q < Q; ++q)
        if (q == slot) xk = x[q];
      xk = __shfl_sync(0xffffffffu, xk, owner) * Li[(int64_t)k * ldi + k];
      const double* lk = L + (int64_t)k * ld;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int i = lane + 32 * q;
        if (i == k) x[q] = xk;
        else if (i > k && i < n) x[q] = fma(-lk[i], xk, x[q]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int i = lane + 32 * q;
      if (i < n && i != j) Li[(int64_t)j * ldi + i] = (i > j) ? x[q] : 0.0;
    }
  }
}

// Li = L^{-1} for a lower-triangular L (n x n), n <= 256.  Li must not alias L.
__device__ inline void cta_lower_inverse(const double* L, int ld, int n, double* Li, int ldi) {
  for (int k = threadIdx.x; k < n; k += blockDim.x) Li[(int64_t)k * ldi + k] = 1.0 / L[(int64_t)k * ld + k];
  __syncthreads();
  if (n <= 32) cta_lower_inverse_q<1>(L, ld, n, Li, ldi);
  else if (n <= 64) cta_lower_inverse_q<2>(L, ld, n, Li, ldi);
  else if (n <= 128) cta_lower_inverse_q<4>(L, ld, n, Li, ldi);
  else cta_lower_inverse_q<8>(L, ld, n, Li, ldi);
}

}  // namespace strom
