// Spatial reduced operators (reference spatial.py:45-67) in one fused pass:
//
//   [A_hat | B_hat | C_hat | xref_hat | x0_hat] = Phi^T [A Phi | B | C | A x_ref | x0 - x_ref]
//
// Each CTA walks 32-row tiles: the right operand tile (A Phi rows from a CSR
// gather, plus the dense extra columns) and the Phi tile are staged in shared
// memory and contracted on the fp64 tensor cores (DMMA m8n8k4).  A Phi is
// never written to HBM.  Per-CTA partial Grams are reduced in a fixed order
// (deterministic).
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "../../include/strom_b200.h"
#include "bulk.cuh"
#include "dmma.cuh"
#include "runtime.cuh"

using namespace strom;

namespace {

constexpr int kRows = 32;  // rows per tile (8 k-steps of 4)
constexpr int kNzReg = 8;  // CSR entries per row kept in registers
constexpr int kLdK = kRows + 4;  // k-major smem tiles: [col][row], padded (conflict-free frags)

template <typename IdxT>
struct SpatialArgs {
  int64_t N;
  const IdxT* indptr;
  const IdxT* indices;
  const double* data;
  const double* phi;
  int64_t phi_rs, phi_cs;
  int ns;
  const double* extra;  // column-major N x ne (ld ext_ld)
  int64_t ext_ld;
  int ne;
  const double* xref;   // N or null
  int q, MA, NQ, ldA, ldY;
  double* part;         // gridDim.x x (MA * NQ)
};

__host__ __device__ inline int pad_ld(int m) { return (m % 16 == 0) ? m + 8 : m; }

template <typename IdxT, int TAW, int TBM>
__global__ void __launch_bounds__(256, 2) k_spatial(SpatialArgs<IdxT> A) {
  extern __shared__ double smem[];
  double* Ph = smem;                          // MA x kLdK   (Ph[a * kLdK + i] = Phi[row0 + i, a])
  double* Ys = smem + (int64_t)A.MA * kLdK;   // NQ x kLdK   (Ys[j * kLdK + i] = Y[row0 + i, j])
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int TA = A.MA / 8, TB = A.NQ / 8;
  const int64_t ntiles = ceil_div(A.N, kRows);
  const int64_t per = ceil_div(ntiles, gridDim.x);
  const int64_t t0 = blockIdx.x * per, t1 = min(ntiles, t0 + per);
  double acc[TAW][TBM][2];
#pragma unroll
  for (int x = 0; x < TAW; ++x)
#pragma unroll
    for (int y = 0; y < TBM; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  const bool phi_colmajor = (A.phi_rs == 1);
  for (int64_t tile = t0; tile < t1; ++tile) {
    const int64_t row0 = tile * kRows;
    __syncthreads();
    // ---- Phi tile (left operand) ----
    for (int idx = threadIdx.x; idx < kRows * A.MA; idx += blockDim.x) {
      int i, a;
      if (phi_colmajor) { i = idx % kRows; a = idx / kRows; }
      else { a = idx % A.MA; i = idx / A.MA; }
      const int64_t row = row0 + i;
      Ph[a * kLdK + i] = (row < A.N && a < A.ns) ? __ldg(A.phi + row * A.phi_rs + (int64_t)a * A.phi_cs) : 0.0;
    }
    // ---- right operand: CSR gather A Phi, extra columns, A x_ref ----
    {
      const int i = lane;
      const int64_t row = row0 + i;
      int64_t nz0 = 0, nz1 = 0;
      if (row < A.N) {
        nz0 = (int64_t)__ldg(A.indptr + row);
        nz1 = (int64_t)__ldg(A.indptr + row + 1);
      }
      const int cnt = (int)((nz1 - nz0) < kNzReg ? (nz1 - nz0) : kNzReg);
      int64_t cidx[kNzReg];
      double cval[kNzReg];
#pragma unroll
      for (int qq = 0; qq < kNzReg; ++qq) {
        cidx[qq] = (qq < cnt) ? (int64_t)__ldg(A.indices + nz0 + qq) * A.phi_rs : 0;
        cval[qq] = (qq < cnt) ? __ldg(A.data + nz0 + qq) : 0.0;
      }
      // A Phi columns j = wid + 8 jj: all (column, nonzero) gathers of the tile are
      // independent loads, issued together (memory-level parallelism)
      double sacc[TBM];
#pragma unroll
      for (int jj = 0; jj < TBM; ++jj) sacc[jj] = 0.0;
      if (row < A.N) {
#pragma unroll
        for (int qq = 0; qq < kNzReg; ++qq) {
          if (qq < cnt) {
            const double* pc = A.phi + cidx[qq];  // cidx holds index * phi_rs
#pragma unroll
            for (int jj = 0; jj < TBM; ++jj) {
              const int j = wid + 8 * jj;
              if (j < A.ns) sacc[jj] = fma(cval[qq], __ldg(pc + (int64_t)j * A.phi_cs), sacc[jj]);
            }
          }
        }
        for (int64_t nz = nz0 + kNzReg; nz < nz1; ++nz) {
          const double v = __ldg(A.data + nz);
          const double* pc = A.phi + (int64_t)__ldg(A.indices + nz) * A.phi_rs;
#pragma unroll
          for (int jj = 0; jj < TBM; ++jj) {
            const int j = wid + 8 * jj;
            if (j < A.ns) sacc[jj] = fma(v, __ldg(pc + (int64_t)j * A.phi_cs), sacc[jj]);
          }
        }
      }
#pragma unroll
      for (int jj = 0; jj < TBM; ++jj) {
        const int j = wid + 8 * jj;
        if (j < A.ns) Ys[j * kLdK + i] = sacc[jj];
      }
      // extra columns and A x_ref
      for (int j = A.ns + wid; j < A.NQ; j += 8) {
        double s = 0.0;
        if (row < A.N) {
          if (j < A.ns + A.ne) {
            s = __ldg(A.extra + (int64_t)(j - A.ns) * A.ext_ld + row);
          } else if (j < A.q) {  // A x_ref
#pragma unroll
            for (int qq = 0; qq < kNzReg; ++qq)
              if (qq < cnt) s = fma(cval[qq], __ldg(A.xref + (A.phi_rs == 1 ? cidx[qq] : cidx[qq] / A.phi_rs)), s);
            for (int64_t nz = nz0 + kNzReg; nz < nz1; ++nz)
              s = fma(__ldg(A.data + nz), __ldg(A.xref + (int64_t)__ldg(A.indices + nz)), s);
          }
        }
        Ys[j * kLdK + i] = s;
      }
    }
    __syncthreads();
    // ---- DMMA: acc += Ph^T Ys over the 32 rows ----
#pragma unroll
    for (int kk = 0; kk < kRows / 4; ++kk) {
      const int kr = kk * 4 + t;
#pragma unroll
      for (int x = 0; x < TAW; ++x) {
        const int ta = wid + 8 * x;
        if (ta < TA) {
          const double a = Ph[(ta * 8 + g) * kLdK + kr];
#pragma unroll
          for (int y = 0; y < TBM; ++y) {
            if (y < TB) {
              const double b = Ys[(y * 8 + g) * kLdK + kr];
              dmma884(acc[x][y][0], acc[x][y][1], a, b);
            }
          }
        }
      }
    }
  }
  double* mp = A.part + (int64_t)blockIdx.x * A.MA * A.NQ;
#pragma unroll
  for (int x = 0; x < TAW; ++x) {
    const int ta = wid + 8 * x;
    if (ta >= TA) continue;
#pragma unroll
    for (int y = 0; y < TBM; ++y) {
      if (y >= TB) continue;
      const int r = ta * 8 + g, c = y * 8 + 2 * t;
      mp[r * A.NQ + c] = acc[x][y][0];
      mp[r * A.NQ + c + 1] = acc[x][y][1];
    }
  }
}

// Row-major Phi (phi_cs == 1): the gather is done row-wise -- warp w builds
// output rows i = w, w+8, ... of the tile, lanes own columns, so every
// neighbour row Phi[c, :] (ns contiguous doubles) is one coalesced load per 32
// columns; the CSR entries of the row are loaded once and broadcast by shuffle.
// The contraction is the same DMMA loop as k_spatial.  NCH = ceil(q / 32).
template <typename IdxT, int TAW, int TBM, int NCH>
__global__ void __launch_bounds__(256) k_spatial_rm(SpatialArgs<IdxT> A) {
  extern __shared__ double smem[];
  double* Ph = smem;                          // MA x kLdK
  double* Ys = smem + (int64_t)A.MA * kLdK;   // NQ x kLdK
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int TA = A.MA / 8, TB = A.NQ / 8;
  const int64_t ntiles = ceil_div(A.N, kRows);
  const int64_t per = ceil_div(ntiles, gridDim.x);
  const int64_t t0 = blockIdx.x * per, t1 = min(ntiles, t0 + per);
  double acc[TAW][TBM][2];
#pragma unroll
  for (int x = 0; x < TAW; ++x)
#pragma unroll
    for (int y = 0; y < TBM; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  const int64_t prs = A.phi_rs;
  for (int64_t tile = t0; tile < t1; ++tile) {
    const int64_t row0 = tile * kRows;
    __syncthreads();
    {
      // warp w owns rows i = w + 8 rr (rr < 4): CSR extents and entries for all
      // four rows in one load each (lane = 8 rr + k), then every neighbour-row
      // gather of the four rows issued together (predicated, fully unrolled)
      constexpr int RPW = kRows / 8, KNZ = 8;
      int64_t myrow = row0 + wid + 8 * (lane & 3);
      int64_t ext0 = 0, ext1 = 0;
      if (lane < RPW && myrow < A.N) {
        ext0 = (int64_t)__ldg(A.indptr + myrow);
        ext1 = (int64_t)__ldg(A.indptr + myrow + 1);
      }
      int64_t rs[RPW], rc[RPW];
#pragma unroll
      for (int rr = 0; rr < RPW; ++rr) {
        rs[rr] = __shfl_sync(0xffffffffu, ext0, rr);
        rc[rr] = __shfl_sync(0xffffffffu, ext1, rr) - rs[rr];
      }
      const int er = lane / KNZ, ek = lane % KNZ;
      int64_t myc = 0;
      double myv = 0.0;
      {
        int64_t st0 = 0, cn = 0;
#pragma unroll
        for (int rr = 0; rr < RPW; ++rr)
          if (er == rr) { st0 = rs[rr]; cn = rc[rr]; }
        if (ek < cn) {
          myc = (int64_t)__ldg(A.indices + st0 + ek);
          myv = __ldg(A.data + st0 + ek);
        }
      }
      double y[RPW][NCH], yx[RPW];
#pragma unroll
      for (int rr = 0; rr < RPW; ++rr) {
        yx[rr] = 0.0;
#pragma unroll
        for (int h = 0; h < NCH; ++h) y[rr][h] = 0.0;
      }
#pragma unroll
      for (int rr = 0; rr < RPW; ++rr) {
#pragma unroll
        for (int k = 0; k < KNZ; ++k) {
          const int64_t cc = __shfl_sync(0xffffffffu, myc, rr * KNZ + k);
          const double vv = __shfl_sync(0xffffffffu, myv, rr * KNZ + k);
          if (k < rc[rr]) {
            const double* prow = A.phi + cc * prs;
#pragma unroll
            for (int h = 0; h < NCH; ++h) {
              const int j = lane + 32 * h;
              if (j < A.ns) y[rr][h] = fma(vv, __ldg(prow + j), y[rr][h]);
            }
            if (A.xref) yx[rr] = fma(vv, __ldg(A.xref + cc), yx[rr]);
          }
        }
        for (int64_t nz = rs[rr] + KNZ; nz < rs[rr] + rc[rr]; ++nz) {  // rows with > 8 entries
          const int64_t cc = (int64_t)__ldg(A.indices + nz);
          const double vv = __ldg(A.data + nz);
          const double* prow = A.phi + cc * prs;
#pragma unroll
          for (int h = 0; h < NCH; ++h) {
            const int j = lane + 32 * h;
            if (j < A.ns) y[rr][h] = fma(vv, __ldg(prow + j), y[rr][h]);
          }
          if (A.xref) yx[rr] = fma(vv, __ldg(A.xref + cc), yx[rr]);
        }
      }
      // right operand rows [A Phi | extra | A x_ref];  left operand rows Phi
#pragma unroll
      for (int rr = 0; rr < RPW; ++rr) {
        const int i = wid + 8 * rr;
        const int64_t row = row0 + i;
        const bool live = row < A.N;
#pragma unroll
        for (int h = 0; h < NCH; ++h) {
          const int j = lane + 32 * h;
          if (j < A.NQ) {
            double v = 0.0;
            if (live) {
              if (j < A.ns) v = y[rr][h];
              else if (j < A.ns + A.ne) v = __ldg(A.extra + (int64_t)(j - A.ns) * A.ext_ld + row);
              else if (j < A.q) v = yx[rr];
            }
            Ys[j * kLdK + i] = v;
          }
          if (j < A.MA) Ph[j * kLdK + i] = (live && j < A.ns) ? __ldg(A.phi + row * prs + j) : 0.0;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kRows / 4; ++kk) {
      const int kr = kk * 4 + t;
#pragma unroll
      for (int x = 0; x < TAW; ++x) {
        const int ta = wid + 8 * x;
        if (ta < TA) {
          const double a = Ph[(ta * 8 + g) * kLdK + kr];
#pragma unroll
          for (int yy = 0; yy < TBM; ++yy) {
            if (yy < TB) {
              const double b = Ys[(yy * 8 + g) * kLdK + kr];
              dmma884(acc[x][yy][0], acc[x][yy][1], a, b);
            }
          }
        }
      }
    }
  }
  double* mp = A.part + (int64_t)blockIdx.x * A.MA * A.NQ;
#pragma unroll
  for (int x = 0; x < TAW; ++x) {
    const int ta = wid + 8 * x;
    if (ta >= TA) continue;
#pragma unroll
    for (int yy = 0; yy < TBM; ++yy) {
      if (yy >= TB) continue;
      const int r = ta * 8 + g, c = yy * 8 + 2 * t;
      mp[r * A.NQ + c] = acc[x][yy][0];
      mp[r * A.NQ + c + 1] = acc[x][yy][1];
    }
  }
}

// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Column-major Phi (phi_rs == 1, ld = phi_cs), n_s <= 64, q <= 64, operator in
// the tiled ELL layout of strom_csr_to_ell (diagonal kept apart, K off-
// diagonal slots per row).  Warp-specialised, one persistent CTA per SM, 64-row
// tiles dealt round-robin (tile = blockIdx.x + it * gridDim.x) so the grid
// advances through Phi as one band of gridDim.x * 64 rows (the rows a banded
// operator reaches stay in L2), through an S-deep shared-memory ring.
//   * Producer warps (two row halves x NPW/2 column groups, lane = row): the
//     tile's ELL slices arrive by bulk copy (issued one tile ahead); each lane
//     gathers kWsCols (4, or 2 when K = 16) columns per round -- all kWsCols x K neighbour loads and
//     the kWsCols Phi(row, j) loads issued before the first FMA -- and forms
//     Y(row, j) = d(row) Phi(row, j) + sum_k a_k Phi(c_k, j), reusing the Phi
//     tile element for the diagonal.  One lane streams the ELL slices two bands
//     ahead and the Phi rows `reach` + one band ahead into L2.
//   * NCW = 4 consumer warps (one per SM sub-partition) contract each stage on
//     the fp64 tensor cores.  For the common fragment grids (TA x TB = 7x7,
//     8x8) the grid is split into four compile-time fragment ranges (no
//     predicated MMAs); other shapes use a runtime x-row split.
// Stage handshakes are named barriers: FULL(s) = 1 + s, EMPTY(s) = 1 + S + s
// (all threads); barrier 15 orders the producers' reuse of ELL buffers.
constexpr int kWsRows = 64;
constexpr int kWsLd = kWsRows + 8;  // 72: conflict-free 16-byte fragment loads
constexpr int kWsNPW = 12, kWsNCW = 4;
constexpr int kWsThreads = (kWsNPW + kWsNCW) * 32;
constexpr int kWsProdBar = 15;
constexpr int kWsProdRegs = 136, kWsConsRegs = 96;  // setmaxnreg targets (see k_spatial_ell)

struct EllArgs {
  int64_t N;
  const uint32_t* eidx;  // per tile: [K][64] off-diagonal column indices
  const double* eval;    // per tile: [K][64] off-diagonal values, then [64] diagonal values
  int64_t reach;         // max (col - row) over off-diagonal entries; < 0: no Phi prefetch
  const double* phi;
  int64_t ld;
  int ns;
  const double* extra;   // column-major N x ne (ld ext_ld)
  int64_t ext_ld;
  int ne;
  const double* xref;    // N or null
  int q, MA, NQ, S;
  int dbg;               // diagnostics: 1 = producers skip the gathers, 2 = consumers skip the MMAs
  int pf_bands;          // Phi L2 prefetch distance past the forward reach, in bands of gridDim.x * 64 rows
  double* part;          // gridDim.x x (MA * NQ)
  unsigned long long* tbuf;  // diagnostics: per-warp phase cycle totals (dbg 5)
};

// Stage position of tile row i: rows 8u + t (k-step 2u) and 8u + 4 + t (k-step
// 2u + 1) sit side by side, so one 16-byte load gives a lane both k-steps'
// fragment values (the Gram sums over rows, so any common row order works).
__device__ __forceinline__ int ws_pos(int i) { return (i & ~7) | ((i & 3) << 1) | ((i >> 2) & 1); }

__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <int TB, int F0, int F1>
__host__ __device__ constexpr bool frag_col_used(int y) {
  for (int f = F0; f < F1; ++f)
    if (f % TB == y) return true;
  return false;
}

// consumer loop over a compile-time fragment range [F0, F1) of the TA x TB grid
template <int TA, int TB, int F0, int F1>
__device__ __forceinline__ void ell_consume(const EllArgs& A, const double* smem, int stage_elems, int nmine,
                                            double* mp) {
  constexpr int NF = F1 - F0, X0 = F0 / TB, X1 = (F1 - 1) / TB;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double acc[NF][2];
#pragma unroll
  for (int f = 0; f < NF; ++f) acc[f][0] = acc[f][1] = 0.0;
  long long pw = 0, pc = 0;
  for (int it = 0; it < nmine; ++it) {
    const int s = it % A.S;
    long long t0 = clock64();
    named_bar_sync(1 + s, kWsThreads);
    long long t1 = clock64(); pw += t1 - t0;
    const double* Ph = smem + (int64_t)s * stage_elems;
    const double* Ys = Ph + A.MA * kWsLd;
#pragma unroll 1
    for (int u = 0; u < (A.dbg == 2 ? 0 : kWsRows / 8); ++u) {  // k-step pairs
      const int kp = u * 8 + 2 * t;
      double2 a[X1 - X0 + 1], b[TB];
#pragma unroll
      for (int x = X0; x <= X1; ++x) a[x - X0] = *reinterpret_cast<const double2*>(Ph + (x * 8 + g) * kWsLd + kp);
#pragma unroll
      for (int y = 0; y < TB; ++y)
        if (frag_col_used<TB, F0, F1>(y)) b[y] = *reinterpret_cast<const double2*>(Ys + (y * 8 + g) * kWsLd + kp);
#pragma unroll
      for (int f = F0; f < F1; ++f) dmma884(acc[f - F0][0], acc[f - F0][1], a[f / TB - X0].x, b[f % TB].x);
#pragma unroll
      for (int f = F0; f < F1; ++f) dmma884(acc[f - F0][0], acc[f - F0][1], a[f / TB - X0].y, b[f % TB].y);
    }
    pc += clock64() - t1;
    if (it + A.S < nmine) named_bar_arrive(1 + A.S + s, kWsThreads);
  }
  if (A.tbuf && lane == 0) {
    atomicAdd(A.tbuf + (threadIdx.x >> 5) * 8 + 0, (unsigned long long)pw);
    atomicAdd(A.tbuf + (threadIdx.x >> 5) * 8 + 1, (unsigned long long)pc);
  }
#pragma unroll
  for (int f = F0; f < F1; ++f) {
    const int r = (f / TB) * 8 + g, cc = (f % TB) * 8 + 2 * t;
    mp[r * A.NQ + cc] = acc[f - F0][0];
    mp[r * A.NQ + cc + 1] = acc[f - F0][1];
  }
}

// consumer loop for runtime TA, TB <= 8: warp c owns x-rows c and c + 4
__device__ __forceinline__ void ell_consume_generic(const EllArgs& A, const double* smem, int stage_elems, int nmine,
                                                    double* mp, int c) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int TA = A.MA / 8, TB = A.NQ / 8;
  double acc[2][8][2];
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 8; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  for (int it = 0; it < nmine; ++it) {
    const int s = it % A.S;
    named_bar_sync(1 + s, kWsThreads);
    const double* Ph = smem + (int64_t)s * stage_elems;
    const double* Ys = Ph + A.MA * kWsLd;
#pragma unroll 1
    for (int u = 0; u < (A.dbg == 2 ? 0 : kWsRows / 8); ++u) {
      const int kp = u * 8 + 2 * t;
      double2 b[8];
#pragma unroll
      for (int y = 0; y < 8; ++y)
        b[y] = (y < TB) ? *reinterpret_cast<const double2*>(Ys + (y * 8 + g) * kWsLd + kp) : make_double2(0.0, 0.0);
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const int ta = c + kWsNCW * x;
        if (ta < TA) {
          const double2 av = *reinterpret_cast<const double2*>(Ph + (ta * 8 + g) * kWsLd + kp);
#pragma unroll
          for (int y = 0; y < 8; ++y)
            if (y < TB) dmma884(acc[x][y][0], acc[x][y][1], av.x, b[y].x);
#pragma unroll
          for (int y = 0; y < 8; ++y)
            if (y < TB) dmma884(acc[x][y][0], acc[x][y][1], av.y, b[y].y);
        }
      }
    }
    if (it + A.S < nmine) named_bar_arrive(1 + A.S + s, kWsThreads);
  }
#pragma unroll
  for (int x = 0; x < 2; ++x) {
    const int ta = c + kWsNCW * x;
    if (ta >= TA) continue;
#pragma unroll
    for (int y = 0; y < 8; ++y) {
      if (y >= TB) continue;
      const int r = ta * 8 + g, cc = y * 8 + 2 * t;
      mp[r * A.NQ + cc] = acc[x][y][0];
      mp[r * A.NQ + cc + 1] = acc[x][y][1];
    }
  }
}

__host__ __device__ inline size_t ell_tile_bytes(int K) { return (size_t)K * kWsRows * 4 + (size_t)(K + 1) * kWsRows * 8; }

template <int K, int TA, int TB>
__global__ void __launch_bounds__(kWsThreads, 1) k_spatial_ell(EllArgs A) {
  extern __shared__ __align__(128) double smem[];
  constexpr int NCG = kWsNPW / 2;
  // columns gathered per round: kWsCols x (K + 1) loads in flight per lane, sized for the
  // producers' 136-register budget after the warpgroup register handoff below
  constexpr int kWsCols = K <= 4 ? 8 : K <= 6 ? 6 : K <= 8 ? 4 : 2;
  const int stage_elems = (A.MA + A.NQ) * kWsLd;
  unsigned char* ebase = reinterpret_cast<unsigned char*>(smem + (int64_t)A.S * stage_elems);
  uint64_t* ebar = reinterpret_cast<uint64_t*>(ebase + 2 * ell_tile_bytes(K));
  const double** colbase = reinterpret_cast<const double**>(ebar + 2);  // Phi column j at colbase[j]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t ntiles = ceil_div(A.N, kWsRows);
  const int nmine = (int)(blockIdx.x < ntiles ? ceil_div(ntiles - blockIdx.x, gridDim.x) : 0);
  auto tile_of = [&](int it) -> int64_t { return blockIdx.x + (int64_t)it * gridDim.x; };
  constexpr unsigned kIdxBytes = K * kWsRows * 4, kValBytes = (K + 1) * kWsRows * 8;
  auto issue_ell = [&](int it) {  // ELL slices of this CTA's tile `it` into buffer it & 1
    const int64_t tile = tile_of(it);
    unsigned char* buf = ebase + (it & 1) * ell_tile_bytes(K);
    mbar_expect_tx(&ebar[it & 1], kIdxBytes + kValBytes);
    bulk_g2s(buf, A.eidx + tile * K * kWsRows, kIdxBytes, &ebar[it & 1]);
    bulk_g2s(buf + kIdxBytes, A.eval + tile * (K + 1) * kWsRows, kValBytes, &ebar[it & 1]);
  };
  if (threadIdx.x == 0) {
    mbar_init(&ebar[0], 1);
    mbar_init(&ebar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (nmine > 0) issue_ell(0);
  }
  if (threadIdx.x < 64) colbase[threadIdx.x] = A.phi + (int64_t)(threadIdx.x < A.ns ? threadIdx.x : 0) * A.ld;
  __syncthreads();

  if (wid < kWsNPW) {
    // ------------------------------------------------------------ producers
    // register handoff inside the CTA's launch allocation (512 x 128): the
    // consumer warpgroup drops to 96 registers, the three producer warpgroups
    // rise to 136 (3 * 128 * 136 + 128 * 96 = 64512; checked on the host)
    asm volatile("setmaxnreg.inc.sync.aligned.u32 136;\n" ::: "memory");
    const int half = wid & 1, cg = wid >> 1;
    const int i = half * 32 + lane;
    const int ip = ws_pos(i);  // stage position of row i
    const int64_t ld = A.ld;
    long long ph[5] = {0, 0, 0, 0, 0};
    for (int it = 0; it < nmine; ++it) {
      const int s = it % A.S;
      const int64_t tile = tile_of(it);
      const int64_t row0 = tile * kWsRows, row = row0 + i;
      const bool live = row < A.N;
      long long tc0 = clock64();
      named_bar_sync(kWsProdBar, kWsNPW * 32);  // every producer is past tile it-1: its ELL buffer is free
      long long tc1 = clock64(); ph[0] += tc1 - tc0;
      if (lane == 0) {
        // L2 prefetch, spread over the producer warps: the operator slices and
        // dense extra columns of the tile three ahead, and Phi rows one band past
        // the operator's forward reach (the gathers' first touch of a row)
        const int64_t tp = it + 3 < nmine ? tile_of(it + 3) : ntiles;
        if (wid == 0) {
          if (it + 1 < nmine) issue_ell(it + 1);
          if (tp < ntiles) {
            prefetch_l2_bulk(A.eidx + tp * K * kWsRows, kIdxBytes);
            prefetch_l2_bulk(A.eval + tp * (K + 1) * kWsRows, kValBytes);
          }
        }
        if (tp * kWsRows + kWsRows <= A.N)
          for (int e = wid; e < A.ne; e += kWsNPW) prefetch_l2_bulk(A.extra + e * A.ext_ld + tp * kWsRows, kWsRows * 8);
        const int64_t pr = row0 + A.reach + (int64_t)A.pf_bands * gridDim.x * kWsRows;
        if (A.reach >= 0 && pr + kWsRows <= A.N)
          for (int j = wid; j < A.ns; j += kWsNPW) prefetch_l2_bulk(A.phi + j * A.ld + pr, kWsRows * 8);
      }
      long long tc2 = clock64();
      mbar_wait(&ebar[it & 1], (it >> 1) & 1);
      ph[1] += clock64() - tc2;
      const unsigned char* buf = ebase + (it & 1) * ell_tile_bytes(K);
      const uint32_t* bi = reinterpret_cast<const uint32_t*>(buf);
      const double* bv = reinterpret_cast<const double*>(buf + kIdxBytes);
      uint32_t ci[K];
      double cv[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        ci[k] = bi[k * kWsRows + i];
        cv[k] = bv[k * kWsRows + i];
      }
      const double dv = bv[K * kWsRows + i];
      if (A.dbg == 3) {  // diagnostics: every neighbour is the row itself (L1-resident gathers)
#pragma unroll
        for (int k = 0; k < K; ++k) ci[k] = (uint32_t)(live ? row : A.N - 1);
      }
      long long tc3 = clock64();
      if (it >= A.S) named_bar_sync(1 + A.S + s, kWsThreads);
      long long tc4 = clock64(); ph[2] += tc4 - tc3;
      double* Ph = smem + (int64_t)s * stage_elems;
      double* Ys = Ph + A.MA * kWsLd;
      // A Phi and Phi columns, kWsCols per round: j_m = cg + NCG * (r * kWsCols + m);
      // a fixed round count with warp-uniform predicates keeps every round's
      // kWsCols x (K + 1) loads in one batch ahead of the FMAs.
      constexpr int kRounds = ((64 + NCG - 1) / NCG + kWsCols - 1) / kWsCols;
      const int nsg = A.dbg == 1 ? 0 : A.ns;
      const uint32_t self = (uint32_t)(live ? row : A.N - 1);
#pragma unroll 1
      for (int r = 0; r < kRounds; ++r) {
        const int jb = cg + NCG * r * kWsCols;
        if (jb >= nsg) break;
        const double* cb[kWsCols];
        bool on[kWsCols];
#pragma unroll
        for (int m = 0; m < kWsCols; ++m) {
          const int jm = jb + m * NCG;
          on[m] = jm < nsg;
          cb[m] = colbase[on[m] ? jm : jb];  // loaded, so address = base + 8 * index stays one IMAD.WIDE
        }
        double v[kWsCols][K + 1];
#pragma unroll
        for (int m = 0; m < kWsCols; ++m) {
#pragma unroll
          for (int k = 0; k < K; ++k) v[m][k] = __ldg(cb[m] + ci[k]);
          v[m][K] = __ldg(cb[m] + self);
        }
#pragma unroll
        for (int m = 0; m < kWsCols; ++m) {
          const double p = live ? v[m][K] : 0.0;
          double y = dv * p;
#pragma unroll
          for (int k = 0; k < K; ++k) y = fma(cv[k], v[m][k], y);
          const int jm = jb + m * NCG;
          if (on[m]) {
            Ph[jm * kWsLd + ip] = p;
            Ys[jm * kWsLd + ip] = y;
          }
        }
      }
      long long tc5 = clock64(); ph[3] += tc5 - tc4;
      // dense extra columns, A x_ref, zero padding (columns of this group past ns)
      for (int j = cg + ((A.ns - cg + NCG - 1) / NCG) * NCG; j < A.NQ; j += NCG) {
        double y = 0.0;
        if (j < A.ns + A.ne) {
          if (live) y = __ldg(A.extra + (int64_t)(j - A.ns) * A.ext_ld + row);
        } else if (j < A.q) {  // A x_ref
          y = live ? dv * __ldg(A.xref + row) : 0.0;
#pragma unroll
          for (int k = 0; k < K; ++k) y = fma(cv[k], __ldg(A.xref + ci[k]), y);
        }
        Ys[j * kWsLd + ip] = y;
        if (j < A.MA) Ph[j * kWsLd + ip] = 0.0;
      }
      ph[4] += clock64() - tc5;
      named_bar_arrive(1 + s, kWsThreads);
    }
    if (A.tbuf && lane == 0)
      for (int q = 0; q < 5; ++q) atomicAdd(A.tbuf + wid * 8 + q, (unsigned long long)ph[q]);
    return;
  }

  // -------------------------------------------------------------- consumers
  asm volatile("setmaxnreg.dec.sync.aligned.u32 96;\n" ::: "memory");
  const int c = wid - kWsNPW;
  double* mp = A.part + (int64_t)blockIdx.x * A.MA * A.NQ;
  if constexpr (TA > 0) {
    constexpr int NF = TA * TB;
    if (c == 0) ell_consume<TA, TB, 0, NF / 4>(A, smem, stage_elems, nmine, mp);
    else if (c == 1) ell_consume<TA, TB, NF / 4, NF / 2>(A, smem, stage_elems, nmine, mp);
    else if (c == 2) ell_consume<TA, TB, NF / 2, 3 * NF / 4>(A, smem, stage_elems, nmine, mp);
    else ell_consume<TA, TB, 3 * NF / 4, NF>(A, smem, stage_elems, nmine, mp);
  } else {
    ell_consume_generic(A, smem, stage_elems, nmine, mp, c);
  }
}

// CSR -> tiled ELL: per 64-row tile, K off-diagonal slots (column index,
// value; an unused slot points at the row itself with value 0) and the
// diagonal (sum of the row's diagonal entries).  Also the operator's forward
// reach max(col - row) over off-diagonal entries and an overflow flag (a row
// with more than K off-diagonal entries).  One thread per row.
template <typename IdxT>
__global__ void k_csr_to_ell(int64_t n, const IdxT* __restrict__ indptr, const IdxT* __restrict__ indices,
                             const double* __restrict__ data, int K, uint32_t* __restrict__ eidx,
                             double* __restrict__ eval, unsigned long long* reach_enc, int* overflow) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nt = ceil_div(n, kWsRows);
  if (row >= nt * kWsRows) return;
  const int64_t tile = row / kWsRows;
  const int i = (int)(row % kWsRows);
  const uint32_t self = (uint32_t)(row < n ? row : n - 1);
  uint32_t* ti = eidx + tile * K * kWsRows;
  double* tv = eval + tile * (K + 1) * kWsRows;
  int64_t e0 = 0, e1 = 0;
  if (row < n) { e0 = (int64_t)indptr[row]; e1 = (int64_t)indptr[row + 1]; }
  long long reach = LLONG_MIN;
  double diag = 0.0;
  int k = 0;
  for (int64_t e = e0; e < e1; ++e) {
    const int64_t c = (int64_t)indices[e];
    if (c == row) { diag += data[e]; continue; }
    if (k == K) { atomicExch(overflow, 1); break; }
    ti[k * kWsRows + i] = (uint32_t)c;
    tv[k * kWsRows + i] = data[e];
    reach = max(reach, (long long)(c - row));
    ++k;
  }
  for (; k < K; ++k) {
    ti[k * kWsRows + i] = self;
    tv[k * kWsRows + i] = 0.0;
  }
  tv[K * kWsRows + i] = diag;
  // order-preserving encoding of a signed max as an unsigned atomicMax
  if (reach != LLONG_MIN) atomicMax(reach_enc, (unsigned long long)reach ^ 0x8000000000000000ull);
}

// out (ns x q, row-major) = sum over CTAs of the partials.  A CTA owns 32
// outputs; warp w sums the partials of its contiguous slice of CTAs, and the
// eight slice sums are added in slice order (deterministic).
__global__ void __launch_bounds__(256) k_spatial_reduce(const double* part, int nparts, int MA, int NQ, int ns, int q,
                                                        double* out) {
  __shared__ double red[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int idx = blockIdx.x * 32 + lane;
  const bool live = idx < ns * q;
  const int a = live ? idx / q : 0, b = live ? idx % q : 0;
  const double* p0 = part + a * NQ + b;
  const int64_t st = (int64_t)MA * NQ;
  const int per = (nparts + 7) / 8, pb = w * per, pe = min(nparts, pb + per);
  double s0 = 0.0, s1 = 0.0;
  int p = pb;
  for (; p + 1 < pe; p += 2) {
    s0 += p0[p * st];
    s1 += p0[(p + 1) * st];
  }
  if (p < pe) s0 += p0[p * st];
  red[w][lane] = s0 + s1;
  __syncthreads();
  if (w == 0 && live) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k][lane];
    out[idx] = t;
  }
}

// grid = SMs x resident CTAs of the chosen kernel (one wave), capped by the tiles
template <class K>
int one_wave(K kernel, size_t smem, int64_t ntiles) {
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, 256, smem);
  return (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)sm_count() * std::max(occ, 1)));
}

template <typename IdxT, int TAW, int TBM>
int launch_spatial_t(SpatialArgs<IdxT> a, int max_grid, cudaStream_t s) {
  const size_t smem = (size_t)kLdK * (a.MA + a.NQ) * 8;
  static PerDevice<bool> configured_dev;
  bool& configured = configured_dev.get();
  if (!configured) {
    STROM_CUDA(cudaFuncSetAttribute(k_spatial<IdxT, TAW, TBM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    64 * 1024));
    STROM_CUDA(cudaFuncSetAttribute(k_spatial_rm<IdxT, TAW, TBM, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    64 * 1024));
    STROM_CUDA(cudaFuncSetAttribute(k_spatial_rm<IdxT, TAW, TBM, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    64 * 1024));
    configured = true;
  }
  const int64_t ntiles = ceil_div(a.N, kRows);
  ProfScope ps(P_SPATIAL, s);
  int grid;
  if (a.phi_cs == 1 && a.phi_rs >= a.ns) {  // row-major Phi: row-wise coalesced gather
    if (a.NQ <= 64 && a.MA <= 64) {
      grid = std::min(max_grid, one_wave(k_spatial_rm<IdxT, TAW, TBM, 2>, smem, ntiles));
      k_spatial_rm<IdxT, TAW, TBM, 2><<<grid, 256, smem, s>>>(a);
    } else {
      grid = std::min(max_grid, one_wave(k_spatial_rm<IdxT, TAW, TBM, 5>, smem, ntiles));
      k_spatial_rm<IdxT, TAW, TBM, 5><<<grid, 256, smem, s>>>(a);
    }
  } else {
    grid = std::min(max_grid, one_wave(k_spatial<IdxT, TAW, TBM>, smem, ntiles));
    k_spatial<IdxT, TAW, TBM><<<grid, 256, smem, s>>>(a);
  }
  STROM_LAUNCH_CHECK();
  return grid;
}

size_t ell_smem(int K, int S, int MA, int NQ) {
  return (size_t)S * (MA + NQ) * kWsLd * 8 + 2 * ell_tile_bytes(K) + 16 + 64 * 8;
}

template <int K, int TA, int TB>
void launch_ell_kernel(const EllArgs& a, int grid, size_t smem, cudaStream_t s) {
  auto kern = k_spatial_ell<K, TA, TB>;
  static PerDevice<bool> configured_dev;
  bool& configured = configured_dev.get();
  if (!configured) {
    STROM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_smem_optin()));
    // the warpgroup register handoff must fit the launch allocation, or the
    // producers' setmaxnreg.inc would wait forever
    cudaFuncAttributes fa{};
    STROM_CUDA(cudaFuncGetAttributes(&fa, kern));
    if ((int64_t)fa.numRegs * kWsThreads < (int64_t)kWsNPW * 32 * kWsProdRegs + (int64_t)kWsNCW * 32 * kWsConsRegs)
      throw Error(kInternal, "spatial ELL kernel: register handoff exceeds the launch allocation");
    configured = true;
  }
  kern<<<grid, kWsThreads, smem, s>>>(a);
  STROM_LAUNCH_CHECK();
}

template <int K>
void launch_spatial_ell_k(const EllArgs& a, int grid, size_t smem, cudaStream_t s) {
  const int TA = a.MA / 8, TB = a.NQ / 8;
  if (TA == 7 && TB == 7) launch_ell_kernel<K, 7, 7>(a, grid, smem, s);
  else if (TA == 8 && TB == 8) launch_ell_kernel<K, 8, 8>(a, grid, smem, s);
  else launch_ell_kernel<K, 0, 0>(a, grid, smem, s);
}

template <typename IdxT>
int launch_spatial(SpatialArgs<IdxT> a, int max_grid, cudaStream_t s) {
  const int TA = a.MA / 8, TB = a.NQ / 8;
  if (TA <= 8 && TB <= 8) return launch_spatial_t<IdxT, 1, 8>(a, max_grid, s);
  if (TA <= 8 && TB <= 17) return launch_spatial_t<IdxT, 1, 17>(a, max_grid, s);
  if (TA <= 16 && TB <= 17) return launch_spatial_t<IdxT, 2, 17>(a, max_grid, s);
  throw Error(kInvalidArgument, "spatial reduction supports n_s <= 128 and <= 136 right columns");
}

}  // namespace

// Y = A X for a CSR operator and a row-major right-hand side (X(j, k) at X[j * ldx + k],
// m columns): one thread per (row, column), a row's entries added in CSR order, so neighbouring
// threads read neighbouring X entries.  The residual evaluations of the a-posteriori bounds
// (system.py:249-275: A x_k for every step) and the sparse applies of operator_norm
// (bounds.py:60-70).
namespace {
template <class I>
__global__ void __launch_bounds__(256) k_csr_spmm(int64_t n, const I* __restrict__ indptr,
                                                  const I* __restrict__ indices, const double* __restrict__ data,
                                                  const double* __restrict__ X, int64_t ldx, int64_t m,
                                                  double* __restrict__ Y, int64_t ldy) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * m) return;
  const int64_t row = idx / m, k = idx - row * m;
  const I p0 = indptr[row], p1 = indptr[row + 1];
  double acc = 0.0;
  for (I p = p0; p < p1; ++p) acc = fma(data[p], X[(int64_t)indices[p] * ldx + k], acc);
  Y[row * ldy + k] = acc;
}
}  // namespace

extern "C" {

// build_spatial_rom's contractions (spatial.py:57-64).  A: CSR (indptr N+1,
// indices, data) with int32 (index_bits 32) or int64 indices.  phi element
// (i, j) at phi[i*phi_rs + j*phi_cs].  extra: column-major N x ne (ld ext_ld),
// typically [B | C | x0 - x_ref].  xref: N-vector or NULL.  Output out_dev:
// row-major ns x q, q = ns + ne + (xref != NULL):
//   out[:, :ns] = A_hat,  out[:, ns:ns+ne] = Phi^T extra,  out[:, -1] = Phi^T A x_ref.
int strom_spatial_reduce_csr(int64_t n, const void* indptr_dev, const void* indices_dev, const double* data_dev,
                             int32_t index_bits, const double* phi_dev, int64_t phi_rs, int64_t phi_cs,
                             int64_t ns, const double* extra_dev, int64_t ext_ld, int64_t ne,
                             const double* xref_dev, double* out_dev, void* stream) {
  return guarded([&] {
    STROM_REQUIRE(n >= 1 && ns >= 1 && ns <= 128 && ne >= 0, "bad spatial-reduction shape");
    STROM_REQUIRE(index_bits == 32 || index_bits == 64, "index_bits must be 32 or 64");
    STROM_REQUIRE(n < (int64_t(1) << 31), "spatial reduction needs n < 2^31 rows");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int q = (int)(ns + ne + (xref_dev ? 1 : 0));
    const int MA = (int)round_up(ns, 8), NQ = (int)round_up(q, 8);
    const int max_grid = sm_count() * 8;
    auto part = dev_alloc((size_t)max_grid * MA * NQ * 8, s, false);
    int grid = 1;
    auto fill = [&](auto& a) {
      a.N = n;
      a.data = data_dev;
      a.phi = phi_dev;
      a.phi_rs = phi_rs;
      a.phi_cs = phi_cs;
      a.ns = (int)ns;
      a.extra = extra_dev;
      a.ext_ld = ext_ld;
      a.ne = (int)ne;
      a.xref = xref_dev;
      a.q = q;
      a.MA = MA;
      a.NQ = NQ;
      a.ldA = pad_ld(MA);
      a.ldY = pad_ld(NQ);
      a.part = part->as<double>();
    };
    if (index_bits == 32) {
      SpatialArgs<int32_t> a{};
      fill(a);
      a.indptr = static_cast<const int32_t*>(indptr_dev);
      a.indices = static_cast<const int32_t*>(indices_dev);
      grid = launch_spatial(a, max_grid, s);
    } else {
      SpatialArgs<int64_t> a{};
      fill(a);
      a.indptr = static_cast<const int64_t*>(indptr_dev);
      a.indices = static_cast<const int64_t*>(indices_dev);
      grid = launch_spatial(a, max_grid, s);
    }
    k_spatial_reduce<<<(unsigned)ceil_div((int64_t)ns * q, 32), 256, 0, s>>>(part->as<double>(), grid, MA, NQ,
                                                                              (int)ns, q, out_dev);
    STROM_LAUNCH_CHECK();
  });
}


// Tiled ELL form of a CSR operator for strom_spatial_reduce_ell (the device
// layout the spatial reduction gathers from; built once per operator).
// K >= max off-diagonal entries per row, K in {4, 6, 8, 16}.  eidx_dev:
// uint32[ceil(n/64) * K * 64], eval_dev: double[ceil(n/64) * (K+1) * 64].
// *reach_out (host) = max(col - row) over the off-diagonal entries (-1: none).
int strom_csr_to_ell(int64_t n, const void* indptr_dev, const void* indices_dev, const double* data_dev,
                     int32_t index_bits, int32_t K, uint32_t* eidx_dev, double* eval_dev, int64_t* reach_out,
                     void* stream) {
  return guarded([&] {
    STROM_REQUIRE(n >= 1 && n < (int64_t(1) << 31), "ELL operator needs 1 <= n < 2^31 rows");
    STROM_REQUIRE(K == 4 || K == 6 || K == 8 || K == 16, "ELL width must be 4, 6, 8 or 16");
    STROM_REQUIRE(index_bits == 32 || index_bits == 64, "index_bits must be 32 or 64");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    auto flags = dev_alloc(16, s, true);
    unsigned long long* enc = flags->as<unsigned long long>();
    int* overflow = reinterpret_cast<int*>(enc + 1);
    const int64_t rows = ceil_div(n, kWsRows) * kWsRows;
    const unsigned grid = (unsigned)ceil_div(rows, 256);
    if (index_bits == 32)
      k_csr_to_ell<int32_t><<<grid, 256, 0, s>>>(n, static_cast<const int32_t*>(indptr_dev),
                                                static_cast<const int32_t*>(indices_dev), data_dev, K, eidx_dev,
                                                eval_dev, enc, overflow);
    else
      k_csr_to_ell<int64_t><<<grid, 256, 0, s>>>(n, static_cast<const int64_t*>(indptr_dev),
                                                static_cast<const int64_t*>(indices_dev), data_dev, K, eidx_dev,
                                                eval_dev, enc, overflow);
    STROM_LAUNCH_CHECK();
    unsigned long long h[2] = {0, 0};
    STROM_CUDA(cudaMemcpyAsync(h, flags->ptr, 16, cudaMemcpyDeviceToHost, s));
    STROM_CUDA(cudaStreamSynchronize(s));
    STROM_REQUIRE((h[1] & 0xffffffffull) == 0, "ELL width too small for a row of the operator");
    *reach_out = h[0] == 0 ? -1 : (int64_t)(h[0] ^ 0x8000000000000000ull);
  });
}

// build_spatial_rom's contractions (spatial.py:57-64) from the tiled ELL form:
// column-major phi (element (i, j) at phi[i + j*ld]), ns <= 64 and
// q = ns + ne + (xref != NULL) <= 64.  Output as strom_spatial_reduce_csr.
int strom_spatial_reduce_ell(int64_t n, int32_t K, const uint32_t* eidx_dev, const double* eval_dev, int64_t reach,
                             const double* phi_dev, int64_t ld, int64_t ns, const double* extra_dev, int64_t ext_ld,
                             int64_t ne, const double* xref_dev, double* out_dev, void* stream) {
  return guarded([&] {
    STROM_REQUIRE(n >= 1 && n < (int64_t(1) << 31) && ld >= n, "bad ELL spatial-reduction shape");
    STROM_REQUIRE(K == 4 || K == 6 || K == 8 || K == 16, "ELL width must be 4, 6, 8 or 16");
    const int q = (int)(ns + ne + (xref_dev ? 1 : 0));
    STROM_REQUIRE(ns >= 1 && ns <= 64 && ne >= 0 && q <= 64, "ELL spatial reduction supports n_s, q <= 64");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    EllArgs a{};
    a.N = n;
    a.eidx = eidx_dev;
    a.eval = eval_dev;
    a.reach = (reach >= 0 && reach < n / 4) ? reach : -1;
    a.phi = phi_dev;
    a.ld = ld;
    a.ns = (int)ns;
    a.extra = extra_dev;
    a.ext_ld = ext_ld;
    a.ne = (int)ne;
    a.xref = xref_dev;
    a.q = q;
    a.MA = (int)round_up(ns, 8);
    a.NQ = (int)round_up(q, 8);
    // two stages: a third buys no producer slack (the wait on a free stage is
    // short) and costs ~64 KB of L1, which the neighbour gathers hit (measured
    // cfg4 build: 0.59 ms with two stages, 0.65 ms with three)
    a.S = 2;
    if (const char* e = getenv("STROM_SPATIAL_DBG")) a.dbg = atoi(e);
    if (getenv("STROM_SPATIAL_NOPF")) a.reach = -1;
    a.pf_bands = 1;
    if (const char* e = getenv("STROM_SPATIAL_PF")) a.pf_bands = std::max(0, atoi(e));
    if (const char* e = getenv("STROM_SPATIAL_STAGES")) a.S = std::max(1, std::min(a.S, atoi(e)));
    const size_t smem = ell_smem(K, a.S, a.MA, a.NQ);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(sm_count(), ceil_div(n, kWsRows)));
    auto part = dev_alloc((size_t)grid * a.MA * a.NQ * 8, s, false);
    a.part = part->as<double>();
    DevMemPtr tb;
    if (a.dbg == 5) {
      tb = dev_alloc(32 * 8 * 8, s, true);
      a.tbuf = tb->as<unsigned long long>();
    }
    {
      ProfScope ps(P_SPATIAL, s);
      if (K == 4) launch_spatial_ell_k<4>(a, grid, smem, s);
      else if (K == 6) launch_spatial_ell_k<6>(a, grid, smem, s);
      else if (K == 8) launch_spatial_ell_k<8>(a, grid, smem, s);
      else launch_spatial_ell_k<16>(a, grid, smem, s);
    }
    k_spatial_reduce<<<(unsigned)ceil_div((int64_t)ns * q, 32), 256, 0, s>>>(part->as<double>(), grid, a.MA, a.NQ,
                                                                            (int)ns, q, out_dev);
    STROM_LAUNCH_CHECK();
    if (tb) {
      unsigned long long h[128];
      STROM_CUDA(cudaMemcpyAsync(h, tb->ptr, sizeof(h), cudaMemcpyDeviceToHost, s));
      STROM_CUDA(cudaStreamSynchronize(s));
      for (int w = 0; w < 16; ++w)
        fprintf(stderr, "warp %2d cycles/CTA: %10.0f %10.0f %10.0f %10.0f %10.0f\n", w, h[w * 8] / (double)grid,
                h[w * 8 + 1] / (double)grid, h[w * 8 + 2] / (double)grid, h[w * 8 + 3] / (double)grid,
                h[w * 8 + 4] / (double)grid);
    }
  });
}

int strom_csr_spmm(int64_t n, const void* indptr_dev, const void* indices_dev, const double* data_dev,
                   int32_t index_bits, const double* x_dev, int64_t ldx, int64_t m, double* y_dev, int64_t ldy,
                   void* stream) {
  return guarded([&] {
    STROM_REQUIRE(n >= 1 && m >= 1 && ldx >= m && ldy >= m, "bad spmm shape");
    STROM_REQUIRE(index_bits == 32 || index_bits == 64, "index_bits must be 32 or 64");
    STROM_REQUIRE(indptr_dev && x_dev && y_dev, "null argument");  // indices / data may be empty (no entries)
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const unsigned grid = (unsigned)ceil_div(n * m, 256);
    if (index_bits == 32)
      k_csr_spmm<int32_t><<<grid, 256, 0, s>>>(n, static_cast<const int32_t*>(indptr_dev),
                                               static_cast<const int32_t*>(indices_dev), data_dev, x_dev, ldx, m,
                                               y_dev, ldy);
    else
      k_csr_spmm<int64_t><<<grid, 256, 0, s>>>(n, static_cast<const int64_t*>(indptr_dev),
                                               static_cast<const int64_t*>(indices_dev), data_dev, x_dev, ldx, m,
                                               y_dev, ldy);
    STROM_LAUNCH_CHECK();
  });
}

}  // extern "C"
