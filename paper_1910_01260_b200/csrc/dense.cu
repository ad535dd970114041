// Dense fp64 factorizations on the device:
//   strom_dense_solve -- LU with partial pivoting + the reference's pivot
//                        floor (linalg.py:75-99), used by solve_st_rom
//                        (spacetime.py:154-162)
//   strom_qr          -- positive-diagonal Householder QR (linalg.py:60-72)
//
// LU: blocked right-looking.  Each 32-column panel is factored by one CTA
// (pivot search, row swap across the full width, scale, rank-1 update inside
// the panel); the trailing matrix is updated by a unit-lower TRSM and a
// register-blocked GEMM across all SMs.  The matrix (<= a few thousand) stays
// L2-resident between kernels.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/strom_b200.h"
#include "runtime.cuh"
#include "dmma.cuh"
#include "small_dense.cuh"

using namespace strom;

namespace {

constexpr int kNb = 32;
constexpr int kNbReg = 16;  // panel width of the register-resident panel factorisation

// Programmatic dependent launch along the factorisation chain (panel ->
// swap/TRSM -> update -> next panel): each kernel lets its successor launch
// at once and waits for its predecessor before touching A, so the launch
// latency hides behind the running kernel.
__device__ __forceinline__ void lu_pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <class... KArgs, class... Args>
void lu_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  STROM_CUDA(cudaLaunchKernelEx(&cfg, kernel, args...));
}

__global__ void k_fro_norm(const double* A, int64_t ld, int64_t n, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    const int64_t i = idx % n, j = idx / n;
    const double v = A[j * ld + i];
    s = fma(v, v, s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) out[0] = sqrt(s);
}

// Factor panel columns [k0, k0+nb) of A (n x n, ld), swapping full rows.
__global__ void __launch_bounds__(1024) k_lu_panel(double* A, int64_t ld, int n, int k0, int nb, int* piv) {
  __shared__ double sv[32];
  __shared__ int si[32];
  __shared__ int s_p;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = k0; j < k0 + nb; ++j) {
    double* cj = A + (int64_t)j * ld;
    // argmax |A[i, j]| over i >= j, first index on ties (idamax)
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int i = j + threadIdx.x; i < n; i += blockDim.x) {
      const double a = fabs(cj[i]);
      if (a > best || (a == best && i < bi)) { best = a; bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (lane == 0) { sv[wid] = best; si[wid] = bi; }
    __syncthreads();
    if (wid == 0) {
      best = (lane < nw) ? sv[lane] : -1.0;
      bi = (lane < nw) ? si[lane] : 0x7fffffff;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (lane == 0) {
        s_p = (bi == 0x7fffffff) ? j : bi;
        piv[j] = s_p;
      }
    }
    __syncthreads();
    const int p = s_p;
    if (p != j) {
      for (int c = threadIdx.x; c < n; c += blockDim.x) {
        const double t = A[(int64_t)c * ld + j];
        A[(int64_t)c * ld + j] = A[(int64_t)c * ld + p];
        A[(int64_t)c * ld + p] = t;
      }
    }
    __syncthreads();
    const double d = cj[j];
    if (d != 0.0) {
      const double inv = 1.0 / d;
      for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) cj[i] *= inv;
    }
    __syncthreads();
    // rank-1 update of the rest of the panel
    const int rem_c = k0 + nb - j - 1;
    for (int c = wid; c < rem_c; c += nw) {
      double* cc = A + (int64_t)(j + 1 + c) * ld;
      const double u = cc[j];
      for (int i = j + 1 + lane; i < n; i += 32) cc[i] = fma(-cj[i], u, cc[i]);
    }
    __syncthreads();
  }
}

// A12 <- L11^{-1} A12 for columns [k0+nb, n): one thread per column.
__global__ void k_lu_trsm(double* A, int64_t ld, int n, int k0, int nb) {
  const int c = k0 + nb + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  double x[kNb];
  double* col = A + (int64_t)c * ld;
#pragma unroll
  for (int i = 0; i < kNb; ++i) x[i] = (i < nb) ? col[k0 + i] : 0.0;
#pragma unroll
  for (int j = 0; j < kNb; ++j) {
    if (j >= nb) break;
    const double xj = x[j];
#pragma unroll
    for (int i = j + 1; i < kNb; ++i)
      if (i < nb) x[i] = fma(-A[(int64_t)(k0 + j) * ld + k0 + i], xj, x[i]);
  }
#pragma unroll
  for (int i = 0; i < kNb; ++i)
    if (i < nb) col[k0 + i] = x[i];
}

// A22 -= L21 U12 ; tiles of 64 x 64, 256 threads, 4 x 4 per thread.
__global__ void __launch_bounds__(256) k_lu_gemm(double* A, int64_t ld, int n, int k0, int nb) {
  lu_pdl_enter();
  __shared__ double Ls[64][kNb + 1];
  __shared__ double Us[kNb][64 + 1];
  const int s0 = k0 + nb;
  const int r0 = s0 + blockIdx.x * 64, c0 = s0 + blockIdx.y * 64;
  if (r0 >= n || c0 >= n) return;
  for (int idx = threadIdx.x; idx < 64 * kNb; idx += blockDim.x) {
    const int i = idx % 64, kk = idx / 64;
    Ls[i][kk] = (r0 + i < n && kk < nb) ? A[(int64_t)(k0 + kk) * ld + r0 + i] : 0.0;
    const int c = idx / kNb, k2 = idx % kNb;
    Us[k2][c] = (c0 + c < n && k2 < nb) ? A[(int64_t)(c0 + c) * ld + k0 + k2] : 0.0;
  }
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4] = {};
#pragma unroll 8
  for (int kk = 0; kk < kNb; ++kk) {
    double a[4], b[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) a[q] = Ls[tx + 16 * q][kk];
#pragma unroll
    for (int q = 0; q < 4; ++q) b[q] = Us[kk][ty + 16 * q];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[p][q] = fma(a[p], b[q], acc[p][q]);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = c0 + ty + 16 * q;
    if (c >= n) continue;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int r = r0 + tx + 16 * p;
      if (r < n) A[(int64_t)c * ld + r] -= acc[p][q];
    }
  }
}

// Pivot check (first |U_ii| <= floor) + triangular solves, one CTA.
// info[0] = first bad index (or -1), info[1] = its |pivot|, info[2] = floor.
__global__ void __launch_bounds__(1024) k_lu_solve(const double* A, int64_t ld, int n, const int* piv, double* X,
                                                   int64_t ldx, int nrhs, const double* fro, double* info) {
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0x7fffffff;
  __syncthreads();
  const double floor = fro ? 1e-14 * fro[0] : -1.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (fabs(A[(int64_t)i * ld + i]) <= floor) atomicMin(&s_bad, i);
  __syncthreads();
  if (threadIdx.x == 0) {
    info[0] = (s_bad == 0x7fffffff) ? -1.0 : (double)s_bad;
    info[1] = (s_bad == 0x7fffffff) ? 0.0 : fabs(A[(int64_t)s_bad * ld + s_bad]);
    info[2] = floor;
  }
  if (s_bad != 0x7fffffff) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int c = wid; c < nrhs; c += nw) {
    double* x = X + (int64_t)c * ldx;
    if (lane == 0)
      for (int j = 0; j < n; ++j) {
        const int p = piv[j];
        if (p != j) { const double t = x[j]; x[j] = x[p]; x[p] = t; }
      }
    __syncwarp();
    // forward: unit lower
    for (int j = 0; j < n; ++j) {
      const double xj = x[j];
      for (int i = j + 1 + lane; i < n; i += 32) x[i] = fma(-A[(int64_t)j * ld + i], xj, x[i]);
      __syncwarp();
    }
    // backward: upper
    for (int j = n - 1; j >= 0; --j) {
      double xj = 0.0;
      if (lane == 0) { xj = x[j] / A[(int64_t)j * ld + j]; x[j] = xj; }
      xj = __shfl_sync(0xffffffffu, xj, 0);
      for (int i = lane; i < j; i += 32) x[i] = fma(-A[(int64_t)j * ld + i], xj, x[i]);
      __syncwarp();
    }
  }
}

// Panel factorisation with the panel held in registers: thread t owns rows
// k0 + t + 512 q (q < RPT) of the nb <= kNbReg panel columns.  Per column: an
// argmax reduction (largest |a|, lowest row on ties, like idamax), the pivot
// row exchanged through shared memory, then scale and rank-1 update in
// registers.  Row interchanges are applied to the panel only; k_lu_swap_trsm
// applies them to the other columns afterwards (LAPACK's getrf order).
template <int RPT>
__global__ void __launch_bounds__(512, 1) k_lu_panel_reg(double* A, int64_t ld, int n, int k0, int nb, int* piv) {
  lu_pdl_enter();
  // per column, double-buffered by column parity: each warp's pivot candidate
  // (value, row, the row's panel entries) and the row the pivot displaces.  One
  // barrier per column: every warp reduces the 16 candidates itself.
  __shared__ double cand[2][16][kNbReg];
  __shared__ double cval[2][16];
  __shared__ int cidx[2][16];
  __shared__ double drow[2][kNbReg];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double a[RPT][kNbReg];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int i = k0 + threadIdx.x + 512 * q;
#pragma unroll
    for (int c = 0; c < kNbReg; ++c) a[q][c] = (i < n && c < nb) ? A[(int64_t)(k0 + c) * ld + i] : 0.0;
  }
  // fully unrolled over the panel width: j is a compile-time constant in each
  // copy, so a[q][j] is a plain register and the update covers c > j statically
  // (no per-column register-select chains)
#pragma unroll
  for (int j = 0; j < kNbReg; ++j) {
    if (j >= nb) break;
    const int jr = k0 + j, buf = j & 1;
    double best = -1.0;
    int bi = 0x7fffffff;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int i = k0 + threadIdx.x + 512 * q;
      double v = 0.0;
#pragma unroll
      for (int c = 0; c < kNbReg; ++c)
        if (c == j) v = a[q][c];
      if (i >= jr && i < n) {
        const double av = fabs(v);
        if (av > best || (av == best && i < bi)) { best = av; bi = i; }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    // the owner of the warp's candidate row and of row jr publish them
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int i = k0 + threadIdx.x + 512 * q;
      if (i == bi)
#pragma unroll
        for (int c = 0; c < kNbReg; ++c) cand[buf][wid][c] = a[q][c];
      if (i == jr)
#pragma unroll
        for (int c = 0; c < kNbReg; ++c) drow[buf][c] = a[q][c];
    }
    if (lane == 0) {
      cval[buf][wid] = best;
      cidx[buf][wid] = bi;
    }
    __syncthreads();
    // every warp: argmax over the 16 warp candidates (same rule), carrying the warp
    double gb = lane < 16 ? cval[buf][lane] : -1.0;
    int gi = lane < 16 ? cidx[buf][lane] : 0x7fffffff;
    int gw = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, gb, o);
      const int oi = __shfl_xor_sync(0xffffffffu, gi, o);
      const int ow = __shfl_xor_sync(0xffffffffu, gw, o);
      if (ob > gb || (ob == gb && oi < gi)) { gb = ob; gi = oi; gw = ow; }
    }
    // a candidate exists unless the whole sub-column is NaN (every |a| > best
    // test fails): then row jr pivots on itself, like k_lu_panel
    const bool none = (gi == 0x7fffffff);
    const int p = none ? jr : gi;
    if (threadIdx.x == 0) piv[jr] = p;
    const double* prow = none ? drow[buf] : cand[buf][gw & 15];
    const double d = prow[j];
    const double inv = d != 0.0 ? 1.0 / d : 0.0;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int i = k0 + threadIdx.x + 512 * q;
      if (i == jr && p != jr) {
#pragma unroll
        for (int c = 0; c < kNbReg; ++c) a[q][c] = prow[c];
      } else if (i == p && p != jr) {
#pragma unroll
        for (int c = 0; c < kNbReg; ++c) a[q][c] = drow[buf][c];
      }
      if (i > jr && i < n && d != 0.0) {
        double l = 0.0;
#pragma unroll
        for (int c = 0; c < kNbReg; ++c)
          if (c == j) { l = a[q][c] * inv; a[q][c] = l; }
#pragma unroll
        for (int c = 0; c < kNbReg; ++c)
          if (c > j) a[q][c] = fma(-l, prow[c], a[q][c]);
      }
    }
    // no trailing barrier: column j+1 writes the other buffers, and column j+2
    // reaches these only after column j+1's barrier, which every thread passes
    // after finishing column j
  }
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int i = k0 + threadIdx.x + 512 * q;
    if (i < n)
#pragma unroll
      for (int c = 0; c < kNbReg; ++c)
        if (c < nb) A[(int64_t)(k0 + c) * ld + i] = a[q][c];
  }
}

// getrf's laswp + trsm for a register panel in one launch: every column
// outside the panel gets the panel's row interchanges in order; the columns
// right of it then U12 = L11^-1 A12 (unit lower L11 staged in shared memory).
// One thread per column; rows k0..k0+nb-1 of it live in registers.
__global__ void __launch_bounds__(64) k_lu_swap_trsm(double* A, int64_t ld, int n, int k0, int nb, const int* piv) {
  lu_pdl_enter();
  __shared__ double sL[kNbReg][kNbReg + 1];
  __shared__ int spv[kNbReg];
  for (int e = threadIdx.x; e < kNbReg * kNbReg; e += blockDim.x) {
    const int i = e % kNbReg, j = e / kNbReg;
    sL[i][j] = (j < i && i < nb) ? A[(int64_t)(k0 + j) * ld + k0 + i] : 0.0;
  }
  if (threadIdx.x < kNbReg) spv[threadIdx.x] = threadIdx.x < nb ? piv[k0 + threadIdx.x] : k0 + threadIdx.x;
  __syncthreads();
  const int cc = blockIdx.x * blockDim.x + threadIdx.x;
  if (cc >= n - nb) return;
  const int c = cc < k0 ? cc : cc + nb;
  double* col = A + (int64_t)c * ld;
  double x[kNbReg];
#pragma unroll
  for (int r = 0; r < kNbReg; ++r) x[r] = r < nb ? col[k0 + r] : 0.0;
#pragma unroll
  for (int j = 0; j < kNbReg; ++j) {
    if (j >= nb) break;
    const int p = spv[j];
    if (p == k0 + j) continue;
    if (p < k0 + nb) {  // both rows in the register block
      double t = 0.0;
#pragma unroll
      for (int r = 0; r < kNbReg; ++r)
        if (r == p - k0) t = x[r];
#pragma unroll
      for (int r = 0; r < kNbReg; ++r)
        if (r == p - k0) x[r] = x[j];
      x[j] = t;
    } else {
      const double t = col[p];
      col[p] = x[j];
      x[j] = t;
    }
  }
  if (c >= k0 + nb) {
#pragma unroll
    for (int j = 0; j < kNbReg; ++j) {
      if (j >= nb) break;
#pragma unroll
      for (int i = j + 1; i < kNbReg; ++i)
        if (i < nb) x[i] = fma(-sL[i][j], x[j], x[i]);
    }
  }
#pragma unroll
  for (int r = 0; r < kNbReg; ++r)
    if (r < nb) col[k0 + r] = x[r];
}

// Row interchanges of panel [k0, k0+nb) applied to the columns outside it,
// in order; one thread per column.
__global__ void k_lu_laswp(double* A, int64_t ld, int n, int k0, int nb, const int* piv) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n - nb) return;
  if (c >= k0) c += nb;
  double* col = A + (int64_t)c * ld;
  for (int j = 0; j < nb; ++j) {
    const int p = piv[k0 + j];
    if (p != k0 + j) {
      const double t = col[k0 + j];
      col[k0 + j] = col[p];
      col[p] = t;
    }
  }
}

// Pivot check + blocked triangular solves with the whole CTA, x in shared
// memory.  Per 32-row block: warp 0 solves the diagonal block (each lane holds
// its row of the block in registers; the columns are broadcast by shuffle),
// then every thread subtracts the block's contribution from its remaining
// rows (coalesced column reads) -- two barriers per block instead of one per row.
__global__ void __launch_bounds__(512) k_lu_solve_cta(const double* A, int64_t ld, int n, const int* piv,
                                                       double* X, int64_t ldx, int nrhs, const double* fro,
                                                       double* info) {
  extern __shared__ double xs[];
  __shared__ int s_bad;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_bad = 0x7fffffff;
  __syncthreads();
  const double floor = fro ? 1e-14 * fro[0] : -1.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (fabs(A[(int64_t)i * ld + i]) <= floor) atomicMin(&s_bad, i);
  __syncthreads();
  if (threadIdx.x == 0) {
    info[0] = (s_bad == 0x7fffffff) ? -1.0 : (double)s_bad;
    info[1] = (s_bad == 0x7fffffff) ? 0.0 : fabs(A[(int64_t)s_bad * ld + s_bad]);
    info[2] = floor;
  }
  if (s_bad != 0x7fffffff) return;
  for (int rc = 0; rc < nrhs; ++rc) {
    double* x = X + (int64_t)rc * ldx;
    for (int i = threadIdx.x; i < n; i += blockDim.x) xs[i] = x[i];
    __syncthreads();
    if (threadIdx.x == 0)
      for (int j = 0; j < n; ++j) {
        const int p = piv[j];
        if (p != j) { const double t = xs[j]; xs[j] = xs[p]; xs[p] = t; }
      }
    __syncthreads();
    // Both sweeps keep one block of look-ahead: warp 0 applies block b's
    // contribution to the next block's rows and solves that block's diagonal
    // while warps 1.. apply it to the rows beyond -- one barrier per block.
    // Every row sees the same fma sequence as in a plain blocked sweep.
    auto diag_fwd = [&](int b0, int bw) {  // warp 0: unit lower diagonal block
      double lrow[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) lrow[j] = (lane < bw && j < lane) ? A[(int64_t)(b0 + j) * ld + b0 + lane] : 0.0;
      double xi = lane < bw ? xs[b0 + lane] : 0.0;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const double xj = __shfl_sync(0xffffffffu, xi, j);
        if (lane > j) xi = fma(-lrow[j], xj, xi);
      }
      if (lane < bw) xs[b0 + lane] = xi;
    };
    auto diag_bwd = [&](int b0, int bw) {  // warp 0: upper diagonal block
      double urow[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) urow[j] = (lane < bw && j >= lane && j < bw) ? A[(int64_t)(b0 + j) * ld + b0 + lane] : 0.0;
      double xi = lane < bw ? xs[b0 + lane] : 0.0;
#pragma unroll
      for (int j = 31; j >= 0; --j) {
        if (j < bw) {
          double xj = __shfl_sync(0xffffffffu, xi, j);
          if (lane == j) { xi = xi / urow[j]; }
          xj = __shfl_sync(0xffffffffu, xi, j);
          if (lane < j) xi = fma(-urow[j], xj, xi);
        }
      }
      if (lane < bw) xs[b0 + lane] = xi;
    };
    // row i minus the contribution of block [b0, b0 + bw) (unrolled: the 32
    // column loads are in flight at once)
    auto apply_block = [&](int i, int b0, int bw) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < bw) acc = fma(A[(int64_t)(b0 + j) * ld + i], xs[b0 + j], acc);
      xs[i] -= acc;
    };
    const int nt_rest = blockDim.x - 32;
    // forward: unit lower L
    if (wid == 0) diag_fwd(0, min(32, n));
    __syncthreads();
    for (int b0 = 0; b0 < n; b0 += 32) {
      const int bw = min(32, n - b0);
      const int nb0 = b0 + bw, nbw = min(32, n - nb0);
      if (wid == 0) {
        if (nbw > 0) {
          if (lane < nbw) apply_block(nb0 + lane, b0, bw);
          __syncwarp();
          diag_fwd(nb0, nbw);
        }
      } else if (nbw > 0) {
        for (int i = nb0 + nbw + (int)threadIdx.x - 32; i < n; i += nt_rest) apply_block(i, b0, bw);
      }
      __syncthreads();
    }
    // backward: upper U (blocks from the bottom)
    {
      const int lb0 = max(0, n - 32);
      if (wid == 0) diag_bwd(lb0, n - lb0);
      __syncthreads();
    }
    for (int b1 = n; b1 > 0; b1 -= 32) {
      const int b0 = max(0, b1 - 32), bw = b1 - b0;
      const int pb0 = max(0, b0 - 32), pbw = b0 - pb0;  // the block above
      if (wid == 0) {
        if (pbw > 0) {
          if (lane < pbw) apply_block(pb0 + lane, b0, bw);
          __syncwarp();
          diag_bwd(pb0, pbw);
        }
      } else {
        for (int i = (int)threadIdx.x - 32; i < pb0; i += nt_rest) apply_block(i, b0, bw);
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = xs[i];
    __syncthreads();
  }
}

// ||A||_F: per-CTA partial sums of squares, then one CTA adds them in order.
// Frobenius norm partials of the rows x cols column-major A (ld); a block that
// saw a non-finite entry writes NaN, so the norm doubles as the finiteness
// test of scipy's lu_factor / lu_solve (check_finite=True).
__global__ void __launch_bounds__(256) k_fro_part(const double* A, int64_t ld, int64_t rows, int64_t cols,
                                                  double* part) {
  __shared__ double red[32];
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  double s = 0.0;
  bool bad = false;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < rows * cols;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const double v = A[(idx / rows) * ld + idx % rows];
    bad |= !isfinite(v);
    s = fma(v, v, s);
  }
  if (bad) s_bad = 1;
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s_bad ? __longlong_as_double(0x7ff8000000000000LL) : s;
}
__global__ void __launch_bounds__(256) k_fro_final(const double* part, int np, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) out[0] = sqrt(s);
}

__global__ void __launch_bounds__(1024) k_qr(double* M, int64_t ld, int rows, int cols, double* R, double* work) {
  __shared__ double red[32];
  cta_householder_qr(M, (int)ld, rows, cols, R, cols, work, work + cols, red);
}

// ---------------------------------------------------------------------------
// Persistent dataflow LU (getrf semantics) with the right-hand sides riding
// along as extra columns.  One CTA per 16-column block column of [A | B], held
// in shared memory for the whole factorisation; CTAs hand work to each other
// through release/acquire flags instead of kernel boundaries:
//   block column j (A part): for k < j, when panel k is published, apply its
//     row interchanges, U_kj = L_kk^{-1} A_kj and the trailing update
//     A_ij -= L_ik U_kj on DMMA (m8n8k4); then factor its own panel (partial
//     pivoting, first index on ties like idamax), publish it, and afterwards
//     apply the later panels' interchanges to its L rows (dlaswp on the left
//     columns) before the final write-back;
//   B block columns: the same updates give L^{-1} P b (the forward solve of
//     getrs), then the backward solve U x = y in the same CTA.
// The critical path is the chain panel k -> update of block column k+1 ->
// panel k+1: one flag hand-off per 16 columns instead of three launches.
// Reference: linalg.py:75-99 (scipy lu_factor / lu_solve).
// ---------------------------------------------------------------------------
constexpr int kPlNb = 16;
constexpr int kPlThreads = 512;  // 16 warps, 2 register rows per thread (256 threads x 4 rows measured slower: 27.9 vs 19.5 us per panel)
constexpr int kPlWarps = kPlThreads / 32;

struct PlArgs {
  double* A;
  int64_t lda;
  double* B;
  int64_t ldb;
  int n, nrhs, nbA, ncb, ldS;
  int* piv;
  int* flag;  // [ncb] panel published (A blocks) / forward updates done (B blocks)
  int* fin;   // [nbA] final write-back of an A block column done
  long long* probe;  // diagnostics (STROM_LU_PROBE): 8 globaltimer stamps per CTA, or null
};
#define PL_PROBE(k)                                                                         \
  do {                                                                                      \
    if (a.probe && threadIdx.x == 0) {                                                      \
      unsigned long long _t;                                                                \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                                \
      a.probe[blockIdx.x * 8 + (k)] = (long long)_t;                                        \
    }                                                                                       \
  } while (0)

__device__ __forceinline__ int pl_ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void pl_wait(const int* f) {
  if (threadIdx.x == 0)
    while (pl_ld_acquire(f) == 0) __nanosleep(20);
  __syncthreads();
}
__device__ __forceinline__ void pl_signal(int* f) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(f), "r"(1) : "memory");
}

// S[lo:hi, 0:16] -= M[lo:hi, k0:k0+kw] * S[k0:k0+kw, 0:16]   (M global, read via L2)
// DMMA m8n8k4: warp w takes 8-row tiles w, w + 16, ...; two 8-column n-tiles.
// The M fragments of kPlBatch tiles are loaded before any of them is used, so
// the L2 latency is paid once per batch, not once per tile.
constexpr int kPlBatch = 4;
__device__ inline void pl_gemm(double* S, int ld, const double* M, int64_t ldm, int lo, int hi, int k0, int kw) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  double b[4][2];
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const int kc = 4 * ks + t;
    b[ks][0] = kc < kw ? S[g * ld + k0 + kc] : 0.0;
    b[ks][1] = kc < kw ? S[(8 + g) * ld + k0 + kc] : 0.0;
  }
  constexpr int kStride = 8 * kPlWarps;
  for (int base = lo + 8 * wid; base < hi; base += kStride * kPlBatch) {
    double a[kPlBatch][4];
#pragma unroll
    for (int q = 0; q < kPlBatch; ++q) {
      const int row = base + q * kStride + g;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const int kc = 4 * ks + t;
        a[q][ks] = (row < hi && kc < kw) ? -__ldcg(M + (int64_t)(k0 + kc) * ldm + row) : 0.0;
      }
    }
#pragma unroll
    for (int q = 0; q < kPlBatch; ++q) {
      const int r0 = base + q * kStride;
      if (r0 >= hi) break;
      const int row = r0 + g;
      const bool ok = row < hi;
      double c00 = 0, c01 = 0, c10 = 0, c11 = 0;
      if (ok) {
        c00 = S[(2 * t) * ld + row];
        c01 = S[(2 * t + 1) * ld + row];
        c10 = S[(8 + 2 * t) * ld + row];
        c11 = S[(9 + 2 * t) * ld + row];
      }
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        dmma884(c00, c01, a[q][ks], b[ks][0]);
        dmma884(c10, c11, a[q][ks], b[ks][1]);
      }
      if (ok) {
        S[(2 * t) * ld + row] = c00;
        S[(2 * t + 1) * ld + row] = c01;
        S[(8 + 2 * t) * ld + row] = c10;
        S[(9 + 2 * t) * ld + row] = c11;
      }
    }
  }
}

// Panel factorisation with the panel's rows in registers (thread tid owns rows
// tid + 512 q, q < kPlRpt): per column one argmax (idamax's rule: largest |a|,
// first row on ties), the pivot row and the row it displaces exchanged through
// shared memory, then scale and rank-1 update in registers; two barriers per
// column.  Fully unrolled over the 16 panel columns so every register index is
// static.
// Warp-wide argmax of (key, row) on the integer reduction unit (redux.sync): the key is the
// IEEE bit pattern of |a| plus one (0 = no candidate; bit patterns of non-negative doubles
// order like their values), the row index breaks ties towards the first row (idamax).  Three
// REDUX instructions instead of five rounds of three shuffles and a double compare.
__device__ __forceinline__ void pl_warp_argmax(unsigned long long key, int row, unsigned long long& kmax, int& rmin) {
  const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
  const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  const bool win = hi == mh && lo == ml;
  rmin = (int)__reduce_min_sync(0xffffffffu, win ? (unsigned)row : 0x7fffffffu);
  kmax = ((unsigned long long)mh << 32) | ml;
}
__device__ __forceinline__ unsigned long long pl_key(double v, bool candidate) {
  // NaN never wins (like `fabs(v) > best` with best = -1): an all-NaN column pivots on itself
  return (candidate && v == v) ? (unsigned long long)__double_as_longlong(fabs(v)) + 1ull : 0ull;
}

constexpr int kPlRpt = 2;  // register panel for n <= kPlThreads * kPlRpt = 1024
__device__ inline void pl_panel_reg(double* S, int ld, int n, int j0, int w, int* piv, unsigned long long* ckey,
                                    int* cidx, double* prow, double* grow) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double v[kPlRpt][kPlNb];
#pragma unroll
  for (int q = 0; q < kPlRpt; ++q) {
    const int r = tid + kPlThreads * q;
#pragma unroll
    for (int c = 0; c < kPlNb; ++c) v[q][c] = (r < n && r >= j0) ? S[c * ld + r] : 0.0;
  }
#pragma unroll
  for (int c = 0; c < kPlNb; ++c) {
    if (c >= w) break;
    const int gr = j0 + c;
    unsigned long long key = 0ull;
    int bi = 0x7fffffff;
#pragma unroll
    for (int q = 0; q < kPlRpt; ++q) {
      const int r = tid + kPlThreads * q;
      const unsigned long long kq = pl_key(v[q][c], r >= gr && r < n);
      if (kq > key) { key = kq; bi = r; }  // rows ascend with q: ties keep the first
    }
    pl_warp_argmax(key, bi, key, bi);
    if (lane == 0) { ckey[wid] = key; cidx[wid] = bi; }
    __syncthreads();
    pl_warp_argmax(ckey[lane & (kPlWarps - 1)], cidx[lane & (kPlWarps - 1)], key, bi);
    const int p = (key == 0ull || bi == 0x7fffffff) ? gr : bi;  // an all-NaN column pivots on itself
#pragma unroll
    for (int q = 0; q < kPlRpt; ++q) {
      const int r = tid + kPlThreads * q;
      if (r == p)
#pragma unroll
        for (int c2 = 0; c2 < kPlNb; ++c2) prow[c2] = v[q][c2];
      if (r == gr)
#pragma unroll
        for (int c2 = 0; c2 < kPlNb; ++c2) grow[c2] = v[q][c2];
    }
    if (tid == 0) piv[gr] = p;
    __syncthreads();
    const double d = prow[c];
    const double inv = d != 0.0 ? __drcp_rn(d) : 0.0;  // = 1.0 / d (correctly rounded), without the division routine
#pragma unroll
    for (int q = 0; q < kPlRpt; ++q) {
      const int r = tid + kPlThreads * q;
      if (r == gr) {
#pragma unroll
        for (int c2 = 0; c2 < kPlNb; ++c2) v[q][c2] = prow[c2];
      } else if (r == p) {
#pragma unroll
        for (int c2 = 0; c2 < kPlNb; ++c2) v[q][c2] = grow[c2];
      }
      if (r > gr && r < n && d != 0.0) {
        const double l = v[q][c] * inv;
        v[q][c] = l;
#pragma unroll
        for (int c2 = c + 1; c2 < kPlNb; ++c2) v[q][c2] = fma(-l, prow[c2], v[q][c2]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kPlRpt; ++q) {
    const int r = tid + kPlThreads * q;
    if (r < n && r >= j0)
#pragma unroll
      for (int c = 0; c < kPlNb; ++c)
        if (c < w) S[c * ld + r] = v[q][c];
  }
}

__global__ void __launch_bounds__(kPlThreads, 1) k_lu_persistent(PlArgs a) {
  extern __shared__ double S[];  // kPlNb columns x ldS rows (column-major)
  __shared__ double sT[kPlNb][kPlNb + 1];
  __shared__ double cval[kPlWarps];
  __shared__ int cidx[kPlWarps];
  __shared__ int spiv[kPlNb];
  __shared__ double prow[kPlNb], grow[kPlNb];
  const int j = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int n = a.n, ld = a.ldS;
  const bool rhs = j >= a.nbA;
  const int c0 = rhs ? (j - a.nbA) * kPlNb : j * kPlNb;
  const int w = rhs ? min(kPlNb, a.nrhs - c0) : min(kPlNb, n - c0);
  double* G = rhs ? a.B + (int64_t)c0 * a.ldb : a.A + (int64_t)c0 * a.lda;
  const int64_t gld = rhs ? a.ldb : a.lda;
  for (int idx = tid; idx < kPlNb * n; idx += kPlThreads) {
    const int c = idx / n, r = idx - c * n;
    S[c * ld + r] = c < w ? G[(int64_t)c * gld + r] : 0.0;
  }
  __syncthreads();
  // ---- updates from the panels to the left
  const int kend = rhs ? a.nbA : j;
  PL_PROBE(0);
  for (int k = 0; k < kend; ++k) {
    if (k == kend - 1) PL_PROBE(1);
    pl_wait(a.flag + k);
    if (k == kend - 1) PL_PROBE(2);
    const int k0 = k * kPlNb, kw = min(kPlNb, n - k0);
    if (tid < kPlNb) spiv[tid] = tid < kw ? __ldcg(a.piv + k0 + tid) : k0 + tid;
    for (int e = tid; e < kPlNb * kPlNb; e += kPlThreads) {  // L_kk (unit lower)
      const int r = e % kPlNb, c = e / kPlNb;
      sT[r][c] = (c < r && r < kw) ? __ldcg(a.A + (int64_t)(k0 + c) * a.lda + k0 + r) : 0.0;
    }
    __syncthreads();
    if (tid < kPlNb) {  // this panel's row interchanges, in order (laswp)
      for (int i = 0; i < kw; ++i) {
        const int p = spiv[i];
        if (p != k0 + i) {
          const double tmp = S[tid * ld + k0 + i];
          S[tid * ld + k0 + i] = S[tid * ld + p];
          S[tid * ld + p] = tmp;
        }
      }
      // U_kj = L_kk^{-1} A_kj: the same thread's column, no barrier needed
    }
    if (tid < kPlNb) {
      double x[kPlNb];
#pragma unroll
      for (int i = 0; i < kPlNb; ++i) x[i] = i < kw ? S[tid * ld + k0 + i] : 0.0;
#pragma unroll
      for (int i = 1; i < kPlNb; ++i)
#pragma unroll
        for (int q = 0; q < i; ++q) x[i] = fma(-sT[i][q], x[q], x[i]);
#pragma unroll
      for (int i = 0; i < kPlNb; ++i)
        if (i < kw) S[tid * ld + k0 + i] = x[i];
    }
    __syncthreads();
    pl_gemm(S, ld, a.A, a.lda, k0 + kw, n, k0, kw);
    __syncthreads();
  }
  if (!rhs) {
    // ---- factor this panel: rows j0.., columns 0..w-1; thread tid owns rows tid + 512 m
    PL_PROBE(3);
    const int j0 = c0;
    if (n <= kPlThreads * kPlRpt) {
      pl_panel_reg(S, ld, n, j0, w, a.piv, reinterpret_cast<unsigned long long*>(cval), cidx, prow, grow);
    } else {
      for (int c = 0; c < w; ++c) {
        const int gr = j0 + c;
        unsigned long long key = 0ull;
        int bi = 0x7fffffff;
        for (int r = tid; r < n; r += kPlThreads) {
          const unsigned long long kq = pl_key(S[c * ld + r], r >= gr);
          if (kq > key) { key = kq; bi = r; }  // rows ascend: ties keep the first
        }
        unsigned long long* ckey = reinterpret_cast<unsigned long long*>(cval);
        pl_warp_argmax(key, bi, key, bi);
        if (lane == 0) { ckey[wid] = key; cidx[wid] = bi; }
        __syncthreads();
        pl_warp_argmax(ckey[lane & (kPlWarps - 1)], cidx[lane & (kPlWarps - 1)], key, bi);
        const int p = (key == 0ull || bi == 0x7fffffff) ? gr : bi;  // an all-NaN column pivots on itself
        if (tid < kPlNb && p != gr) {
          const double tmp = S[tid * ld + gr];
          S[tid * ld + gr] = S[tid * ld + p];
          S[tid * ld + p] = tmp;
        }
        if (tid == 0) a.piv[gr] = p;
        __syncthreads();
        const double d = S[c * ld + gr];
        if (d != 0.0) {
          const double inv = 1.0 / d;
          for (int r = tid; r < n; r += kPlThreads)
            if (r > gr) {
              const double l = S[c * ld + r] * inv;
              S[c * ld + r] = l;
#pragma unroll
              for (int c2 = 0; c2 < kPlNb; ++c2)
                if (c2 > c && c2 < w) S[c2 * ld + r] = fma(-l, S[c2 * ld + gr], S[c2 * ld + r]);
            }
        }
        // no trailing barrier: the next column's search reads only this thread's
        // own rows; the pivot row it broadcasts is swapped before the next barrier
      }
    }
    __syncthreads();
    for (int idx = tid; idx < kPlNb * n; idx += kPlThreads) {
      const int c = idx / n, r = idx - c * n;
      if (c < w) G[(int64_t)c * gld + r] = S[c * ld + r];  // U blocks above, this panel's LU below
    }
    PL_PROBE(4);
    pl_signal(a.flag + j);
    // ---- the later panels' interchanges reach this block column's L rows
    for (int k = j + 1; k < a.nbA; ++k) {
      pl_wait(a.flag + k);
      const int k0 = k * kPlNb, kw = min(kPlNb, n - k0);
      if (tid < kPlNb) spiv[tid] = tid < kw ? __ldcg(a.piv + k0 + tid) : k0 + tid;
      __syncthreads();
      if (tid < w)
        for (int i = 0; i < kw; ++i) {
          const int p = spiv[i];
          if (p != k0 + i) {
            const double tmp = S[tid * ld + k0 + i];
            S[tid * ld + k0 + i] = S[tid * ld + p];
            S[tid * ld + p] = tmp;
          }
        }
    }
    // every reader of this panel's L is done once all later block columns have
    // published (A) or finished their forward updates (B)
    for (int m = a.nbA; m < a.ncb; ++m) pl_wait(a.flag + m);
    __syncthreads();
    for (int idx = tid; idx < kPlNb * n; idx += kPlThreads) {
      const int c = idx / n, r = idx - c * n;
      if (c < w && r >= j0 + kPlNb) G[(int64_t)c * gld + r] = S[c * ld + r];
    }
    PL_PROBE(5);
    pl_signal(a.fin + j);
    return;
  }
  // ---- right-hand sides: S = L^{-1} P B; now U X = S, block rows from the bottom
  PL_PROBE(3);
  pl_signal(a.flag + j);
  for (int m = 0; m < a.nbA; ++m) pl_wait(a.fin + m);
  PL_PROBE(4);
  for (int J = a.nbA - 1; J >= 0; --J) {
    const int b0 = J * kPlNb, bw = min(kPlNb, n - b0);
    for (int e = tid; e < kPlNb * kPlNb; e += kPlThreads) {  // U_JJ (upper, with the diagonal)
      const int r = e % kPlNb, c = e / kPlNb;
      sT[r][c] = (r <= c && c < bw) ? __ldcg(a.A + (int64_t)(b0 + c) * a.lda + b0 + r) : 0.0;
    }
    __syncthreads();
    if (tid < w) {
      double x[kPlNb];
#pragma unroll
      for (int i = 0; i < kPlNb; ++i) x[i] = i < bw ? S[tid * ld + b0 + i] : 0.0;
#pragma unroll
      for (int i = kPlNb - 1; i >= 0; --i) {
        if (i < bw) {
#pragma unroll
          for (int q = i + 1; q < kPlNb; ++q) x[i] = fma(-sT[i][q], x[q], x[i]);
          x[i] = x[i] / sT[i][i];
        }
      }
#pragma unroll
      for (int i = 0; i < kPlNb; ++i)
        if (i < bw) S[tid * ld + b0 + i] = x[i];
    }
    __syncthreads();
    pl_gemm(S, ld, a.A, a.lda, 0, b0, b0, bw);
    __syncthreads();
  }
  for (int idx = tid; idx < kPlNb * n; idx += kPlThreads) {
    const int c = idx / n, r = idx - c * n;
    if (c < w) G[(int64_t)c * gld + r] = S[c * ld + r];
  }
  PL_PROBE(5);
}

// Pivot-floor test of a stored factor: info[0] = first i with |U_ii| <= 1e-14
// ||A||_F (or -1), info[1] = |U_ii|, info[2] = the floor (linalg.py:91-98).
__global__ void __launch_bounds__(1024) k_lu_check(const double* A, int64_t ld, int n, const double* fro,
                                                   double* info) {
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0x7fffffff;
  __syncthreads();
  const double floor = 1e-14 * fro[0];
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (fabs(A[(int64_t)i * ld + i]) <= floor) atomicMin(&s_bad, i);
  __syncthreads();
  if (threadIdx.x == 0) {
    info[0] = (s_bad == 0x7fffffff) ? -1.0 : (double)s_bad;
    info[1] = (s_bad == 0x7fffffff) ? 0.0 : fabs(A[(int64_t)s_bad * ld + s_bad]);
    info[2] = floor;
  }
}

size_t pl_smem(int n) { return (size_t)kPlNb * (((n + 7) & ~7) + 4) * 8; }

// The persistent LU applies when every block column fits one co-resident CTA.
bool pl_fits(int64_t n, int64_t nrhs) {
  if (n < 1 || n > 4096 || nrhs < 0) return false;
  const int64_t ncb = ceil_div(n, kPlNb) + ceil_div(nrhs, kPlNb);
  const size_t smem = pl_smem((int)n);
  if (smem > max_smem_optin()) return false;
  static PerDevice<int> occ_cache;
  int& occ = occ_cache.get();
  static PerDevice<size_t> cfg;
  if (cfg.get() < smem) {
    STROM_CUDA(cudaFuncSetAttribute(k_lu_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cfg.get() = smem;
  }
  int o = 0;
  STROM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_lu_persistent, kPlThreads, smem));
  occ = o;
  if (getenv("STROM_LU_LEGACY")) return false;
  return (int64_t)o * sm_count() >= ncb;
}

long long* g_lu_probe = nullptr;  // strom_debug_lu_probe

// LU of A (and, with nrhs > 0, the solve A X = B in place) by the persistent kernel.
void pl_run(int64_t n, double* A, int64_t lda, double* B, int64_t ldb, int64_t nrhs, int* piv, cudaStream_t s) {
  const int nbA = (int)ceil_div(n, kPlNb);
  const int ncb = nbA + (int)ceil_div(nrhs, kPlNb);
  auto flags = dev_alloc((size_t)(ncb + nbA) * 4, s, true);
  PlArgs a;
  a.A = A; a.lda = lda; a.B = B; a.ldb = ldb;
  a.n = (int)n; a.nrhs = (int)nrhs; a.nbA = nbA; a.ncb = ncb; a.ldS = (((int)n + 7) & ~7) + 4;
  a.piv = piv;
  a.flag = flags->as<int>();
  a.fin = flags->as<int>() + ncb;
  a.probe = g_lu_probe;
  void* args[] = {&a};
  ProfScope ps(P_LU, s);
  STROM_CUDA(cudaLaunchCooperativeKernel((const void*)k_lu_persistent, dim3(ncb), dim3(kPlThreads), args,
                                         pl_smem((int)n), s));
}

// Blocked right-looking LU with partial pivoting of the n x n column-major a (in place).
void lu_factor(int64_t n, double* a_dev, int* piv, cudaStream_t s) {
  if (pl_fits(n, 0)) {
    pl_run(n, a_dev, n, nullptr, 0, 0, piv, s);
    return;
  }
  const bool reg_panel = n <= 1024;  // panel rows fit two per thread (512 threads) in registers
  const int step = reg_panel ? kNbReg : kNb;
  for (int64_t k0 = 0; k0 < n; k0 += step) {
    const int nb = (int)std::min<int64_t>(step, n - k0);
    if (reg_panel) {
      if (n - k0 <= 512) lu_launch(k_lu_panel_reg<1>, dim3(1), dim3(512), s, a_dev, (int64_t)n, (int)n, (int)k0, nb, piv);
      else lu_launch(k_lu_panel_reg<2>, dim3(1), dim3(512), s, a_dev, (int64_t)n, (int)n, (int)k0, nb, piv);
      if (n > nb)  // interchanges outside the panel + TRSM, one launch
        lu_launch(k_lu_swap_trsm, dim3((unsigned)ceil_div(n - nb, 64)), dim3(64), s, a_dev, (int64_t)n, (int)n,
                  (int)k0, nb, (const int*)piv);
    } else {
      k_lu_panel<<<1, 1024, 0, s>>>(a_dev, n, (int)n, (int)k0, nb, piv);
      STROM_LAUNCH_CHECK();
    }
    const int64_t rest = n - k0 - nb;
    if (rest > 0) {
      if (!reg_panel) {
        k_lu_trsm<<<(unsigned)ceil_div(rest, 128), 128, 0, s>>>(a_dev, n, (int)n, (int)k0, nb);
        STROM_LAUNCH_CHECK();
      }
      dim3 g((unsigned)ceil_div(rest, 64), (unsigned)ceil_div(rest, 64));
      lu_launch(k_lu_gemm, g, dim3(256), s, a_dev, (int64_t)n, (int)n, (int)k0, nb);
    }
  }
}

// Pivot-floor check (floor = 1e-14 fro[0]; fro NULL: no check) and the two
// triangular solves of nrhs columns of x (ldx).
void lu_solve(int64_t n, const double* a_dev, const int* piv, double* x_dev, int64_t ldx, int64_t nrhs,
              const double* fro, double* info, cudaStream_t s) {
  if ((size_t)n * 8 <= 96 * 1024) {
    static PerDevice<bool> cfgs;
    bool& cfg = cfgs.get();
    if (!cfg) {
      STROM_CUDA(cudaFuncSetAttribute(k_lu_solve_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
      cfg = true;
    }
    k_lu_solve_cta<<<1, 512, (size_t)n * 8, s>>>(a_dev, n, (int)n, piv, x_dev, ldx, (int)nrhs, fro, info);
  } else {
    k_lu_solve<<<1, 1024, 0, s>>>(a_dev, n, (int)n, piv, x_dev, ldx, (int)nrhs, fro, info);
  }
  STROM_LAUNCH_CHECK();
}

}  // namespace

extern "C" {

// LU of the n x n column-major a_dev in place (pivots in piv_dev, n ints) and
// the solves with a stored factor -- the reference's StepSolver pattern
// (system.py:106-125: factor once per dt, solve per step).  Asynchronous; no
// pivot-floor test (a singular factor yields non-finite solutions).
int strom_dense_lu(int64_t n, double* a_dev, int32_t* piv_dev, void* stream) {
  return guarded([&] {
    STROM_REQUIRE(n >= 1 && a_dev && piv_dev, "bad LU arguments");
    lu_factor(n, a_dev, piv_dev, reinterpret_cast<cudaStream_t>(stream));
  });
}

int strom_dense_lu_solve(int64_t n, const double* lu_dev, const int32_t* piv_dev, double* x_dev, int64_t nrhs,
                         void* stream) {
  return guarded([&] {
    STROM_REQUIRE(n >= 1 && lu_dev && piv_dev && x_dev && nrhs >= 0, "bad LU-solve arguments");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    auto info = dev_alloc(3 * 8, s, false);
    lu_solve(n, lu_dev, piv_dev, x_dev, n, nrhs, nullptr, info->as<double>(), s);
  });
}


// LU factorization with partial pivoting of A (n x n, column-major, in place)
// and solve for nrhs right-hand sides X (in place).  On a pivot with
// |U_ii| <= 1e-14 ||A||_F returns STROM_ESINGULAR ("pivot i") -- synchronizes.
// piv_dev may be NULL; info_dev (3 doubles) may be NULL.
int strom_dense_solve(int64_t n, double* a_dev, double* x_dev, int64_t nrhs, int32_t* piv_dev,
                      double* info_dev, void* stream) {
  return guarded([&] {
    STROM_REQUIRE(n >= 1 && a_dev && x_dev && nrhs >= 0, "bad solve arguments");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    auto scratch = dev_alloc(8 * 8 + (size_t)n * 4, s, true);
    double* fro = scratch->as<double>();  // [0] ||A||_F, [1] ||B||_F (NaN: non-finite entry)
    double* info = info_dev ? info_dev : fro + 2;
    int* piv = piv_dev ? piv_dev : reinterpret_cast<int*>(fro + 8);
    {
      const int np = 256;
      auto fp = dev_alloc((size_t)2 * np * 8, s, false);
      k_fro_part<<<np, 256, 0, s>>>(a_dev, n, n, n, fp->as<double>());
      k_fro_final<<<1, 256, 0, s>>>(fp->as<double>(), np, fro);
      k_fro_part<<<np, 256, 0, s>>>(x_dev, n, n, nrhs, fp->as<double>() + np);
      k_fro_final<<<1, 256, 0, s>>>(fp->as<double>() + np, np, fro + 1);
      STROM_LAUNCH_CHECK();
    }
    if (pl_fits(n, nrhs)) {  // factor + forward + backward solve in one persistent launch
      pl_run(n, a_dev, n, x_dev, n, nrhs, piv, s);
      k_lu_check<<<1, 1024, 0, s>>>(a_dev, n, (int)n, fro, info);
      STROM_LAUNCH_CHECK();
    } else {
      lu_factor(n, a_dev, piv, s);
      lu_solve(n, a_dev, piv, x_dev, n, nrhs, fro, info, s);
    }
    double h[3], nf[2];
    STROM_CUDA(cudaMemcpyAsync(h, info, 3 * 8, cudaMemcpyDeviceToHost, s));
    STROM_CUDA(cudaMemcpyAsync(nf, fro, 2 * 8, cudaMemcpyDeviceToHost, s));
    STROM_CUDA(cudaStreamSynchronize(s));
    // scipy.linalg.lu_factor / lu_solve (check_finite=True), linalg.py:90,99
    if (!std::isfinite(nf[0]) || !std::isfinite(nf[1]))
      throw Error(kInvalidArgument, "array must not contain infs or NaNs");
    if (h[0] >= 0.0) {
      char buf[160];
      snprintf(buf, sizeof(buf), "matrix numerically singular: pivot %lld is %.3e (floor %.3e)",
               (long long)h[0], h[1], h[2]);
      throw Error(kSingularMatrix, buf);
    }
  });
}

// Diagnostics: 8 globaltimer stamps per CTA of the persistent LU into dev_buf
// (ncb x 8 int64), or NULL to disable.
void strom_debug_lu_probe(long long* dev_buf) { g_lu_probe = dev_buf; }

// Positive-diagonal thin QR of M (rows x cols, column-major, ld) in place
// (M <- Q); R (cols x cols, column-major) receives the matching R.
int strom_qr(int64_t rows, int64_t cols, double* m_dev, int64_t ld, double* r_dev, void* stream) {
  return guarded([&] {
    STROM_REQUIRE(rows >= cols && cols >= 1 && m_dev && r_dev, "need rows >= cols");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    auto work = dev_alloc((size_t)2 * cols * 8, s, false);
    k_qr<<<1, 1024, 0, s>>>(m_dev, ld, (int)rows, (int)cols, r_dev, work->as<double>());
    STROM_LAUNCH_CHECK();
  });
}

}  // extern "C"
