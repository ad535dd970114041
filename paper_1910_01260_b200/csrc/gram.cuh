// Tall-skinny Gram G = A^T A (A: n x q, column-major or row-tiled, q <= 128) on the fp64
// tensor cores (DMMA m8n8k4).  Used to measure the exact Gram of a freshly
// compacted U (so the small-space Cholesky factor L describes the stored U,
// not an assumed identity) and when loading a state from an explicit phi.
#pragma once

#include "common.cuh"
#include "dmma.cuh"

namespace strom {

constexpr int kGramRows = 32;
constexpr int kGramLd = kGramRows + 4;

template <int TAW, int TBM>
__global__ void __launch_bounds__(256) k_tall_gram(Tall A, const int32_t* col0_dev, const int32_t* q_dev, int q_fixed,
                                                   int64_t n, double* __restrict__ part, int QP) {
  extern __shared__ double gsm[];  // QP x kGramLd
  const int q = q_dev ? *q_dev : q_fixed;
  const int col0 = col0_dev ? *col0_dev : 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int T8 = (q + 7) / 8;
  const int64_t ntiles = ceil_div(n, kGramRows);
  const int64_t per = ceil_div(ntiles, gridDim.x);
  const int64_t t0 = blockIdx.x * per, t1 = min(ntiles, t0 + per);
  double acc[TAW][TBM][2];
#pragma unroll
  for (int x = 0; x < TAW; ++x)
#pragma unroll
    for (int y = 0; y < TBM; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  for (int64_t tile = t0; tile < t1; ++tile) {
    const int64_t row0 = tile * kGramRows;
    __syncthreads();
    for (int idx = threadIdx.x; idx < kGramRows * T8 * 8; idx += blockDim.x) {
      const int i = idx % kGramRows, a = idx / kGramRows;
      const int64_t row = row0 + i;
      gsm[a * kGramLd + i] = (row < n && a < q) ? __ldg(A.p + A.off(row, col0 + a)) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kGramRows / 4; ++kk) {
      const int kr = kk * 4 + t;
#pragma unroll
      for (int x = 0; x < TAW; ++x) {
        const int ta = wid + 8 * x;
        if (ta < T8) {
          const double av = gsm[(ta * 8 + g) * kGramLd + kr];
#pragma unroll
          for (int y = 0; y < TBM; ++y) {
            if (y < T8) {
              const double bv = gsm[(y * 8 + g) * kGramLd + kr];
              dmma884(acc[x][y][0], acc[x][y][1], av, bv);
            }
          }
        }
      }
    }
  }
  double* mp = part + (int64_t)blockIdx.x * QP * QP;
#pragma unroll
  for (int x = 0; x < TAW; ++x) {
    const int ta = wid + 8 * x;
    if (ta >= T8) continue;
#pragma unroll
    for (int y = 0; y < TBM; ++y) {
      if (y >= T8) continue;
      const int r = ta * 8 + g, c = y * 8 + 2 * t;
      mp[r * QP + c] = acc[x][y][0];
      mp[r * QP + c + 1] = acc[x][y][1];
    }
  }
}

// G (q x q, column-major, ld) = sum of the partials in CTA order (symmetrised).
__global__ void k_gram_reduce(const double* part, int nparts, int QP, const int32_t* q_dev, int q_fixed,
                              double* G, int ldg) {
  const int q = q_dev ? *q_dev : q_fixed;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= q * q) return;
  const int a = idx % q, b = idx / q;
  const int i = a < b ? a : b, j = a < b ? b : a;  // use the upper entry for both halves
  double s = 0.0;
  for (int p = 0; p < nparts; ++p) s += part[(int64_t)p * QP * QP + i * QP + j];
  G[(int64_t)b * ldg + a] = s;
}

}  // namespace strom
