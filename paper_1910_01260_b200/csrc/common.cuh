// Shared device helpers for the strom B200 kernels (sm_100a, fp64 throughout).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>

namespace strom {

constexpr int kWarp = 32;
constexpr int kNumSM = 148;

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// A tall matrix: element (i, j) at p[(i >> tshift) * ts + j * cs + (i & (2^tshift - 1))].
// Column-major (ld) is tshift = 40, ts = 0, cs = ld; the iSVD store U is
// row-tiled: 64-row tiles, each holding its ccap column segments contiguously.
constexpr int kUTileShift = 6;
constexpr int kUTile = 1 << kUTileShift;  // rows per U tile
struct Tall {
  double* p;
  int64_t ts, cs;
  int32_t tshift;
  __host__ __device__ __forceinline__ int64_t off(int64_t i, int64_t j) const {
    return (i >> tshift) * ts + j * cs + (i & ((int64_t(1) << tshift) - 1));
  }
};
inline Tall tall_cm(const double* p, int64_t ld) { return Tall{const_cast<double*>(p), 0, ld, 40}; }
inline Tall tall_tiled(const double* p, int64_t ccap) {
  return Tall{const_cast<double*>(p), (int64_t)kUTile * ccap, kUTile, kUTileShift};
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Deterministic block-wide sum (fixed tree).  `red` needs blockDim.x/32 doubles.
// Every thread gets the result.  Contains two __syncthreads.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = (lane < nw) ? red[lane] : 0.0;
  t = warp_sum(t);
  return t;
}

__device__ __forceinline__ double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = (lane < nw) ? red[lane] : -INFINITY;
  return warp_max(t);
}

}  // namespace strom
