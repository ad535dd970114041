// Device-side workload generator for the capacity configuration (BASELINE
// configs[4]): a low-rank-plus-noise snapshot stream too large for host memory
// (2^26 rows x 1000 snapshots = 537 GB) and too large to keep its factor Q
// resident next to the iSVD store.
//
//   X[:, t] = Q diag(sigma) W[t, :]^T + E[:, t]
//   Q[i, c] = s_i H(i, p_c) / sqrt(n)      (randomized Hadamard: orthonormal
//                                            columns, never stored; n = 2^m)
//   H(i, p)  = (-1)^popcount(i & p),  s_i = +-1 from a hash of (seed, i),
//   p_c      = distinct Hadamard rows,  E = noise * N(0, 1) from a counter hash.
//
// The caller passes coef[c * nb + b] = sigma_c W[t0 + b, c] (rank x nb,
// row-major) and receives nb columns (n x nb, column-major, leading dim ldo).  Test and bench support, not
// a reference interface.
#include <cstdint>

#include "../../include/strom_b200.h"
#include "common.cuh"
#include "runtime.cuh"

using namespace strom;

namespace {

constexpr int kGenMaxRank = 128;
constexpr int kGenMaxCols = 16;

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// standard normal from a 64-bit counter (Box-Muller on two 24-bit uniforms)
__device__ __forceinline__ float counter_normal(uint64_t key) {
  const uint64_t h = splitmix64(key);
  const float u1 = ((float)(h >> 40) + 0.5f) * (1.0f / 16777216.0f);
  const float u2 = ((float)((h >> 16) & 0xFFFFFF) + 0.5f) * (1.0f / 16777216.0f);
  return sqrtf(-2.0f * __logf(u1)) * __cosf(6.28318530718f * u2);
}

template <int NB>
__global__ void __launch_bounds__(256) k_gen_lowrank(int64_t n, int rank, const double* __restrict__ coef,
                                                     const int64_t* __restrict__ prow, uint64_t seed, int64_t t0,
                                                     double noise, double scale, double* __restrict__ out,
                                                     int64_t ldo) {
  __shared__ double sc[kGenMaxRank * NB];
  __shared__ int64_t sp[kGenMaxRank];
  for (int e = threadIdx.x; e < rank * NB; e += blockDim.x) sc[e] = coef[e];
  for (int e = threadIdx.x; e < rank; e += blockDim.x) sp[e] = prow[e];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) acc[b] = 0.0;
    for (int c = 0; c < rank; ++c) {
      const bool neg = __popcll((unsigned long long)(i & sp[c])) & 1;
#pragma unroll
      for (int b = 0; b < NB; ++b) acc[b] += neg ? -sc[c * NB + b] : sc[c * NB + b];
    }
    const double si = (splitmix64(seed ^ 0x5bd1e995ull ^ (uint64_t)i) & 1) ? -scale : scale;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const uint64_t key = (seed * 0x100000001B3ull) ^ ((uint64_t)(t0 + b) << 40) ^ (uint64_t)i;
      out[(int64_t)b * ldo + i] = si * acc[b] + noise * (double)counter_normal(key);
    }
  }
}

}  // namespace

extern "C" {

int strom_gen_lowrank_batch(int64_t n, int32_t rank, int32_t nb, const double* coef_dev, const int64_t* prow_dev,
                            uint64_t seed, int64_t t0, double noise, double* out_dev, int64_t ldo, void* stream) {
  return guarded([&] {
    STROM_REQUIRE(n >= 2 && (n & (n - 1)) == 0, "the randomized-Hadamard generator needs n = 2^m");
    STROM_REQUIRE(rank >= 1 && rank <= kGenMaxRank, "generator rank must be 1..128");
    STROM_REQUIRE(nb >= 1 && nb <= kGenMaxCols && ldo >= n, "generator batch must be 1..16 columns");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const double scale = 1.0 / sqrt((double)n);
    const int grid = sm_count() * 8;
    switch (nb) {
#define GEN_CASE(B)                                                                                         \
  case B:                                                                                                   \
    k_gen_lowrank<B><<<grid, 256, 0, s>>>(n, rank, coef_dev, prow_dev, seed, t0, noise, scale, out_dev, ldo); \
    break;
      GEN_CASE(1) GEN_CASE(2) GEN_CASE(4) GEN_CASE(8) GEN_CASE(16)
#undef GEN_CASE
      default:
        throw Error(kInvalidArgument, "generator batch must be 1, 2, 4, 8 or 16 columns");
    }
    STROM_LAUNCH_CHECK();
  });
}

}  // extern "C"
