// Microbenchmark: dependent-issue latency of DFMA / DADD / MUFU.RCP64H+Newton / SHFL and
// the per-SM DFMA throughput at 1..16 warps (one CTA).  nvcc -arch=sm_100a -o tools/bin/fp64_lat tools/fp64_lat.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_chain(int iters, double* out, long long* cyc, int mode) {
  double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-12, c = 1e-13;
  double a2 = a + 1, a3 = a + 2, a4 = a + 3;
  __syncthreads();
  long long t0 = clock64();
  if (mode == 0) {
#pragma unroll 16
    for (int i = 0; i < iters; ++i) a = fma(a, b, c);
  } else if (mode == 1) {
#pragma unroll 16
    for (int i = 0; i < iters; ++i) a = a + c;
  } else if (mode == 2) {
#pragma unroll 4
    for (int i = 0; i < iters; ++i) a = __drcp_rn(a) + 0.5;
  } else if (mode == 3) {
#pragma unroll 16
    for (int i = 0; i < iters; ++i) a = __shfl_xor_sync(0xffffffffu, a, 1);
  } else if (mode == 4) {  // 4 independent chains
#pragma unroll 4
    for (int i = 0; i < iters; ++i) { a = fma(a, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c); a4 = fma(a4, b, c); }
  } else if (mode == 5) {
#pragma unroll 4
    for (int i = 0; i < iters; ++i) a = 1.0 / a + 0.5;
  } else if (mode == 6) {
#pragma unroll 4
    for (int i = 0; i < iters; ++i) a = sqrt(a) + 0.5;
  }
  else if (mode == 7) {  // 4 independent chains, only the low half of every warp active
    if ((threadIdx.x & 31) < 16) {
#pragma unroll 4
      for (int i = 0; i < iters; ++i) { a = fma(a, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c); a4 = fma(a4, b, c); }
    }
  } else if (mode == 8) {  // 4 independent chains, lanes 0-7 only
    if ((threadIdx.x & 31) < 8) {
#pragma unroll 4
      for (int i = 0; i < iters; ++i) { a = fma(a, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c); a4 = fma(a4, b, c); }
    }
  } else if (mode == 9) {  // 4 chains, two of them predicated off by a runtime flag
    const bool pr = out[0] == 12345.0;
#pragma unroll 4
    for (int i = 0; i < iters; ++i) {
      a = fma(a, b, c); a2 = fma(a2, b, c);
      if (pr) { a3 = fma(a3, b, c); a4 = fma(a4, b, c); }
    }
  } else if (mode == 10) {  // even lanes only
    if ((threadIdx.x & 1) == 0) {
#pragma unroll 4
      for (int i = 0; i < iters; ++i) { a = fma(a, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c); a4 = fma(a4, b, c); }
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = a + a2 + a3 + a4;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 8 * 1024); cudaMalloc(&cyc, 8);
  const char* names[] = {"DFMA chain", "DADD chain", "drcp_rn+add chain", "SHFL64 chain", "4x DFMA indep", "div+add chain", "sqrt+add chain", "4x DFMA lanes<16", "4x DFMA lanes<8", "4x DFMA 2 pred-off", "4x DFMA even lanes"};
  for (int mode = 0; mode < 11; ++mode)
    for (int warps : {1, 4, 8, 16}) {
      const int iters = 4096;
      k_chain<<<1, 32 * warps>>>(iters, out, cyc, mode);
      k_chain<<<1, 32 * warps>>>(iters, out, cyc, mode);
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("%-20s warps %2d: %.1f cycles / iteration\n", names[mode], warps, (double)c / iters);
    }
  return 0;
}
