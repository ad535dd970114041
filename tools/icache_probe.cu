// Microbenchmark: cycles per instruction of straight-line code executed once (cold instruction
// fetch) against the same code executed again inside the kernel (warm), for 1 and 16 warps.
// nvcc -arch=sm_100a -o tools/bin/icache_probe tools/icache_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int N>
__device__ __forceinline__ void body(unsigned& a, unsigned& b, unsigned& c, unsigned& d, unsigned k) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    a = a * k + b; b = b * k + c; c = c * k + d; d = d * k + a;
  }
}
template <int N>
__global__ void k_probe(unsigned k, unsigned* out, long long* cyc, int reps) {
  unsigned a = threadIdx.x, b = 1, c = 2, d = 3;
  __syncthreads();
  for (int r = 0; r < reps; ++r) {
    long long t0 = clock64();
    body<N>(a, b, c, d, k);
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[r] = t1 - t0;
    __syncthreads();
  }
  out[threadIdx.x] = a + b + c + d;
}
template <int N>
void run(const char* name) {
  unsigned* out; long long* cyc;
  cudaMalloc(&out, 4096); cudaMalloc(&cyc, 64);
  for (int warps : {1, 16}) {
    for (int launch = 0; launch < 2; ++launch) {
      k_probe<N><<<1, 32 * warps>>>(3u, out, cyc, 3);
      long long c[3]; cudaMemcpy(c, cyc, 24, cudaMemcpyDeviceToHost);
      printf("%s (%d IMADs) warps %2d launch %d: first pass %.2f cyc/instr, second %.2f, third %.2f\n", name, 4 * N,
             warps, launch, (double)c[0] / (4 * N), (double)c[1] / (4 * N), (double)c[2] / (4 * N));
    }
  }
}
int main() {
  run<256>("1k");
  run<1024>("4k");
  run<4096>("16k");
  return 0;
}
