// fp64 tensor-core MMA for sm_100a.  tcgen05 has no f64 kind, so fp64 tensor
// math on Blackwell is the warp-level mma.sync m8n8k4 (SASS: DMMA.884).
//
// Fragment layout (one warp, g = lane >> 2, t = lane & 3):
//   A (8x4, row-major)   a  = A[g][t]
//   B (4x8, col-major)   b  = B[t][g]
//   C/D (8x8)            c0 = C[g][2t], c1 = C[g][2t+1]
#pragma once

#include "common.cuh"

namespace strom {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

}  // namespace strom
