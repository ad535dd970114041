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

#include "../../include/strom_b200.h"
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

// out (ns x q, row-major) = sum over CTAs of the partials, in CTA order.
__global__ void k_spatial_reduce(const double* part, int nparts, int MA, int NQ, int ns, int q, double* out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= ns * q) return;
  const int a = idx / q, b = idx % q;
  double s = 0.0;
  for (int p = 0; p < nparts; ++p) s += part[(int64_t)p * MA * NQ + a * NQ + b];
  out[idx] = s;
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
  static bool configured = false;
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

template <typename IdxT>
int launch_spatial(SpatialArgs<IdxT> a, int max_grid, cudaStream_t s) {
  const int TA = a.MA / 8, TB = a.NQ / 8;
  if (TA <= 8 && TB <= 8) return launch_spatial_t<IdxT, 1, 8>(a, max_grid, s);
  if (TA <= 8 && TB <= 17) return launch_spatial_t<IdxT, 1, 17>(a, max_grid, s);
  if (TA <= 16 && TB <= 17) return launch_spatial_t<IdxT, 2, 17>(a, max_grid, s);
  throw Error(kInvalidArgument, "spatial reduction supports n_s <= 128 and <= 136 right columns");
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
    k_spatial_reduce<<<(unsigned)ceil_div((int64_t)ns * q, 256), 256, 0, s>>>(part->as<double>(), grid, MA, NQ,
                                                                              (int)ns, q, out_dev);
    STROM_LAUNCH_CHECK();
  });
}

}  // extern "C"
