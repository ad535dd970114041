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
__global__ void __launch_bounds__(256) k_spatial(SpatialArgs<IdxT> A) {
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
        cidx[qq] = (qq < cnt) ? (int64_t)__ldg(A.indices + nz0 + qq) : 0;
        cval[qq] = (qq < cnt) ? __ldg(A.data + nz0 + qq) : 0.0;
      }
      for (int j = wid; j < A.NQ; j += 8) {
        double s = 0.0;
        if (row < A.N) {
          if (j < A.ns) {
            const double* pj = A.phi + (int64_t)j * A.phi_cs;
#pragma unroll
            for (int qq = 0; qq < kNzReg; ++qq)
              if (qq < cnt) s = fma(cval[qq], __ldg(pj + cidx[qq] * A.phi_rs), s);
            for (int64_t nz = nz0 + kNzReg; nz < nz1; ++nz)
              s = fma(__ldg(A.data + nz), __ldg(pj + (int64_t)__ldg(A.indices + nz) * A.phi_rs), s);
          } else if (j < A.ns + A.ne) {
            s = __ldg(A.extra + (int64_t)(j - A.ns) * A.ext_ld + row);
          } else if (j < A.q) {  // A x_ref
#pragma unroll
            for (int qq = 0; qq < kNzReg; ++qq)
              if (qq < cnt) s = fma(cval[qq], __ldg(A.xref + cidx[qq]), s);
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

// out (ns x q, row-major) = sum over CTAs of the partials, in CTA order.
__global__ void k_spatial_reduce(const double* part, int nparts, int MA, int NQ, int ns, int q, double* out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= ns * q) return;
  const int a = idx / q, b = idx % q;
  double s = 0.0;
  for (int p = 0; p < nparts; ++p) s += part[(int64_t)p * MA * NQ + a * NQ + b];
  out[idx] = s;
}

template <typename IdxT, int TAW, int TBM>
void launch_spatial_t(SpatialArgs<IdxT> a, int grid, cudaStream_t s) {
  const size_t smem = (size_t)kLdK * (a.MA + a.NQ) * 8;
  static bool configured = false;
  if (!configured) {
    STROM_CUDA(cudaFuncSetAttribute(k_spatial<IdxT, TAW, TBM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    64 * 1024));
    configured = true;
  }
  ProfScope ps(P_SPATIAL, s);
  k_spatial<IdxT, TAW, TBM><<<grid, 256, smem, s>>>(a);
  STROM_LAUNCH_CHECK();
}

template <typename IdxT>
void launch_spatial(SpatialArgs<IdxT> a, int grid, cudaStream_t s) {
  const int TA = a.MA / 8, TB = a.NQ / 8;
  if (TA <= 8 && TB <= 8) launch_spatial_t<IdxT, 1, 8>(a, grid, s);
  else if (TA <= 8 && TB <= 17) launch_spatial_t<IdxT, 1, 17>(a, grid, s);
  else if (TA <= 16 && TB <= 17) launch_spatial_t<IdxT, 2, 17>(a, grid, s);
  else throw Error(kInvalidArgument, "spatial reduction supports n_s <= 128 and <= 136 right columns");
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
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int q = (int)(ns + ne + (xref_dev ? 1 : 0));
    const int MA = (int)round_up(ns, 8), NQ = (int)round_up(q, 8);
    const int64_t ntiles = ceil_div(n, kRows);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)sm_count() * 2));
    auto part = dev_alloc((size_t)grid * MA * NQ * 8, s, false);
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
      launch_spatial(a, grid, s);
    } else {
      SpatialArgs<int64_t> a{};
      fill(a);
      a.indptr = static_cast<const int64_t*>(indptr_dev);
      a.indices = static_cast<const int64_t*>(indices_dev);
      launch_spatial(a, grid, s);
    }
    k_spatial_reduce<<<(unsigned)ceil_div((int64_t)ns * q, 256), 256, 0, s>>>(part->as<double>(), grid, MA, NQ,
                                                                              (int)ns, q, out_dev);
    STROM_LAUNCH_CHECK();
  });
}

}  // extern "C"
