// Block-structured space-time reduced operator (reference spacetime.py:37-115)
// assembled without ever forming the space-time basis.
//
// With F (N_t x n_s n_t), F[k, j*n_s + i] = Psi_i[k, j]  (the diagonals of
// E_k^(j), spacetime.py:37-40):
//
//   A_st[(j',i), (j,i')] = -(F^T diag(dt) F)[(j',i), (j,i')] * A_hat[i, i']
//                          + delta_{i i'} (S - Cp)[i, j', j]
//   S[i,j',j]  = sum_k   Psi_i[k,j'] Psi_i[k,j]        (same-step)
//   Cp[i,j',j] = sum_k>0 Psi_i[k,j'] Psi_i[k-1,j]      (step coupling)
//
// The (n_s n_t)^2 temporal Gram runs on the fp64 tensor cores (DMMA m8n8k4)
// with the Hadamard-with-tiled-A_hat and the diagonal terms fused into the
// epilogue.  f_st (spacetime.py:72-99) and x0_st (spacetime.py:102-115) are
// O(n_s n_t N_t) and come from one small kernel.
#include <algorithm>

#include "../../include/strom_b200.h"
#include "dmma.cuh"
#include "runtime.cuh"

using namespace strom;

namespace {

// F and dt-scaled F, both N_t x NT row-major (k-major), NT = n_s * n_t.
__global__ void k_st_pack(const double* __restrict__ psi, const double* __restrict__ dt, int nsteps, int ns,
                          int nt, int kpad, double* __restrict__ F, double* __restrict__ Fd) {
  const int NT = ns * nt;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)kpad * NT) return;
  const int k = (int)(idx / NT), col = (int)(idx % NT);
  const int j = col / ns, i = col % ns;
  double v = 0.0, vd = 0.0;
  if (k < nsteps) {
    v = psi[((int64_t)i * nsteps + k) * nt + j];
    vd = dt[k] * v;
  }
  F[idx] = v;
  Fd[idx] = vd;
}

// D[i, j', j] = S - Cp  (n_s x n_t x n_t)
__global__ void k_st_diag(const double* __restrict__ psi, int nsteps, int ns, int nt, double* __restrict__ D) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= ns * nt * nt) return;
  const int i = idx / (nt * nt), jp = (idx / nt) % nt, j = idx % nt;
  const double* p = psi + (int64_t)i * nsteps * nt;
  double same = 0.0, coup = 0.0;
  for (int k = 0; k < nsteps; ++k) same = fma(p[(int64_t)k * nt + jp], p[(int64_t)k * nt + j], same);
  for (int k = 1; k < nsteps; ++k) coup = fma(p[(int64_t)k * nt + jp], p[(int64_t)(k - 1) * nt + j], coup);
  D[idx] = same - coup;
}

// f_st and x0_st.  Thread per (j, i).  f: constant -> m values; else N_t x m.
__global__ void k_st_vecs(const double* __restrict__ psi, const double* __restrict__ dt, int nsteps, int ns,
                          int nt, const double* __restrict__ bhat, int m, const double* __restrict__ f,
                          int constant_input, const double* __restrict__ x0hat, double* __restrict__ fst,
                          double* __restrict__ x0st) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= ns * nt) return;
  const int j = idx / ns, i = idx % ns;
  const double* p = psi + (int64_t)i * nsteps * nt;
  double out = 0.0;
  if (constant_input) {
    double w = 0.0;
    for (int k = 0; k < nsteps; ++k) w += dt[k] * p[(int64_t)k * nt + j];
    double bf = 0.0;
    for (int q = 0; q < m; ++q) bf = fma(bhat[(int64_t)i * m + q], f[q], bf);
    out = w * bf;
  } else {
    for (int k = 0; k < nsteps; ++k) {
      double g = 0.0;
      for (int q = 0; q < m; ++q) g = fma(bhat[(int64_t)i * m + q], f[(int64_t)k * m + q], g);
      out += dt[k] * p[(int64_t)k * nt + j] * g;
    }
  }
  fst[idx] = out;
  x0st[idx] = p[j] * x0hat[i];
}

constexpr int kTile = 64;   // output tile (rows and cols)
constexpr int kKc = 32;     // K chunk staged in shared memory
constexpr int kLd = kTile + 4;

// A_st (NT x NT, row-major) = -(F^T Fd) o tile(A_hat) + diag terms.
__global__ void __launch_bounds__(256) k_st_gemm(const double* __restrict__ F, const double* __restrict__ Fd,
                                                 int kpad, int ns, int nt, const double* __restrict__ ahat,
                                                 const double* __restrict__ D, double* __restrict__ out) {
  __shared__ double As[kKc][kLd];
  __shared__ double Bs[kKc][kLd];
  const int NT = ns * nt;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int r0 = blockIdx.x * kTile, c0 = blockIdx.y * kTile;
  double acc[8][2];
#pragma unroll
  for (int y = 0; y < 8; ++y) acc[y][0] = acc[y][1] = 0.0;
  for (int k0 = 0; k0 < kpad; k0 += kKc) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < kKc * kTile; idx += blockDim.x) {
      const int kk = idx / kTile, cc = idx % kTile;
      const int k = k0 + kk;
      const bool inK = k < kpad;
      As[kk][cc] = (inK && r0 + cc < NT) ? F[(int64_t)k * NT + r0 + cc] : 0.0;
      Bs[kk][cc] = (inK && c0 + cc < NT) ? Fd[(int64_t)k * NT + c0 + cc] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < kKc / 4; ++ks) {
      const double a = As[ks * 4 + t][wid * 8 + g];
#pragma unroll
      for (int y = 0; y < 8; ++y) {
        const double b = Bs[ks * 4 + t][y * 8 + g];
        dmma884(acc[y][0], acc[y][1], a, b);
      }
    }
  }
  const int row = r0 + wid * 8 + g;
  if (row >= NT) return;
  const int jp = row / ns, i = row % ns;
#pragma unroll
  for (int y = 0; y < 8; ++y) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int col = c0 + y * 8 + 2 * t + e;
      if (col >= NT) continue;
      const int j = col / ns, i2 = col % ns;
      double v = -acc[y][e] * ahat[(int64_t)i * ns + i2];
      if (i == i2) v += D[((int64_t)i * nt + jp) * nt + j];
      out[(int64_t)row * NT + col] = v;
    }
  }
}

}  // namespace

extern "C" {

// build_st_matrix / build_st_input / build_st_init (spacetime.py:43-115).
//   ahat: n_s x n_s row-major; psi: (n_s, N_t, n_t) C-order (BasisSet.temporal_stack);
//   dt: N_t; bhat: n_s x m row-major; f: m (constant_input) or N_t x m row-major
//   (row k = input of step k+1); x0hat: n_s.
//   Outputs: a_st (NT x NT row-major), f_st, x0_st (NT), NT = n_s n_t,
//   index j*n_s + i.  Any of f_st/x0_st may be NULL (then bhat/f/x0hat unused).
int strom_st_assemble(const double* ahat_dev, const double* psi_dev, const double* dt_dev, int64_t nsteps,
                      int64_t ns, int64_t nt, const double* bhat_dev, int64_t m, const double* f_dev,
                      int32_t constant_input, const double* x0hat_dev, double* ast_dev, double* fst_dev,
                      double* x0st_dev, void* stream) {
  return guarded([&] {
    STROM_REQUIRE(nsteps >= 1 && ns >= 1 && nt >= 1, "bad space-time shape");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t NT = ns * nt;
    const int kpad = (int)round_up(nsteps, kKc);
    auto ws = dev_alloc(((size_t)2 * kpad * NT + (size_t)ns * nt * nt) * 8, s, false);
    double* F = ws->as<double>();
    double* Fd = F + (size_t)kpad * NT;
    double* D = Fd + (size_t)kpad * NT;
    if (ast_dev) {
      k_st_pack<<<(unsigned)ceil_div((int64_t)kpad * NT, 256), 256, 0, s>>>(psi_dev, dt_dev, (int)nsteps, (int)ns,
                                                                             (int)nt, kpad, F, Fd);
      STROM_LAUNCH_CHECK();
      k_st_diag<<<(unsigned)ceil_div(ns * nt * nt, 128), 128, 0, s>>>(psi_dev, (int)nsteps, (int)ns, (int)nt, D);
      STROM_LAUNCH_CHECK();
      dim3 grid((unsigned)ceil_div(NT, kTile), (unsigned)ceil_div(NT, kTile));
      ProfScope ps(P_ST_GEMM, s);
      k_st_gemm<<<grid, 256, 0, s>>>(F, Fd, kpad, (int)ns, (int)nt, ahat_dev, D, ast_dev);
      STROM_LAUNCH_CHECK();
    }
    if (fst_dev || x0st_dev) {
      STROM_REQUIRE(fst_dev && x0st_dev && bhat_dev && f_dev && x0hat_dev, "f_st/x0_st need b_hat, f, x0_hat");
      k_st_vecs<<<(unsigned)ceil_div(NT, 128), 128, 0, s>>>(psi_dev, dt_dev, (int)nsteps, (int)ns, (int)nt,
                                                           bhat_dev, (int)m, f_dev, constant_input, x0hat_dev,
                                                           fst_dev, x0st_dev);
      STROM_LAUNCH_CHECK();
    }
  });
}

}  // extern "C"
