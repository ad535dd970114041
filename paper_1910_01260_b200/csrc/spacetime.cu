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
// The (n_s n_t)^2 temporal Gram (symmetric: upper-triangle tiles only) runs on
// the fp64 tensor cores (DMMA m8n8k4) with the Hadamard-with-tiled-A_hat and
// the diagonal terms fused into the epilogue.  f_st (spacetime.py:72-99) and x0_st (spacetime.py:102-115) are
// O(n_s n_t N_t) and come from one small kernel.
#include <algorithm>

#include "../../include/strom_b200.h"
#include "bulk.cuh"
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

// Per-mode temporal sums over one chunk of kDiagChunk steps (CTA (i, c)):
//   Dpart[c, i, j', j] = sum_k Psi_i[k,j'] Psi_i[k,j] - sum_{k>0} Psi_i[k,j'] Psi_i[k-1,j]
//   Wpart[c, i, j]     = sum_k dt_k Psi_i[k,j] g_k,   g_k = b_hat_i . f_k (1 for constant input)
// Psi_i's chunk (plus the step before it, for the coupling term) is staged in
// shared memory; thread o < nt^2 owns (j', j).  The chunk partials are summed
// in chunk order by the consumers (k_st_gemm's epilogue, k_st_vec_final).
constexpr int kDiagChunk = 64;
__global__ void __launch_bounds__(256) k_st_temporal(const double* __restrict__ psi, const double* __restrict__ dt,
                                                     int nsteps, int ns, int nt, const double* __restrict__ bhat,
                                                     int m, const double* __restrict__ f, int constant_input,
                                                     double* __restrict__ Dpart, double* __restrict__ Wpart) {
  extern __shared__ double sp[];  // (kDiagChunk + 1) x nt, then kDiagChunk weights dt_k g_k
  const int i = blockIdx.x, c = blockIdx.y;
  const int k0 = c * kDiagChunk, k1 = min(nsteps, k0 + kDiagChunk), nk = k1 - k0;
  const double* p = psi + (int64_t)i * nsteps * nt;
  double* wk = sp + (kDiagChunk + 1) * nt;
  for (int e = threadIdx.x; e < (nk + 1) * nt; e += blockDim.x) {  // row r = step k0 - 1 + r
    const int k = k0 - 1 + e / nt;
    sp[e] = k >= 0 ? p[(int64_t)k * nt + e % nt] : 0.0;
  }
  for (int r = threadIdx.x; r < nk; r += blockDim.x) {
    const int k = k0 + r;
    double g = 1.0;
    if (!constant_input) {
      g = 0.0;
      for (int q = 0; q < m; ++q) g = fma(bhat[(int64_t)i * m + q], f[(int64_t)k * m + q], g);
    }
    wk[r] = dt[k] * g;
  }
  __syncthreads();
  const int no = nt * nt;
  double* Dp = Dpart + ((int64_t)c * ns + i) * no;
  for (int o = threadIdx.x; o < no; o += blockDim.x) {
    const int jp = o / nt, j = o % nt;
    double s0 = 0.0, s1 = 0.0, c0 = 0.0, c1 = 0.0;
    int r = 1;
    for (; r + 1 <= nk; r += 2) {  // two independent chains per sum
      const double a0 = sp[r * nt + jp], a1 = sp[(r + 1) * nt + jp];
      s0 = fma(a0, sp[r * nt + j], s0);
      c0 = fma(a0, sp[(r - 1) * nt + j], c0);
      s1 = fma(a1, sp[(r + 1) * nt + j], s1);
      c1 = fma(a1, sp[r * nt + j], c1);
    }
    if (r <= nk) {
      const double a0 = sp[r * nt + jp];
      s0 = fma(a0, sp[r * nt + j], s0);
      c0 = fma(a0, sp[(r - 1) * nt + j], c0);
    }
    Dp[o] = (s0 + s1) - (c0 + c1);  // coupling row 0 is zero for the first chunk (no step before k = 0)
  }
  for (int j = threadIdx.x; j < nt; j += blockDim.x) {
    double w = 0.0;
    for (int r = 0; r < nk; ++r) w = fma(wk[r], sp[(r + 1) * nt + j], w);
    Wpart[((int64_t)c * ns + i) * nt + j] = w;
  }
}

// Chunk sums in chunk order: D[i, j', j] = sum_c Dpart[c, i, j', j];
// f_st[j n_s + i] = (b_hat_i . f) sum_c Wpart (constant input) or sum_c Wpart;
// x0_st[j n_s + i] = Psi_i[0, j] x0_hat_i  (the reference code's choice, spacetime.py:102-115).
__global__ void k_st_final(const double* __restrict__ psi, int nsteps, int ns, int nt, int nchunks,
                           const double* __restrict__ Dpart, double* __restrict__ D, const double* __restrict__ bhat,
                           int m, const double* __restrict__ f, int constant_input, const double* __restrict__ x0hat,
                           const double* __restrict__ Wpart, double* __restrict__ fst, double* __restrict__ x0st) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nd = (int64_t)ns * nt * nt;
  if (D && idx < nd) {
    double d = 0.0;
    for (int c = 0; c < nchunks; ++c) d += Dpart[c * nd + idx];
    D[idx] = d;
  }
  if (!fst || idx >= ns * nt) return;
  const int j = idx / ns, i = idx % ns;
  double w = 0.0;
  for (int c = 0; c < nchunks; ++c) w += Wpart[((int64_t)c * ns + i) * nt + j];
  if (constant_input) {
    double bf = 0.0;
    for (int q = 0; q < m; ++q) bf = fma(bhat[(int64_t)i * m + q], f[q], bf);
    w *= bf;
  }
  fst[idx] = w;
  x0st[idx] = psi[(int64_t)i * nsteps * nt + j] * x0hat[i];
}

constexpr int kTile = 64;   // output tile (rows and cols)
constexpr int kKc = 32;     // K chunk staged in shared memory
constexpr int kLd = kTile + 4;

// A_st (NT x NT, row-major) = -(F^T Fd) o tile(A_hat) + diag terms.  The
// temporal Gram G = F^T diag(dt) F is symmetric, so only the upper-triangle
// 64 x 64 tiles are computed (one wave for NT = 1000) and each writes both
// A_st blocks it determines, each with its own Hadamard factor and diagonal
// term.  K chunks are prefetched into registers while the previous chunk is
// contracted.
__device__ __forceinline__ double st_entry(double gval, int row, int col, int ns, int nt, const double* ahat,
                                           const double* D) {
  const int jp = row / ns, i = row % ns, j = col / ns, i2 = col % ns;
  double v = -gval * ahat[(int64_t)i * ns + i2];
  if (i == i2) v += D[((int64_t)i * nt + jp) * nt + j];
  return v;
}

__global__ void __launch_bounds__(256) k_st_gemm(const double* __restrict__ F, const double* __restrict__ Fd,
                                                 int kpad, int ns, int nt, const double* __restrict__ ahat,
                                                 const double* __restrict__ D, double* __restrict__ out) {
  __shared__ double As[kKc][kLd];
  __shared__ double Bs[kKc][kLd];
  const int NT = ns * nt;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  // upper-triangle tile (bx <= by) from the linear block index
  const int nb = (int)ceil_div(NT, kTile);
  int bx = 0, rem = blockIdx.x;
  while (rem >= nb - bx) { rem -= nb - bx; ++bx; }
  const int by = bx + rem;
  const int r0 = bx * kTile, c0 = by * kTile;
  constexpr int kPer = kKc * kTile / 256;  // elements per thread per operand per chunk
  double pa[kPer], pb[kPer];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int idx = threadIdx.x + q * 256;
      const int kk = idx / kTile, cc = idx % kTile, k = k0 + kk;
      const bool inK = k < kpad;
      pa[q] = (inK && r0 + cc < NT) ? F[(int64_t)k * NT + r0 + cc] : 0.0;
      pb[q] = (inK && c0 + cc < NT) ? Fd[(int64_t)k * NT + c0 + cc] : 0.0;
    }
  };
  double acc[8][2];
#pragma unroll
  for (int y = 0; y < 8; ++y) acc[y][0] = acc[y][1] = 0.0;
  fetch(0);
  for (int k0 = 0; k0 < kpad; k0 += kKc) {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int idx = threadIdx.x + q * 256;
      As[idx / kTile][idx % kTile] = pa[q];
      Bs[idx / kTile][idx % kTile] = pb[q];
    }
    __syncthreads();
    if (k0 + kKc < kpad) fetch(k0 + kKc);
#pragma unroll
    for (int ks = 0; ks < kKc / 4; ++ks) {
      const double a = As[ks * 4 + t][wid * 8 + g];
#pragma unroll
      for (int y = 0; y < 8; ++y) dmma884(acc[y][0], acc[y][1], a, Bs[ks * 4 + t][y * 8 + g]);
    }
  }
  const int row = r0 + wid * 8 + g;
  if (row >= NT) return;
#pragma unroll
  for (int y = 0; y < 8; ++y) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int col = c0 + y * 8 + 2 * t + e;
      if (col >= NT) continue;
      out[(int64_t)row * NT + col] = st_entry(acc[y][e], row, col, ns, nt, ahat, D);
      if (bx != by) out[(int64_t)col * NT + row] = st_entry(acc[y][e], col, row, ns, nt, ahat, D);
    }
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// reconstruct_states (spacetime.py:180-186): X = Phi_s C with
// C[i, k] = sum_j Psi_i[k, j] xhat[j n_s + i]  (n_s x N_t), the space-time
// basis never formed.  At cfg4 (N = 10^6, n_s = 50, N_t = 500) the tall GEMM
// is 50 GFlop against a 4 GB output: fp64 tensor-core bound, so it runs on
// DMMA m8n8k4 -- 128-row x 64-column CTA tiles, 32 x 32 warp tiles, K = n_s
// (padded to 4) in one shared-memory stage, the Phi tile kept while the CTA
// walks its row block's column tiles; output written straight from the
// accumulators (row-major, 16-byte pairs).
// ---------------------------------------------------------------------------
__global__ void k_rc_coeffs(const double* __restrict__ psi, const double* __restrict__ xhat, int ns, int nsteps,
                            int nt, double* __restrict__ C) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)ns * nsteps) return;
  const int i = (int)(idx / nsteps), k = (int)(idx % nsteps);
  const double* ps = psi + ((int64_t)i * nsteps + k) * nt;
  double acc = 0.0;
  for (int j = 0; j < nt; ++j) acc = fma(ps[j], xhat[(int64_t)j * ns + i], acc);
  C[(int64_t)i * nsteps + k] = acc;
}

constexpr int kRcRows = 128, kRcCols = 64, kRcThreads = 256;

// One CTA: a 128-row block of Phi (K4 x 128, one cp.async stage) against every
// 64-column tile of C in turn (double-buffered cp.async stages, the next tile's
// copy in flight while the current one is multiplied).
__global__ void __launch_bounds__(kRcThreads, 2) k_reconstruct(int64_t N, int ns, int nsteps,
                                                               const double* __restrict__ phi, int64_t ldphi,
                                                               const double* __restrict__ C,
                                                               double* __restrict__ out, int64_t ldo) {
  extern __shared__ __align__(16) double rsm[];
  const int K4 = (ns + 3) & ~3;
  constexpr int LA = kRcRows + 4, LB = kRcCols + 4;  // = 4 (mod 16): conflict-free fragment loads
  double* As = rsm;                              // As[k * LA + r] = Phi[r0 + r, k]
  double* Bs0 = As + (size_t)K4 * LA;             // Bs[k * LB + c] = C[k, c0 + c], two buffers
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, g = lane >> 2, t = lane & 3;
  const int wm = wid & 3, wn = wid >> 2;  // warp tile: rows 32 wm.., columns 32 wn..
  const bool pairs = (ldo % 2) == 0;
  const int ntiles = (nsteps + kRcCols - 1) / kRcCols;
  auto load_b = [&](double* Bs, int c0) {
    for (int idx = tid; idx < K4 * kRcCols; idx += kRcThreads) {
      const int k = idx / kRcCols, c = idx % kRcCols;
      const bool ok = k < ns && c0 + c < nsteps;
      cp_async8(Bs + k * LB + c, ok ? C + (int64_t)k * nsteps + c0 + c : C, ok);
    }
  };
  for (int64_t rb = blockIdx.x; rb * kRcRows < N; rb += gridDim.x) {
    const int64_t r0 = rb * kRcRows;
    __syncthreads();  // the previous row block's last tile is consumed
    for (int idx = tid; idx < K4 * kRcRows; idx += kRcThreads) {
      const int k = idx / kRcRows, r = idx % kRcRows;
      const bool ok = k < ns && r0 + r < N;
      cp_async8(As + k * LA + r, ok ? phi + (int64_t)k * ldphi + r0 + r : phi, ok);
    }
    load_b(Bs0, 0);
    cp_async_commit();
    for (int ct = 0; ct < ntiles; ++ct) {
      const int c0 = ct * kRcCols;
      double* Bs = Bs0 + (size_t)(ct & 1) * K4 * LB;
      if (ct + 1 < ntiles) load_b(Bs0 + (size_t)((ct + 1) & 1) * K4 * LB, c0 + kRcCols);
      cp_async_commit();
      cp_async_wait<1>();  // everything but the copy just issued
      __syncthreads();
      double acc[4][4][2];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
      for (int ks = 0; ks < K4; ks += 4) {
        double fa[4], fb[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) fa[a] = As[(ks + t) * LA + 32 * wm + 8 * a + g];
#pragma unroll
        for (int b = 0; b < 4; ++b) fb[b] = Bs[(ks + t) * LB + 32 * wn + 8 * b + g];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) dmma884(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
      }
      __syncthreads();  // this buffer may be refilled by the next iteration's copy
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int64_t row = r0 + 32 * wm + 8 * a + g;
        if (row >= N) continue;
        double* orow = out + row * ldo;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int col = c0 + 32 * wn + 8 * b + 2 * t;
          if (pairs && col + 1 < nsteps) {
            __stcs(reinterpret_cast<double2*>(orow + col), make_double2(acc[a][b][0], acc[a][b][1]));
          } else {
            if (col < nsteps) orow[col] = acc[a][b][0];
            if (col + 1 < nsteps) orow[col + 1] = acc[a][b][1];
          }
        }
      }
    }
  }
}

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
    const int nch = (int)ceil_div(nsteps, kDiagChunk);
    const bool vecs = fst_dev || x0st_dev;
    if (vecs) STROM_REQUIRE(fst_dev && x0st_dev && bhat_dev && f_dev && x0hat_dev, "f_st/x0_st need b_hat, f, x0_hat");
    auto ws = dev_alloc(((size_t)2 * kpad * NT + (size_t)(nch + 1) * ns * nt * nt + (size_t)nch * ns * nt) * 8, s,
                        false);
    double* F = ws->as<double>();
    double* Fd = F + (size_t)kpad * NT;
    double* D = Fd + (size_t)kpad * NT;
    double* Dp = D + (size_t)ns * nt * nt;
    double* Wp = Dp + (size_t)nch * ns * nt * nt;
    k_st_temporal<<<dim3((unsigned)ns, (unsigned)nch), 256, (size_t)((kDiagChunk + 1) * nt + kDiagChunk) * 8, s>>>(
        psi_dev, dt_dev, (int)nsteps, (int)ns, (int)nt, vecs ? bhat_dev : nullptr, (int)m, vecs ? f_dev : nullptr,
        vecs ? constant_input : 1, Dp, Wp);
    STROM_LAUNCH_CHECK();
    const int64_t nfin = std::max<int64_t>(ast_dev ? ns * nt * nt : 0, vecs ? NT : 0);
    k_st_final<<<(unsigned)ceil_div(nfin, 256), 256, 0, s>>>(psi_dev, (int)nsteps, (int)ns, (int)nt, nch,
                                                           Dp, ast_dev ? D : nullptr, bhat_dev, (int)m, f_dev,
                                                           constant_input, x0hat_dev, Wp, vecs ? fst_dev : nullptr,
                                                           x0st_dev);
    STROM_LAUNCH_CHECK();
    if (ast_dev) {
      k_st_pack<<<(unsigned)ceil_div((int64_t)kpad * NT, 256), 256, 0, s>>>(psi_dev, dt_dev, (int)nsteps, (int)ns,
                                                                             (int)nt, kpad, F, Fd);
      STROM_LAUNCH_CHECK();
      const int64_t nb = ceil_div(NT, kTile);
      ProfScope ps(P_ST_GEMM, s);
      k_st_gemm<<<(unsigned)(nb * (nb + 1) / 2), 256, 0, s>>>(F, Fd, kpad, (int)ns, (int)nt, ahat_dev, D, ast_dev);
      STROM_LAUNCH_CHECK();
    }
  });
}

// reconstruct_states: out (N x N_t, row-major, ldo) = Phi_s C,
// C[i, k] = sum_j psi[i, k, j] xhat[j n_s + i]; phi column-major (ldphi).
int strom_st_reconstruct(int64_t N, int64_t ns, int64_t nt, int64_t nsteps, const double* phi_dev, int64_t ldphi,
                         const double* psi_dev, const double* xhat_dev, double* out_dev, int64_t ldo, void* stream) {
  return guarded([&] {
    STROM_REQUIRE(N >= 1 && ns >= 1 && nt >= 1 && nsteps >= 1 && phi_dev && psi_dev && xhat_dev && out_dev,
                  "bad reconstruct arguments");
    STROM_REQUIRE(ldphi >= N && ldo >= nsteps, "bad leading dimensions");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    auto cbuf = dev_alloc((size_t)ns * nsteps * 8, s, false);
    double* C = cbuf->as<double>();
    ProfScope ps(P_ST_SMALL, s);
    k_rc_coeffs<<<(unsigned)ceil_div(ns * nsteps, 256), 256, 0, s>>>(psi_dev, xhat_dev, (int)ns, (int)nsteps, (int)nt,
                                                                     C);
    STROM_LAUNCH_CHECK();
    const int K4 = (int)((ns + 3) & ~3);
    const size_t smem = (size_t)K4 * ((kRcRows + 4) + 2 * (kRcCols + 4)) * 8;
    STROM_REQUIRE(smem <= max_smem_optin(), "reconstruct: n_s too large for one shared-memory K stage");
    static PerDevice<size_t> cfg;
    if (cfg.get() < smem) {
      STROM_CUDA(cudaFuncSetAttribute(k_reconstruct, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      cfg.get() = smem;
    }
    int occ = 0;
    STROM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_reconstruct, kRcThreads, smem));
    const int64_t nrb = ceil_div(N, (int64_t)kRcRows);
    const int grid = (int)std::min<int64_t>(nrb, (int64_t)sm_count() * std::max(occ, 1));
    k_reconstruct<<<grid, kRcThreads, smem, s>>>(N, (int)ns, (int)nsteps, phi_dev, ldphi, C, out_dev, ldo);
    STROM_LAUNCH_CHECK();
  });
}

}  // extern "C"
