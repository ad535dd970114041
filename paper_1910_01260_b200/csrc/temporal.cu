// Batched small SVDs: the per-mode temporal bases (reference basis.py:275-302)
// and the device thin_svd (linalg.py:41-57).
//
// One CTA per matrix.  QR-preconditioned one-sided Jacobi: A = Q R by
// Householder, Jacobi on R^T (tall) or R (wide) with the rotations
// accumulated, so the LEFT singular vectors -- the ones the temporal basis and
// the sign rule use -- are products of orthogonal factors.
#include <algorithm>

#include "../../include/strom_b200.h"
#include "runtime.cuh"
#include "small_dense.cuh"

using namespace strom;

namespace {

struct SvdBatchArgs {
  const double* a;   // matrix b starts at a + b * a_bstride; column-major, lda
  int64_t a_bstride, lda;
  int rows, cols;
  // outputs (any may be null)
  double* w;         // left vectors, w[b * w_bstride + i * w_rs + j * w_cs]
  int64_t w_bstride, w_rs, w_cs;
  int w_ncols;       // how many left vectors to write
  double* s;         // sigma, s[b * kmin + j]
  double* v;         // right vectors, column-major cols x kmin per batch
  int32_t* rank;     // rank[b] with threshold max(rows, cols) * eps * sigma_0
  double* work;      // per-CTA global fallback workspace
  int64_t work_per;
  int use_smem;
};

__host__ __device__ inline int64_t svd_work_elems(int rows, int cols) {
  const int tall = rows >= cols;
  const int64_t big = tall ? rows : cols, small = tall ? cols : rows;
  // M (big x small) + B, W (small^2 each) + norms/tau/beta (3 small) + perm
  return big * small + 2 * small * small + 4 * small + 8;
}

__global__ void __launch_bounds__(512) k_small_svd(SvdBatchArgs A) {
  extern __shared__ double smem[];
  __shared__ double red[32];
  __shared__ int flag;
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int rows = A.rows, cols = A.cols;
  const bool tall = rows >= cols;
  const int big = tall ? rows : cols, sm = tall ? cols : rows;
  double* base = A.use_smem ? smem : A.work + (int64_t)b * A.work_per;
  double* M = base;                       // big x sm (ld = big): A (tall) or A^T (wide)
  double* B = M + (int64_t)big * sm;      // sm x sm
  double* W = B + (int64_t)sm * sm;       // sm x sm accumulated rotations
  double* nrm = W + (int64_t)sm * sm;     // sm
  double* tau = nrm + sm;
  double* beta = tau + sm;
  int* perm = reinterpret_cast<int*>(beta + sm);
  const double* a = A.a + (int64_t)b * A.a_bstride;
  for (int64_t idx = threadIdx.x; idx < (int64_t)rows * cols; idx += blockDim.x) {
    const int i = idx % rows, j = idx / rows;
    const double val = a[(int64_t)j * A.lda + i];
    if (tall) M[(int64_t)j * big + i] = val;
    else M[(int64_t)i * big + j] = val;
  }
  __syncthreads();
  cta_householder_qr(M, big, big, sm, B, sm, tau, beta, red);  // M <- Q, B <- R
  // tall: Jacobi on R^T (B transposed in place); wide: on R
  if (tall) {
    for (int64_t idx = threadIdx.x; idx < (int64_t)sm * sm; idx += blockDim.x) {
      const int i = idx % sm, j = idx / sm;
      if (i < j) {
        const double t = B[(int64_t)j * sm + i];
        B[(int64_t)j * sm + i] = B[(int64_t)i * sm + j];
        B[(int64_t)i * sm + j] = t;
      }
    }
  }
  for (int64_t idx = threadIdx.x; idx < (int64_t)sm * sm; idx += blockDim.x)
    W[idx] = (idx % sm == idx / sm) ? 1.0 : 0.0;
  __syncthreads();
  cta_jacobi(B, sm, sm, sm, W, sm, sm, &flag);
  cta_col_norms(B, sm, sm, sm, nrm);
  cta_argsort_desc(nrm, sm, perm);
  const double s0 = nrm[perm[0]];
  const double thr = (double)max(rows, cols) * 2.220446049250313e-16 * s0;
  if (threadIdx.x == 0 && A.rank) {
    int rk = 0;
    for (int j = 0; j < sm; ++j) rk += nrm[j] > thr;
    A.rank[b] = rk;
  }
  if (A.s)
    for (int j = threadIdx.x; j < sm; j += blockDim.x) A.s[(int64_t)b * sm + j] = nrm[perm[j]];
  // left vectors: tall -> Q W (big x sm); wide -> W (sm x sm, rows == sm)
  // right vectors: tall -> B col / sigma (sm == cols); wide -> Q (B col / sigma)
  const int nout = A.w_ncols;
  for (int k = wid; k < sm; k += nw) {
    const int jj = perm[k];
    // sign rule on the left vector (linalg.py:31-38): argmax |w|, first index on ties
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int i = lane; i < rows; i += 32) {
      double wv;
      if (tall) {
        wv = 0.0;
        for (int q = 0; q < sm; ++q) wv = fma(M[(int64_t)q * big + i], W[(int64_t)jj * sm + q], wv);
      } else {
        wv = W[(int64_t)jj * sm + i];
      }
      if (fabs(wv) > best) { best = fabs(wv); bi = i; }
    }
    double bv = 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    // value at bi (recompute by the owning lane)
    if ((bi & 31) == lane) {
      if (tall) {
        bv = 0.0;
        for (int q = 0; q < sm; ++q) bv = fma(M[(int64_t)q * big + bi], W[(int64_t)jj * sm + q], bv);
      } else {
        bv = W[(int64_t)jj * sm + bi];
      }
    }
    bv = __shfl_sync(0xffffffffu, bv, bi & 31);
    const double sg = (bv < 0.0) ? -1.0 : 1.0;
    if (A.w && k < nout) {
      double* wo = A.w + (int64_t)b * A.w_bstride + (int64_t)k * A.w_cs;
      for (int i = lane; i < rows; i += 32) {
        double wv;
        if (tall) {
          wv = 0.0;
          for (int q = 0; q < sm; ++q) wv = fma(M[(int64_t)q * big + i], W[(int64_t)jj * sm + q], wv);
        } else {
          wv = W[(int64_t)jj * sm + i];
        }
        wo[(int64_t)i * A.w_rs] = sg * wv;
      }
    }
    if (A.v) {
      const double sj = nrm[jj];
      double* vo = A.v + (int64_t)b * cols * sm + (int64_t)k * cols;
      for (int i = lane; i < cols; i += 32) {
        double vv;
        if (tall) {
          vv = (sj > 0.0) ? B[(int64_t)jj * sm + i] / sj : (i == jj ? 1.0 : 0.0);
        } else {
          vv = 0.0;
          for (int q = 0; q < sm; ++q) vv = fma(M[(int64_t)q * big + i], B[(int64_t)jj * sm + q], vv);
          vv = (sj > 0.0) ? vv / sj : 0.0;
        }
        vo[i] = sg * vv;
      }
    }
  }
}

void launch_small_svd(SvdBatchArgs args, int batch, cudaStream_t s, DevMemPtr* keep) {
  const int64_t elems = svd_work_elems(args.rows, args.cols);
  const size_t bytes = (size_t)elems * 8;
  const size_t limit = max_smem_optin() - 4 * 1024;
  args.use_smem = bytes <= limit;
  if (!args.use_smem) {
    *keep = dev_alloc((size_t)elems * batch * 8, s, false);
    args.work = (*keep)->as<double>();
    args.work_per = elems;
  }
  const size_t smem = args.use_smem ? bytes : 0;
  static PerDevice<size_t> configured_dev;
  size_t& configured = configured_dev.get();
  if (smem > 48 * 1024 && smem > configured) {
    STROM_CUDA(cudaFuncSetAttribute(k_small_svd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = smem;
  }
  k_small_svd<<<batch, 512, smem, s>>>(args);
  STROM_LAUNCH_CHECK();
}

}  // namespace

extern "C" {

// build_basis_set's temporal loop (basis.py:292-301), batched over modes.
// v_dev: k x r column-major (ld ldv), k = n_mu * n_steps.  Outputs: psi
// (n_s, n_steps, n_t) C-order, ranks (n_s), sigma (n_s, min(n_steps, n_mu)).
int strom_temporal_bases(const double* v_dev, int64_t ldv, int64_t r, int64_t n_steps, int64_t n_mu,
                         int64_t n_s, int64_t n_t, double* psi_dev, int32_t* ranks_dev, double* sigma_dev,
                         void* stream) {
  return guarded([&] {
    STROM_REQUIRE(v_dev && n_steps >= 1 && n_mu >= 1 && n_s >= 1 && n_s <= r, "bad temporal-basis shape");
    STROM_REQUIRE(n_t >= 1 && n_t <= std::min(n_steps, n_mu), "n_t above the temporal ceiling");
    STROM_REQUIRE(ldv >= n_steps * n_mu, "ldv too small");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    SvdBatchArgs a{};
    a.a = v_dev;
    a.a_bstride = ldv;  // mode b = column b of v
    a.lda = n_steps;    // T_b[i, p] = v[p * n_steps + i, b]
    a.rows = (int)n_steps;
    a.cols = (int)n_mu;
    a.w = psi_dev;
    a.w_bstride = n_steps * n_t;
    a.w_rs = n_t;
    a.w_cs = 1;
    a.w_ncols = (int)n_t;
    a.s = sigma_dev;
    a.rank = ranks_dev;
    DevMemPtr keep;
    launch_small_svd(a, (int)n_s, s, &keep);
  });
}

// linalg.thin_svd (linalg.py:41-57) on the device: m (rows x cols,
// column-major, ld) -> w (rows x kmin col-major), sigma, v (cols x kmin).
int strom_thin_svd(int64_t rows, int64_t cols, const double* m_dev, double* w_dev, double* s_dev,
                   double* v_dev, void* stream) {
  return guarded([&] {
    STROM_REQUIRE(rows >= 1 && cols >= 1 && m_dev, "need a non-empty 2-D matrix");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t kmin = std::min(rows, cols);
    SvdBatchArgs a{};
    a.a = m_dev;
    a.a_bstride = 0;
    a.lda = rows;
    a.rows = (int)rows;
    a.cols = (int)cols;
    a.w = w_dev;
    a.w_bstride = 0;
    a.w_rs = 1;
    a.w_cs = rows;
    a.w_ncols = (int)kmin;
    a.s = s_dev;
    a.v = v_dev;
    DevMemPtr keep;
    launch_small_svd(a, 1, s, &keep);
  });
}

}  // extern "C"
