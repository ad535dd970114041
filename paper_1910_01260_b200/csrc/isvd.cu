// Host orchestration + C ABI of the streaming incremental SVD
// (reference basis.py:30-194).  See isvd_kernels.cuh for the representation.
#include <algorithm>
#include <cstring>
#include <memory>
#include <vector>

#include "../../include/strom_b200.h"
#include "gram.cuh"
#include "isvd_kernels.cuh"
#include "runtime.cuh"

using namespace strom;

namespace {

// ------------------------------------------------------------------ helpers
__global__ void k_rm_to_cm(const double* __restrict__ src, int64_t rows, int64_t cols, double* __restrict__ dst,
                           int64_t ldd) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * cols) return;
  const int64_t i = idx / cols, j = idx % cols;
  dst[j * ldd + i] = src[idx];
}

__global__ void k_cm_to_rm(const double* __restrict__ src, int64_t lds, int64_t rows, int64_t cols,
                           double* __restrict__ dst) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * cols) return;
  const int64_t i = idx / cols, j = idx % cols;
  dst[idx] = src[j * lds + i];
}

__global__ void k_copy_cm(const double* __restrict__ src, int64_t lds, int64_t rows, int64_t cols,
                          double* __restrict__ dst, int64_t ldd) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * cols) return;
  const int64_t i = idx % rows, j = idx / rows;
  dst[j * ldd + i] = src[j * lds + i];
}

__global__ void k_set_hdr(IsvdHdr* h, int32_t r, int32_t c, int32_t base, int32_t rej, int32_t dep, int32_t tr,
                          int32_t rs) {
  IsvdHdr o;
  memset(&o, 0, sizeof(o));
  o.r = r;
  o.c = c;
  o.base = base;
  o.n_rejected = rej;
  o.n_dependent = dep;
  o.n_truncated = tr;
  o.n_restarts = rs;
  *h = o;
}

__global__ void __launch_bounds__(1024) k_lower_inverse(const double* L, int ld, const IsvdHdr* h_c_from,
                                                       int c_fixed, double* Li) {
  const int c = h_c_from ? h_c_from->c : c_fixed;
  cta_lower_inverse(L, ld, c, Li, ld);
}

// In-place lower Cholesky of A (c x c, ld); sets *status = 1 on a non-positive pivot.
__global__ void k_cholesky(double* A, int ld, const IsvdHdr* h_c_from, int c_fixed, int* status) {
  const int c = h_c_from ? h_c_from->c : c_fixed;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < c; ++j) {
    if (threadIdx.x == 0) {
      const double d = A[(int64_t)j * ld + j];
      if (!(d > 0.0)) bad = 1;
      A[(int64_t)j * ld + j] = sqrt(fmax(d, 0.0));
    }
    __syncthreads();
    if (bad) break;
    const double piv = A[(int64_t)j * ld + j];
    for (int i = j + 1 + threadIdx.x; i < c; i += blockDim.x) A[(int64_t)j * ld + i] /= piv;
    __syncthreads();
    const int rem = c - j - 1;
    for (int64_t idx = threadIdx.x; idx < (int64_t)rem * rem; idx += blockDim.x) {
      const int i = j + 1 + idx % rem, k = j + 1 + idx / rem;
      if (k <= i) A[(int64_t)k * ld + i] -= A[(int64_t)j * ld + i] * A[(int64_t)j * ld + k];
    }
    __syncthreads();
  }
  // zero the strict upper triangle
  for (int64_t idx = threadIdx.x; idx < (int64_t)c * c; idx += blockDim.x) {
    const int i = idx % c, k = idx / c;
    if (k > i) A[(int64_t)k * ld + i] = 0.0;
  }
  if (threadIdx.x == 0 && bad) *status = 1;
}

__global__ void k_copy_g_col(const double* g, int c, double* G, int ld, int j) {
  for (int i = threadIdx.x; i < c; i += blockDim.x) G[(int64_t)j * ld + i] = g[i];
}

inline int maxj_for(int ccap) {
  const int need = (ccap + 7) / 8;
  if (need <= 2) return 2;
  if (need <= 4) return 4;
  if (need <= 8) return 8;
  if (need <= 16) return 16;
  return 32;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

long long* g_tprobe = nullptr;  // step-B phase timestamps (strom_debug_tprobe)

// ------------------------------------------------------------------ state
struct UBuf {
  DevMemPtr mem;
  int64_t ldu = 0;
  int32_t ccap = 0;
  int32_t claimed = 0;  // host bound: no live state uses a physical column >= claimed
  double* ptr() const { return mem->as<double>(); }
};

struct Caps {
  int32_t rcap = 0, ccap = 0;
  int64_t kcap = 0;
};

}  // namespace

struct strom_isvd {
  int64_t n = 0, ldu = 0, k = 0;
  double tol_svd = 0.0, tol_sv = 0.0;
  int32_t r_max = -1, cap_mode = 0;
  Caps caps;
  int32_t c_ub = 0;  // bound on base + c (physical end of used columns)
  int32_t r_ub = 0;  // bound on rank
  std::shared_ptr<UBuf> U;
  DevMemPtr small, vmem;
  StateView view{};
};

namespace {

// ccap = rcap + 1 + slack; 2 rcap keeps c_cap = 128 (8 columns per warp) at rank 64
int32_t slack_for(int32_t rcap) { return std::max<int32_t>(16, rcap - 1); }

Caps make_caps(int64_t n, int32_t r_max, int32_t want_r, int64_t k) {
  Caps c;
  int64_t rc;
  if (r_max >= 0) rc = std::min<int64_t>(std::max<int32_t>(r_max, 1), n);
  else rc = std::min<int64_t>(std::max<int32_t>(want_r, 32), n);
  rc = std::max<int64_t>(rc, 1);
  if (rc > 254) throw Error(kInvalidArgument, "rank capacity above 254 is not supported by this build");
  c.rcap = (int32_t)rc;
  c.ccap = std::min<int32_t>(256, c.rcap + 1 + slack_for(c.rcap));
  c.kcap = std::max<int64_t>(64, round_up(std::max<int64_t>(k, 1) * 2, 64));
  return c;
}

void alloc_small(strom_isvd* h, cudaStream_t s) {
  const Caps& c = h->caps;
  const size_t wsz = (size_t)c.ccap * (c.rcap + 1);
  const size_t lsz = (size_t)c.ccap * c.ccap;
  const size_t ssz = (size_t)c.rcap + 2;
  const size_t bytes = 256 + 8 * (wsz + 2 * lsz + ssz);
  h->small = dev_alloc(bytes, s, true);
  char* p = h->small->as<char>();
  h->view.hdr = reinterpret_cast<IsvdHdr*>(p);
  h->view.N = reinterpret_cast<double*>(p + 256);
  h->view.L = h->view.N + wsz;
  h->view.Li = h->view.L + lsz;
  h->view.sigma = h->view.Li + lsz;
  h->view.ldn = c.ccap;
  h->view.ldl = c.ccap;
}

void alloc_v(strom_isvd* h, cudaStream_t s) {
  h->vmem = dev_alloc((size_t)h->caps.kcap * (h->caps.rcap + 1) * 8, s, false);
  h->view.V = h->vmem->as<double>();
  h->view.ldv = h->caps.kcap;
}

std::shared_ptr<UBuf> alloc_u(int64_t ldu, int32_t ccap, cudaStream_t s) {
  auto u = std::make_shared<UBuf>();
  u->mem = dev_alloc((size_t)ldu * ccap * 8, s, true);
  u->ldu = ldu;
  u->ccap = ccap;
  return u;
}

strom_isvd* new_like(const strom_isvd* src, const Caps& caps) {
  auto* h = new strom_isvd();
  h->n = src->n;
  h->ldu = src->ldu;
  h->k = src->k;
  h->tol_svd = src->tol_svd;
  h->tol_sv = src->tol_sv;
  h->r_max = src->r_max;
  h->cap_mode = src->cap_mode;
  h->caps = caps;
  return h;
}

// per-call scratch
struct ScratchMem {
  DevMemPtr mem;
  Scratch sc{};
  int grid = 0;
  int pstride = 0, work_stride = 0;
  size_t work_elems = 0;
};

int pass_grid(int64_t ldu) {
  const int64_t ntiles = ldu / kTileRows;
  return (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)sm_count() * 4));
}

ScratchMem make_scratch(int64_t ldu, const Caps& c, cudaStream_t s) {
  ScratchMem m;
  m.grid = pass_grid(ldu);
  m.pstride = (int)round_up(c.ccap + 2, 8);
  const int64_t rc2 = c.rcap + 2;
  m.work_stride = (int)round_up(std::max<int64_t>(c.ccap, rc2), 32);
  m.work_elems = 4 * (size_t)m.work_stride + 3 * rc2 * rc2 + 16 * (size_t)m.work_stride +
                 (size_t)c.ccap * rc2;  // step B's layout (global fallback)
  const size_t n_g = round_up(c.ccap, 2), n_ell = round_up(rc2, 2), n_vbar = rc2 * rc2, n_T = (size_t)c.ccap * rc2;
  const size_t n_part = (size_t)m.grid * m.pstride;
  size_t total = 8 * n_g + n_ell + n_vbar + m.work_elems + n_T + n_part;
  total = round_up(total, 32);
  const size_t bytes = total * 8 + 256 + 64;
  m.mem = dev_alloc(bytes, s, true);
  double* p = m.mem->as<double>();
  m.sc.g = p; p += n_g;
  m.sc.gt = p; p += n_g;
  m.sc.y = p; p += n_g;
  m.sc.e = p; p += n_g;
  m.sc.h = p; p += n_g;
  m.sc.lvec = p; p += n_g;
  m.sc.tmp = p; p += n_g;
  m.sc.l1 = p; p += n_g;
  m.sc.ell = p; p += n_ell;
  m.sc.vbar = p; p += n_vbar;
  m.sc.work = p; p += m.work_elems;
  m.sc.T = p; p += n_T;
  m.sc.part = p; p += n_part;
  char* q = m.mem->as<char>() + total * 8;
  m.sc.step = reinterpret_cast<IsvdStep*>(q);
  m.sc.counter = reinterpret_cast<unsigned*>(q + 256);
  return m;
}

IsvdParams make_params(const strom_isvd* h, const ScratchMem& m, int64_t k_new, bool init_call) {
  IsvdParams P;
  P.n = h->n;
  P.ldu = h->ldu;
  P.ccap = h->caps.ccap;
  P.rcap = h->caps.rcap;
  P.tol_svd = h->tol_svd;
  P.tol_sv = h->tol_sv;
  P.r_max = init_call ? -1 : h->r_max;
  P.cap_mode = h->cap_mode;
  P.k_new = k_new;
  P.pstride = m.pstride;
  P.work_stride = m.work_stride;
  P.prof = prof_dev_bytes();
  P.tprobe = g_tprobe;
  return P;
}

template <int MAXJ>
void launch_proj_t(const double* U, const double* x, const StateView& v, const ScratchMem& m, const IsvdParams& P,
                   cudaStream_t s) {
  ProfScope ps(P_PROJ, s);
  k_proj<MAXJ><<<m.grid, kPassThreads, 0, s>>>(U, x, v, m.sc, P);
  STROM_LAUNCH_CHECK();
}

void launch_proj(int ccap, const double* U, const double* x, const StateView& v, const ScratchMem& m,
                 const IsvdParams& P, cudaStream_t s) {
  switch (maxj_for(ccap)) {
    case 2: launch_proj_t<2>(U, x, v, m, P, s); break;
    case 4: launch_proj_t<4>(U, x, v, m, P, s); break;
    case 8: launch_proj_t<8>(U, x, v, m, P, s); break;
    case 16: launch_proj_t<16>(U, x, v, m, P, s); break;
    default: launch_proj_t<32>(U, x, v, m, P, s); break;
  }
}

template <int MAXJ>
void launch_resid_t(double* U, const double* x, const StateView& v, const ScratchMem& m, const IsvdParams& P,
                    cudaStream_t s, int phase) {
  const size_t smem = ((size_t)kTileRows * P.ccap + P.ccap + 1 + 3 * kTileRows + 4 * kTileRows) * 8;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    STROM_CUDA(cudaFuncSetAttribute(k_resid<MAXJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = smem;
  }
  ProfScope ps(P_RESID, s);
  k_resid<MAXJ><<<m.grid, kPassThreads, smem, s>>>(U, x, v, m.sc, P, phase);
  STROM_LAUNCH_CHECK();
}

void launch_resid(int ccap, double* U, const double* x, const StateView& v, const ScratchMem& m,
                  const IsvdParams& P, cudaStream_t s, int phase = 0) {
  switch (maxj_for(ccap)) {
    case 2: launch_resid_t<2>(U, x, v, m, P, s, phase); break;
    case 4: launch_resid_t<4>(U, x, v, m, P, s, phase); break;
    case 8: launch_resid_t<8>(U, x, v, m, P, s, phase); break;
    case 16: launch_resid_t<16>(U, x, v, m, P, s, phase); break;
    default: launch_resid_t<32>(U, x, v, m, P, s, phase); break;
  }
}

size_t small_kernel_smem(const Caps& c, int* use_smem) {
  // step B layout: 3 m^2 + 16 ms (secular work) + ccap m (staged W_b / QR's M)
  const size_t m = c.rcap + 1;
  const size_t ms = round_up(std::max<int64_t>(c.ccap, c.rcap + 2), 32);
  const size_t need = (3 * m * m + 16 * ms + (size_t)c.ccap * m) * 8;
  const size_t limit = max_smem_optin() - 8 * 1024;
  *use_smem = need <= limit ? 1 : 0;
  return *use_smem ? need : 0;
}

void launch_step_b(const StateView& src, const StateView& dst, const ScratchMem& m, const IsvdParams& P,
                   const Caps& caps, cudaStream_t s) {
  int use_smem = 0;
  const size_t smem = small_kernel_smem(caps, &use_smem);
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    STROM_CUDA(cudaFuncSetAttribute(k_step_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = smem;
  }
  ProfScope ps(P_STEP_B, s);
  k_step_b<<<1, kSmallThreads, smem, s>>>(src, dst, m.sc, P, use_smem);
  STROM_LAUNCH_CHECK();
}

void launch_compact_prep(const StateView& src, const StateView& dst, const ScratchMem& m, const IsvdParams& P,
                         const Caps& caps, cudaStream_t s) {
  int use_smem = 0;
  const size_t smem = small_kernel_smem(caps, &use_smem);
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    STROM_CUDA(cudaFuncSetAttribute(k_compact_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = smem;
  }
  ProfScope ps(P_COMPACT, s);
  k_compact_prep<<<1, kSmallThreads, smem, s>>>(src, dst, m.sc, P, use_smem);
  STROM_LAUNCH_CHECK();
}

void launch_tall_gemm(const double* A, int64_t lda, const int32_t* col0_dev, const double* T, int64_t ldt,
                      const int32_t* p_dev, const int32_t* q_dev, double* out, int64_t ldo, bool row_major,
                      int64_t n, int64_t nrows_pad, cudaStream_t s) {
  const int64_t tiles = ceil_div(nrows_pad, kGemmRows);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sm_count() * 4));
  ProfScope ps(P_TALL_GEMM, s);
  k_tall_gemm<<<grid, 256, kGemmKc * 64 * 8, s>>>(A, lda, col0_dev, 0, T, ldt, p_dev, q_dev, 0, out, ldo,
                                                  row_major ? 1 : 0, n, nrows_pad);
  STROM_LAUNCH_CHECK();
}

// L = chol(A[:, col0:col0+q]^T A[:, col0:col0+q]) with the DMMA tall Gram.
// q is read on the device (q_dev) or fixed; the Cholesky reads c from hdr_c.
void gram_cholesky(const double* A, int64_t lda, const int32_t* col0_dev, const int32_t* q_dev, int q_fixed,
                   int qmax, int64_t n, double* L, double* Li, int ldl, const IsvdHdr* hdr_c, int* status_dev,
                   cudaStream_t s) {
  const int QP = (int)round_up(std::max(qmax, 1), 8);
  const int64_t ntiles = ceil_div(n, kGramRows);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)sm_count() * 2));
  auto part = dev_alloc((size_t)grid * QP * QP * 8, s, false);
  const size_t smem = (size_t)QP * kGramLd * 8;
  ProfScope ps(P_OTHER, s);
  if (QP <= 64) {
    k_tall_gram<1, 8><<<grid, 256, smem, s>>>(A, lda, col0_dev, q_dev, q_fixed, n, part->as<double>(), QP);
  } else if (QP <= 128) {
    static bool cfg = false;
    if (!cfg) {
      STROM_CUDA(cudaFuncSetAttribute(k_tall_gram<2, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
      cfg = true;
    }
    k_tall_gram<2, 16><<<grid, 256, smem, s>>>(A, lda, col0_dev, q_dev, q_fixed, n, part->as<double>(), QP);
  } else {
    throw Error(kInvalidArgument, "Gram of more than 128 columns is not supported");
  }
  STROM_LAUNCH_CHECK();
  k_gram_reduce<<<(unsigned)ceil_div((int64_t)QP * QP, 256), 256, 0, s>>>(part->as<double>(), grid, QP, q_dev,
                                                                          q_fixed, L, ldl);
  STROM_LAUNCH_CHECK();
  k_cholesky<<<1, 256, 0, s>>>(L, ldl, hdr_c, q_fixed, status_dev);
  STROM_LAUNCH_CHECK();
  k_lower_inverse<<<1, 1024, 0, s>>>(L, ldl, hdr_c, q_fixed, Li);
  STROM_LAUNCH_CHECK();
}

// Compaction into fresh buffers (also used to grow capacities):
// U_new = U[:, base:base+c] L^{-T} Q_c,  W_new = R_c,  L_new = I.
strom_isvd* compact(strom_isvd* src, const Caps& caps, cudaStream_t s) {
  strom_isvd* t = new_like(src, caps);
  alloc_small(t, s);
  t->vmem = src->vmem;  // V is immutable: share it
  t->view.V = src->view.V;
  t->view.ldv = src->view.ldv;
  t->caps.kcap = src->caps.kcap;
  t->U = alloc_u(src->ldu, caps.ccap, s);
  ScratchMem m = make_scratch(src->ldu, caps.ccap >= src->caps.ccap ? caps : src->caps, s);
  IsvdParams P = make_params(src, m, src->k, false);
  P.ccap = std::max(caps.ccap, src->caps.ccap);
  P.work_stride = m.work_stride;
  Caps kc = caps;
  kc.ccap = std::max(caps.ccap, src->caps.ccap);
  kc.rcap = std::max(caps.rcap, src->caps.rcap);
  launch_compact_prep(src->view, t->view, m, P, kc, s);
  // p = source c (step->m), q = r (step->mkeep)
  launch_tall_gemm(src->U->ptr(), src->ldu, &src->view.hdr->base, m.sc.T, P.ccap, &m.sc.step->m,
                   &m.sc.step->mkeep, t->U->ptr(), t->ldu, false, t->n, t->ldu, s);
  // measure the Gram of the stored U_new: L describes the memory, not an assumed identity
  gram_cholesky(t->U->ptr(), t->ldu, nullptr, &m.sc.step->mkeep, 0, caps.rcap, t->n, t->view.L, t->view.Li,
                t->view.ldl, t->view.hdr, reinterpret_cast<int*>(&m.sc.step->pad_status), s);
  k_compact_finish<<<1, 256, 0, s>>>(t->view, m.sc.T, P.ccap);
  STROM_LAUNCH_CHECK();
  t->r_ub = std::min(src->r_ub, caps.rcap);
  t->c_ub = t->r_ub;
  t->U->claimed = t->c_ub;
  return t;
}

void read_hdr(const strom_isvd* h, cudaStream_t s, IsvdHdr* out) {
  STROM_CUDA(cudaMemcpyAsync(out, h->view.hdr, sizeof(IsvdHdr), cudaMemcpyDeviceToHost, s));
  STROM_CUDA(cudaStreamSynchronize(s));
}

// One functional update cur -> new state (all device-side decisions).
strom_isvd* update_once(strom_isvd* src, const double* x, ScratchMem* scratch, cudaStream_t s,
                        std::shared_ptr<strom_isvd>* keep) {
  strom_isvd* cur = src;
  std::unique_ptr<strom_isvd> tmp;
  // rank capacity (uncapped streams grow; capped streams are sized by r_max)
  if (cur->r_max < 0 && cur->r_ub + 1 > cur->caps.rcap && cur->caps.rcap < cur->n) {
    IsvdHdr hh;
    read_hdr(cur, s, &hh);
    cur->r_ub = hh.r;
    cur->c_ub = std::min(cur->c_ub, hh.base + hh.c);
    if (hh.r + 1 > cur->caps.rcap) {
      Caps nc = make_caps(cur->n, -1, std::min<int64_t>(cur->n, 2 * (int64_t)cur->caps.rcap), cur->k);
      nc.kcap = cur->caps.kcap;
      tmp.reset(compact(cur, nc, s));
      cur = tmp.get();
      *scratch = ScratchMem();
    }
  }
  // physical column capacity: host-scheduled compaction
  if (cur->c_ub + 1 > cur->caps.ccap) {
    strom_isvd* t = compact(cur, cur->caps, s);
    tmp.reset(t);
    cur = t;
  }
  if (!scratch->mem || scratch->pstride != (int)round_up(cur->caps.ccap + 2, 8)) {
    *scratch = make_scratch(cur->ldu, cur->caps, s);
  }
  Caps nc = cur->caps;
  if (cur->k + 1 > nc.kcap) nc.kcap = round_up((cur->k + 1) * 2, 64);
  strom_isvd* dst = new_like(cur, nc);
  dst->k = cur->k + 1;
  alloc_small(dst, s);
  alloc_v(dst, s);
  // append-only store: share unless another state already claimed beyond cur
  if (cur->U->claimed != cur->c_ub) {
    auto u = alloc_u(cur->ldu, cur->caps.ccap, s);
    STROM_CUDA(cudaMemcpyAsync(u->ptr(), cur->U->ptr(), (size_t)cur->ldu * cur->c_ub * 8,
                               cudaMemcpyDeviceToDevice, s));
    dst->U = u;
  } else {
    dst->U = cur->U;
  }
  IsvdParams P = make_params(cur, *scratch, dst->k, false);
  launch_proj(P.ccap, dst->U->ptr(), x, cur->view, *scratch, P, s);
  {
    ProfScope ps(P_STEP_A, s);
    k_step_a<<<1, 256, 0, s>>>(cur->view, scratch->sc, P);
    STROM_LAUNCH_CHECK();
  }
  launch_resid(P.ccap, dst->U->ptr(), x, cur->view, *scratch, P, s, 0);
  {
    ProfScope ps(P_STEP_B, s);
    k_step_b1<<<1, 256, 0, s>>>(cur->view, scratch->sc, P);
    STROM_LAUNCH_CHECK();
  }
  launch_resid(P.ccap, dst->U->ptr(), nullptr, cur->view, *scratch, P, s, 1);
  launch_step_b(cur->view, dst->view, *scratch, P, cur->caps, s);
  {
    dim3 grid((unsigned)ceil_div(dst->k, kVRows), (unsigned)ceil_div(cur->caps.rcap + 1, kVCols));
    ProfScope ps(P_VUPDATE, s);
    k_vupdate<<<grid, kVRows, (size_t)(cur->caps.rcap + 2) * kVCols * 8, s>>>(cur->view, dst->view, scratch->sc, P);
    STROM_LAUNCH_CHECK();
  }
  dst->c_ub = cur->c_ub + 1;
  dst->U->claimed = std::max(dst->U->claimed, dst->c_ub);
  dst->r_ub = std::min(cur->r_ub + 1, cur->caps.rcap);
  (void)keep;
  return dst;
}

strom_isvd* init_state(int64_t n, const double* x, int64_t k, double tol_svd, double tol_sv, int64_t r_max,
                       int32_t cap_mode, cudaStream_t s) {
  STROM_REQUIRE(n >= 1, "need n >= 1");
  STROM_REQUIRE(k >= 1, "need k >= 1");
  STROM_REQUIRE(cap_mode == 0 || cap_mode == 1, "unknown cap_mode");
  auto* h = new strom_isvd();
  h->n = n;
  h->ldu = round_up(n, kGemmRows);
  h->k = k;
  h->tol_svd = tol_svd;
  h->tol_sv = tol_sv;
  h->r_max = (int32_t)r_max;
  h->cap_mode = cap_mode;
  h->caps = make_caps(n, h->r_max, 1, k);
  alloc_small(h, s);
  alloc_v(h, s);
  h->U = alloc_u(h->ldu, h->caps.ccap, s);
  ScratchMem m = make_scratch(h->ldu, h->caps, s);
  // fresh header: r = c = base = 0 (zeroed allocation) -> the restart path
  IsvdParams P = make_params(h, m, k, true);
  // run the update machinery from an empty source state into h itself
  auto src_small = dev_alloc(256, s, true);
  StateView sv = h->view;
  sv.hdr = src_small->as<IsvdHdr>();
  launch_proj(P.ccap, h->U->ptr(), x, sv, m, P, s);
  k_step_a<<<1, 256, 0, s>>>(sv, m.sc, P);
  STROM_LAUNCH_CHECK();
  launch_resid(P.ccap, h->U->ptr(), x, sv, m, P, s);
  launch_step_b(sv, h->view, m, P, h->caps, s);
  {
    dim3 grid((unsigned)ceil_div(k, kVRows), 1);
    k_vupdate<<<grid, kVRows, (size_t)(h->caps.rcap + 2) * kVCols * 8, s>>>(sv, h->view, m.sc, P);
    STROM_LAUNCH_CHECK();
  }
  h->c_ub = 1;
  h->U->claimed = 1;
  h->r_ub = 1;
  return h;
}

}  // namespace

// =========================================================================
extern "C" {

int strom_isvd_init(int64_t n, const double* x_dev, int64_t k, double tol_svd, double tol_sv, int64_t r_max,
                    int32_t cap_mode, void* stream, strom_isvd** out) {
  return guarded([&] {
    STROM_REQUIRE(out && x_dev, "null argument");
    *out = init_state(n, x_dev, k, tol_svd, tol_sv, r_max, cap_mode, as_stream(stream));
  });
}

int strom_isvd_update(strom_isvd* src, const double* x_dev, void* stream, strom_isvd** out) {
  return guarded([&] {
    STROM_REQUIRE(src && out && x_dev, "null argument");
    ScratchMem m;
    *out = update_once(src, x_dev, &m, as_stream(stream), nullptr);
  });
}

int strom_isvd_ingest(strom_isvd* src, const double* X, int64_t ldx, int64_t ncols, int32_t x_on_host,
                      void* stream, strom_isvd** out) {
  return guarded([&] {
    STROM_REQUIRE(src && out, "null argument");
    STROM_REQUIRE(ncols >= 0 && ldx >= src->n, "bad ingest shape");
    cudaStream_t s = as_stream(stream);
    ScratchMem m;
    std::unique_ptr<strom_isvd> cur;
    strom_isvd* c0 = src;
    if (ncols == 0) {
      // a copy of the state (new handle sharing immutable buffers)
      auto* h = new strom_isvd(*src);
      *out = h;
      return;
    }
    if (!x_on_host) {
      for (int64_t t = 0; t < ncols; ++t) {
        strom_isvd* nx = update_once(cur ? cur.get() : c0, X + t * ldx, &m, s, nullptr);
        cur.reset(nx);
      }
      *out = cur.release();
      return;
    }
    // host columns: chunked H2D on a copy stream, overlapped with the updates
    const int64_t chunk = 16;
    const int nring = 3;
    const int64_t n = src->n;
    cudaStream_t cs;
    STROM_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    std::vector<DevMemPtr> ring(nring);
    std::vector<cudaEvent_t> ready(nring), freed(nring);
    for (int i = 0; i < nring; ++i) {
      ring[i] = dev_alloc((size_t)n * chunk * 8, s, false);
      STROM_CUDA(cudaEventCreateWithFlags(&ready[i], cudaEventDisableTiming));
      STROM_CUDA(cudaEventCreateWithFlags(&freed[i], cudaEventDisableTiming));
      STROM_CUDA(cudaEventRecord(freed[i], s));
    }
    const int64_t nchunks = ceil_div(ncols, chunk);
    auto issue = [&](int64_t q) {
      const int slot = (int)(q % nring);
      const int64_t c0i = q * chunk, cn = std::min(chunk, ncols - c0i);
      STROM_CUDA(cudaStreamWaitEvent(cs, freed[slot], 0));
      STROM_CUDA(cudaMemcpy2DAsync(ring[slot]->ptr, n * 8, X + c0i * ldx, ldx * 8, n * 8, cn,
                                   cudaMemcpyHostToDevice, cs));
      STROM_CUDA(cudaEventRecord(ready[slot], cs));
    };
    for (int64_t q = 0; q < std::min<int64_t>(nring, nchunks); ++q) issue(q);
    for (int64_t q = 0; q < nchunks; ++q) {
      const int slot = (int)(q % nring);
      STROM_CUDA(cudaStreamWaitEvent(s, ready[slot], 0));
      const int64_t c0i = q * chunk, cn = std::min(chunk, ncols - c0i);
      for (int64_t t = 0; t < cn; ++t) {
        strom_isvd* nx = update_once(cur ? cur.get() : c0, ring[slot]->as<double>() + t * n, &m, s, nullptr);
        cur.reset(nx);
      }
      STROM_CUDA(cudaEventRecord(freed[slot], s));
      if (q + nring < nchunks) issue(q + nring);
    }
    STROM_CUDA(cudaStreamSynchronize(cs));
    for (int i = 0; i < nring; ++i) {
      cudaEventDestroy(ready[i]);
      cudaEventDestroy(freed[i]);
    }
    cudaStreamDestroy(cs);
    *out = cur.release();
  });
}

int strom_isvd_query(strom_isvd* h, void* stream, strom_isvd_info* out) {
  return guarded([&] {
    STROM_REQUIRE(h && out, "null argument");
    IsvdHdr hh;
    read_hdr(h, as_stream(stream), &hh);
    h->r_ub = hh.r;  // refine the host bounds while we are synchronised
    memset(out, 0, sizeof(*out));
    out->n = h->n;
    out->k = h->k;
    out->rank = hh.r;
    out->ncols_u = hh.c;
    out->n_rejected = hh.n_rejected;
    out->n_dependent = hh.n_dependent;
    out->n_truncated = hh.n_truncated;
    out->n_restarts = hh.n_restarts;
    out->flags = hh.flags;
    out->status = hh.status ? STROM_ENUMERIC : 0;
    out->last_p = hh.p;
    out->last_drift = hh.drift;
    out->last_xnorm = hh.xnorm;
    out->last_p_sq = hh.p_sq;
    out->tol_svd = h->tol_svd;
    out->tol_sv = h->tol_sv;
    out->r_max = h->r_max;
    out->cap_mode = h->cap_mode;
  });
}

int strom_isvd_export(strom_isvd* h, double* phi_dev, double* sigma_dev, double* v_dev, void* stream) {
  return guarded([&] {
    STROM_REQUIRE(h, "null argument");
    cudaStream_t s = as_stream(stream);
    IsvdHdr hh;
    read_hdr(h, s, &hh);
    const int r = hh.r;
    if (phi_dev && r > 0) {
      auto wtmp = dev_alloc((size_t)std::max(hh.c, 1) * r * 8, s, false);
      k_n_to_w<<<(unsigned)std::max<int64_t>(1, ceil_div((int64_t)hh.c * r, 256)), 256, 0, s>>>(h->view,
                                                                                              wtmp->as<double>());
      STROM_LAUNCH_CHECK();
      launch_tall_gemm(h->U->ptr(), h->ldu, &h->view.hdr->base, wtmp->as<double>(), hh.c, &h->view.hdr->c,
                       &h->view.hdr->r, phi_dev, r, true, h->n, h->ldu, s);
    }
    if (sigma_dev && r > 0)
      STROM_CUDA(cudaMemcpyAsync(sigma_dev, h->view.sigma, r * 8, cudaMemcpyDeviceToDevice, s));
    if (v_dev && r > 0) {
      const int64_t tot = h->k * r;
      k_cm_to_rm<<<(unsigned)ceil_div(tot, 256), 256, 0, s>>>(h->view.V, h->view.ldv, h->k, r, v_dev);
      STROM_LAUNCH_CHECK();
    }
  });
}

int strom_isvd_load_factored(int64_t n, int64_t k, int64_t c, int64_t r, const double* u_dev, int64_t ldu,
                             const double* w_dev, int64_t ldw, const double* l_dev, int64_t ldl,
                             const double* sigma_dev, const double* v_dev, double tol_svd, double tol_sv,
                             int64_t r_max, int32_t cap_mode, const int32_t* counters4, void* stream,
                             strom_isvd** out) {
  return guarded([&] {
    STROM_REQUIRE(out, "null argument");
    STROM_REQUIRE(n >= 1 && k >= 1 && r >= 0 && c >= r && c <= n, "bad load shape");
    STROM_REQUIRE(cap_mode == 0 || cap_mode == 1, "unknown cap_mode");
    cudaStream_t s = as_stream(stream);
    auto* h = new strom_isvd();
    std::unique_ptr<strom_isvd> guard(h);
    h->n = n;
    h->ldu = round_up(n, kGemmRows);
    h->k = k;
    h->tol_svd = tol_svd;
    h->tol_sv = tol_sv;
    h->r_max = (int32_t)r_max;
    h->cap_mode = cap_mode;
    h->caps = make_caps(n, h->r_max, (int32_t)std::max<int64_t>(c, r + 1), k);
    STROM_REQUIRE(c + 1 <= h->caps.ccap, "too many factored columns for this capacity");
    alloc_small(h, s);
    alloc_v(h, s);
    h->U = alloc_u(h->ldu, h->caps.ccap, s);
    if (c > 0) {
      STROM_CUDA(cudaMemcpy2DAsync(h->U->ptr(), h->ldu * 8, u_dev, ldu * 8, n * 8, c, cudaMemcpyDeviceToDevice, s));
    }
    const int th = 256;
    if (c > 0 && r > 0) {
      k_copy_cm<<<(unsigned)ceil_div(c * r, th), th, 0, s>>>(w_dev, ldw, c, r, h->view.N, h->view.ldn);
      STROM_LAUNCH_CHECK();
      STROM_CUDA(cudaMemcpyAsync(h->view.sigma, sigma_dev, r * 8, cudaMemcpyDeviceToDevice, s));
    }
    if (r > 0) {
      k_rm_to_cm<<<(unsigned)ceil_div(k * r, th), th, 0, s>>>(v_dev, k, r, h->view.V, h->view.ldv);
      STROM_LAUNCH_CHECK();
    }
    int zero[4] = {0, 0, 0, 0};
    const int32_t* cnt = counters4 ? counters4 : zero;
    k_set_hdr<<<1, 1, 0, s>>>(h->view.hdr, (int32_t)r, (int32_t)c, 0, cnt[0], cnt[1], cnt[2], cnt[3]);
    STROM_LAUNCH_CHECK();
    if (c > 0) {
      if (l_dev) {
        k_copy_cm<<<(unsigned)ceil_div(c * c, th), th, 0, s>>>(l_dev, ldl, c, c, h->view.L, h->view.ldl);
        STROM_LAUNCH_CHECK();
        k_lower_inverse<<<1, 1024, 0, s>>>(h->view.L, h->view.ldl, nullptr, (int)c, h->view.Li);
        STROM_LAUNCH_CHECK();
      } else {
        // measure the Gram of the stored U (exact L even for a nearly orthonormal U)
        auto st = dev_alloc(sizeof(int), s, true);
        gram_cholesky(h->U->ptr(), h->ldu, nullptr, nullptr, (int)c, (int)c, n, h->view.L, h->view.Li,
                      h->view.ldl, nullptr, st->as<int>(), s);
        int bad = 0;
        STROM_CUDA(cudaMemcpyAsync(&bad, st->ptr, sizeof(int), cudaMemcpyDeviceToHost, s));
        STROM_CUDA(cudaStreamSynchronize(s));
        if (bad) throw Error(kNumericalError, "U is numerically rank-deficient (Gram not positive definite)");
      }
    }
    if (c > 0 && r > 0) {  // coordinates in the orthonormal basis U L^{-T}: N = L^T W
      auto tmp = dev_alloc((size_t)c * r * 8, s, false);
      k_w_to_n<<<1, 256, 0, s>>>(h->view, tmp->as<double>());
      STROM_LAUNCH_CHECK();
    }
    h->c_ub = (int32_t)c;
    h->U->claimed = (int32_t)c;
    h->r_ub = (int32_t)r;
    *out = guard.release();
  });
}

int strom_isvd_load(int64_t n, int64_t k, int64_t r, const double* phi_dev, const double* sigma_dev,
                    const double* v_dev, double tol_svd, double tol_sv, int64_t r_max, int32_t cap_mode,
                    const int32_t* counters4, void* stream, strom_isvd** out) {
  return guarded([&] {
    STROM_REQUIRE(out, "null argument");
    STROM_REQUIRE(n >= 1 && k >= 1 && r >= 0 && r <= n, "bad load shape");
    cudaStream_t s = as_stream(stream);
    // phi (row-major n x r) -> column-major U; W = I; L = chol(U^T U)
    auto ucm = dev_alloc((size_t)std::max<int64_t>(1, n * r) * 8, s, false);
    auto wid = dev_alloc((size_t)std::max<int64_t>(1, r * r) * 8, s, true);
    const int th = 256;
    if (r > 0) {
      k_rm_to_cm<<<(unsigned)ceil_div(n * r, th), th, 0, s>>>(phi_dev, n, r, ucm->as<double>(), n);
      STROM_LAUNCH_CHECK();
      std::vector<double> eye((size_t)r * r, 0.0);
      for (int64_t i = 0; i < r; ++i) eye[i * r + i] = 1.0;
      STROM_CUDA(cudaMemcpyAsync(wid->ptr, eye.data(), eye.size() * 8, cudaMemcpyHostToDevice, s));
      STROM_CUDA(cudaStreamSynchronize(s));
    }
    strom_isvd* h = nullptr;
    int rc = strom_isvd_load_factored(n, k, r, r, ucm->as<double>(), n, wid->as<double>(), std::max<int64_t>(r, 1),
                                      nullptr, 0, sigma_dev, v_dev, tol_svd, tol_sv, r_max, cap_mode, counters4,
                                      stream, &h);
    if (rc) throw Error(rc, strom_last_error());
    std::unique_ptr<strom_isvd> guard(h);
    *out = guard.release();
  });
}

// Representation dump for the invariant tests: U[:, base:base+c] (n x c,
// column-major, ld n), W (c x r, column-major, ld c), L (c x c, ld c).
int strom_isvd_factors(strom_isvd* h, double* u_dev, double* w_dev, double* l_dev, void* stream) {
  return guarded([&] {
    STROM_REQUIRE(h, "null argument");
    cudaStream_t s = as_stream(stream);
    IsvdHdr hh;
    read_hdr(h, s, &hh);
    if (u_dev && hh.c > 0)
      STROM_CUDA(cudaMemcpy2DAsync(u_dev, h->n * 8, h->U->ptr() + (int64_t)hh.base * h->ldu, h->ldu * 8, h->n * 8,
                                   hh.c, cudaMemcpyDeviceToDevice, s));
    if (w_dev && hh.c > 0 && hh.r > 0) {
      k_n_to_w<<<(unsigned)ceil_div((int64_t)hh.c * hh.r, 256), 256, 0, s>>>(h->view, w_dev);
      STROM_LAUNCH_CHECK();
    }
    if (l_dev && hh.c > 0)
      STROM_CUDA(cudaMemcpy2DAsync(l_dev, hh.c * 8, h->view.L, h->view.ldl * 8, hh.c * 8, hh.c,
                                   cudaMemcpyDeviceToDevice, s));
    STROM_CUDA(cudaStreamSynchronize(s));
  });
}

// Diagnostics: point step B's phase timestamps (clock64, 8 slots) at a device
// buffer, or NULL to disable.
void strom_debug_tprobe(long long* dev_buf) { g_tprobe = dev_buf; }

void strom_isvd_free(strom_isvd* h) { delete h; }

}  // extern "C"
