// Host orchestration + C ABI of the streaming incremental SVD
// (reference basis.py:30-194).  See isvd_kernels.cuh for the representation.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <thread>
#include <string>
#include <mutex>
#include <condition_variable>
#include <vector>

#include "../../include/strom_b200.h"
#include "gram.cuh"
#include "isvd_kernels.cuh"
#include "isvd_window.cuh"
#include "runtime.cuh"
#include "shard.cuh"

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

// out(i, j) = in(i, j) for i < rows, j < cols (layout conversion between Tall views)
__global__ void k_copy_tall(Tall in, int64_t rows, int64_t cols, Tall out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * cols) return;
  const int64_t i = idx % rows, j = idx / rows;
  out.p[out.off(i, j)] = in.p[in.off(i, j)];
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

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Launch with programmatic stream serialization (PDL): the kernel may start
// while its predecessor on the stream is still running; it calls pdl_enter()
// before touching the predecessor's results.  STROM_NO_PDL=1 disables it.
bool pdl_enabled() {
  static const bool v = [] {
    const char* e = getenv("STROM_NO_PDL");
    return !(e && atoi(e) != 0);
  }();
  return v;
}

template <class... KArgs, class... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  STROM_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// diagnostics: STROM_TRACE=1 synchronises and names every launch of the update
void trace_point(const char* what, cudaStream_t s) {
  static const bool on = [] {
    const char* e = getenv("STROM_TRACE");
    return e && atoi(e) != 0;
  }();
  if (!on) return;
  fprintf(stderr, "[strom] %s ...", what);
  fflush(stderr);
  cudaError_t e = cudaStreamSynchronize(s);
  fprintf(stderr, " %s\n", cudaGetErrorString(e));
}

long long* g_tprobe = nullptr;     // step-B phase timestamps (strom_debug_tprobe)
long long* g_trace = nullptr;      // strom_debug_trace: 16 stamps per update of the next ingest calls
int64_t g_trace_rows = 0;
long long* g_cur_trace = nullptr;  // the row of the update being launched (window mode)

// ------------------------------------------------------------------ state
// The append-only store shared by a state and its successors: U (ldu x ccap,
// row-tiled: kUTile-row tiles, each holding its ccap column segments
// contiguously, so one pass stage is one contiguous bulk copy) and the exact factors L, L^{-1} of G = U^T U, indexed
// by physical column.  `claimed` bounds the physical columns any live state
// may have written: a successor that would append past a state whose c_ub is
// below `claimed` copies the store first (copy-on-write).
// A large store's U block outlives its Store in a one-slot spare cache (per device): a
// compaction ping-pongs between two blocks of the same size, and a fresh 75 GB allocation
// costs the driver ~0.4 s (cfg5) even from the stream-ordered pool's point of view when the
// pool cannot hand the freed block back.  Reuse is on the stream that allocated the block
// (stream order covers the last owner's kernels); anything else takes the allocator.
constexpr size_t kSpareStoreMin = (size_t)1 << 30;
struct SpareStore {
  std::mutex mu;
  DevMemPtr mem[kMaxDevices];
  int live[kMaxDevices] = {};  // stores alive per device: the spare goes when the last one does
};
SpareStore& spare_store() {
  static SpareStore s;
  return s;
}

struct Store {
  DevMemPtr umem, lmem;
  int64_t ldu = 0;
  int32_t ccap = 0;
  int32_t claimed = 0;
  int dev = 0;
  Store() {
    dev = current_device_id();
    SpareStore& sp = spare_store();
    std::lock_guard<std::mutex> g(sp.mu);
    ++sp.live[dev];
  }
  Store(const Store&) = delete;
  Store& operator=(const Store&) = delete;
  ~Store() {
    SpareStore& sp = spare_store();
    std::lock_guard<std::mutex> g(sp.mu);
    DevMemPtr& slot = sp.mem[dev];
    if (--sp.live[dev] <= 0) {
      slot.reset();  // nothing left to compact: hold no memory
    } else if (umem && umem->bytes >= kSpareStoreMin && umem.use_count() == 1) {
      if (!slot || slot->bytes < umem->bytes) slot = std::move(umem);  // the smaller one goes back to the pool
    }
  }
  double* U() const { return umem->as<double>(); }
  double* L() const { return lmem->as<double>(); }
  double* Li() const { return L() + (size_t)ccap * ccap; }
};

struct Caps {
  int32_t rcap = 0, ccap = 0;
  int64_t kcap = 0;
};


// ------------------------------------------------------------------ row sharding (shard.cuh)
// Single-process groups (the one-GPU test harness): the ranks are host threads
// of one process; their exchanges are ordered by stream events, so no kernel
// ever waits for another rank's kernel.
struct LocalSync {
  std::mutex mu;
  std::condition_variable cv;
  int world = 1, arrived = 0;
  uint64_t gen = 0;
  bool broken = false;
  static constexpr int kRing = 4;
  cudaEvent_t ev[kShardMax][kRing] = {};
  ~LocalSync() {
    for (int r = 0; r < kShardMax; ++r)
      for (int i = 0; i < kRing; ++i)
        if (ev[r][i]) cudaEventDestroy(ev[r][i]);
  }
  void barrier() {
    std::unique_lock<std::mutex> g(mu);
    if (broken) throw Error(kInternal, "shard group: a rank left the exchange");
    const uint64_t my = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    if (!cv.wait_for(g, std::chrono::seconds(60), [&] { return gen != my || broken; })) {
      broken = true;
      cv.notify_all();
      throw Error(kInternal, "shard group: the ranks' exchange sequences diverged (host barrier timed out)");
    }
    if (broken && gen == my) throw Error(kInternal, "shard group: a rank left the exchange");
  }
};

struct MailboxMem {  // one rank's [flags | boxes] block (cudaMalloc: exportable by CUDA IPC)
  void* ptr = nullptr;
  explicit MailboxMem(size_t bytes) {
    STROM_CUDA(cudaMalloc(&ptr, bytes));
    STROM_CUDA(cudaMemset(ptr, 0, bytes));
  }
  ~MailboxMem() {
    if (ptr) cudaFree(ptr);
  }
};

struct ShardImpl {
  int rank = 0, world = 1, device = 0;
  int64_t n_global = 0;
  std::shared_ptr<MailboxMem> box_mem;
  std::vector<std::shared_ptr<MailboxMem>> peers_mem;  // single-process groups: the peers' blocks stay alive
  void* mailbox = nullptr;
  size_t mailbox_bytes = 0;
  void* peer[kShardMax] = {};
  bool ipc_opened[kShardMax] = {};
  void* local = nullptr;  // seq counter + error word
  bool connected = false;
  ShardDev dev{};
  std::shared_ptr<LocalSync> lsync;  // event-ordered mode
  uint64_t nsync = 0;
  static constexpr size_t kFlagBytes = 1024;
  static size_t bytes_for(int world) {
    return kFlagBytes + (size_t)kShardSlots * world * kShardMaxCount * 8;
  }
  void alloc(int world_) {
    world = world_;
    STROM_CUDA(cudaGetDevice(&device));
    mailbox_bytes = bytes_for(world);
    box_mem = std::make_shared<MailboxMem>(mailbox_bytes);
    mailbox = box_mem->ptr;
    STROM_CUDA(cudaMalloc(&local, 64));
    STROM_CUDA(cudaMemset(local, 0, 64));
    STROM_CUDA(cudaDeviceSynchronize());
  }
  void finish(int rank_, int64_t n_global_) {
    rank = rank_;
    n_global = n_global_;
    dev.rank = rank;
    dev.world = world;
    dev.maxcount = kShardMaxCount;
    for (int p = 0; p < world; ++p) {
      dev.flag[p] = static_cast<unsigned long long*>(peer[p]);
      dev.box[p] = reinterpret_cast<double*>(static_cast<char*>(peer[p]) + kFlagBytes);
    }
    dev.seq = static_cast<unsigned long long*>(local);
    dev.err = reinterpret_cast<int32_t*>(static_cast<char*>(local) + 16);
    const char* e = getenv("STROM_SHARD_TIMEOUT_MS");
    dev.timeout_ns = (long long)(e && atoll(e) > 0 ? atoll(e) : 5000) * 1000000ll;
    connected = true;
  }
  ~ShardImpl() {
    for (int p = 0; p < kShardMax; ++p)
      if (ipc_opened[p] && peer[p]) cudaIpcCloseMemHandle(peer[p]);
    if (local) cudaFree(local);
  }
};

thread_local std::shared_ptr<ShardImpl> t_current_shard;  // strom_shard_make_current

}  // namespace

struct strom_shard {
  std::shared_ptr<ShardImpl> impl;
};

struct strom_isvd {
  int64_t n = 0, ldu = 0, k = 0;
  int64_t n_global = 0;  // rows of the whole (sharded) matrix; == n for an unsharded state
  std::shared_ptr<ShardImpl> shard;  // row-sharded: the exchange after every partial reduction
  double tol_svd = 0.0, tol_sv = 0.0;
  int32_t r_max = -1, cap_mode = 0;
  Caps caps;
  int32_t c_ub = 0;  // bound on base + c (physical end of used columns)
  int32_t r_ub = 0;  // bound on rank
  std::shared_ptr<Store> store;
  DevMemPtr small, vmem;
  StateView view{};
};

namespace {

// ccap = rcap + 1 + slack
int32_t slack_for(int32_t rcap) {
  static const int env = [] {
    const char* e = getenv("STROM_SLACK");
    return e ? atoi(e) : 0;
  }();
  if (env > 0) return env;  // diagnostics
  // passes read ~r + slack/2 columns; a compaction (one DMMA sweep) costs about
  // as much as ~1000 column reads and recurs every ~3 slack updates at cfg2
  return std::max<int32_t>(16, rcap / 2);
}

// n bounds the rank (the matrix's rows: the GLOBAL count of a sharded state);
// mem_rows sizes the store (this GPU's rows; for a sharded state the largest
// row block of the group, so that every rank derives the same capacities and
// with them the same compaction schedule).
Caps make_caps(int64_t n, int32_t r_max, int32_t want_r, int64_t k, int64_t mem_rows = -1) {
  if (mem_rows < 0) mem_rows = n;
  Caps c;
  int64_t rc;
  if (r_max >= 0) rc = std::min<int64_t>(std::max<int32_t>(r_max, 1), n);
  else rc = std::min<int64_t>(std::max<int32_t>(want_r, 32), n);
  rc = std::max<int64_t>(rc, 1);
  if (rc > 254) throw Error(kInvalidArgument, "rank capacity above 254 is not supported by this build");
  c.rcap = (int32_t)rc;
  c.ccap = std::min<int32_t>(256, c.rcap + 1 + slack_for(c.rcap));
  // capacity: a compaction holds two stores at once; keep both within ~80% of
  // HBM by trimming the slack (cfg5: 2^26 rows, 0.54 GB per column)
  const size_t total_b = device_total_mem();
  if (total_b > 0) {
    const int64_t col_bytes = round_up(mem_rows, 128) * 8;
    const int64_t max_cols = (int64_t)(0.40 * (double)total_b) / col_bytes;
    if (c.ccap > max_cols) c.ccap = (int32_t)std::max<int64_t>(c.rcap + 1 + 8, max_cols);
  }
  c.kcap = std::max<int64_t>(64, round_up(std::max<int64_t>(k, 1) * 2, 64));
  return c;
}

int64_t rank_rows(const strom_isvd* h) { return h->n_global > 0 ? h->n_global : h->n; }
int64_t mem_rows(const strom_isvd* h) {
  if (!h->shard) return h->n;
  return round_up(ceil_div(rank_rows(h), h->shard->world), 128);
}

std::shared_ptr<Store> alloc_store(int64_t n, int64_t ldu, int32_t ccap, cudaStream_t s) {
  auto st = std::make_shared<Store>();
  const size_t ubytes = (size_t)ldu * ccap * 8;
  if (ubytes >= kSpareStoreMin) {
    SpareStore& sp = spare_store();
    std::lock_guard<std::mutex> g(sp.mu);
    DevMemPtr& slot = sp.mem[current_device_id()];
    if (slot && slot->bytes == ubytes && slot->stream == s) st->umem = std::move(slot);
    else slot.reset();  // another shape or stream: do not sit on the memory
  }
  if (!st->umem) st->umem = dev_alloc(ubytes, s, false);
  if (ubytes >= kSpareStoreMin) {
    // The first store of this size: reserve its compaction partner now (make_caps sized the
    // store so that two fit) -- a fresh allocation of tens of GB costs the driver 0.4 - 4 s,
    // which would otherwise land on the first compaction in the middle of the stream.
    SpareStore& sp = spare_store();
    std::lock_guard<std::mutex> g(sp.mu);
    DevMemPtr& slot = sp.mem[current_device_id()];
    if (!slot && sp.live[current_device_id()] == 1) {
      try {
        slot = dev_alloc(ubytes, s, false);
      } catch (const Error&) {
        (void)cudaGetLastError();  // no room for it now: the compaction will ask again
      }
    }
  }
  // tiles holding padding rows (>= n) are read by the passes: keep them zero (never NaN)
  const int64_t first_pad_tile = n / kUTile;
  const int64_t ntile = ldu / kUTile;
  if (first_pad_tile < ntile)
    STROM_CUDA(cudaMemsetAsync(st->umem->as<double>() + first_pad_tile * kUTile * ccap, 0,
                               (size_t)(ntile - first_pad_tile) * kUTile * ccap * 8, s));
  st->lmem = dev_alloc((size_t)2 * ccap * ccap * 8, s, true);
  st->ldu = ldu;
  st->ccap = ccap;
  return st;
}

void set_store(strom_isvd* h, const std::shared_ptr<Store>& st) {
  h->store = st;
  h->view.L = st->L();
  h->view.Li = st->Li();
  h->view.ldl = st->ccap;
}

// copy-on-write: a private store holding the first c_ub physical columns
std::shared_ptr<Store> clone_store(const Store& src, int64_t n, int32_t c_ub, cudaStream_t s) {
  auto st = alloc_store(n, src.ldu, src.ccap, s);
  if (c_ub > 0)  // the first c_ub column segments of every tile
    STROM_CUDA(cudaMemcpy2DAsync(st->U(), (size_t)kUTile * src.ccap * 8, src.U(), (size_t)kUTile * src.ccap * 8,
                                 (size_t)kUTile * c_ub * 8, src.ldu / kUTile, cudaMemcpyDeviceToDevice, s));
  STROM_CUDA(cudaMemcpyAsync(st->L(), src.L(), (size_t)2 * src.ccap * src.ccap * 8, cudaMemcpyDeviceToDevice, s));
  st->claimed = c_ub;
  return st;
}

void alloc_small(strom_isvd* h, cudaStream_t s) {
  const Caps& c = h->caps;
  const size_t wsz = (size_t)c.ccap * (c.rcap + 1);
  const size_t ssz = (size_t)c.rcap + 2;
  const size_t bytes = 256 + 8 * (wsz + ssz);
  h->small = dev_alloc(bytes, s, true);
  char* p = h->small->as<char>();
  h->view.hdr = reinterpret_cast<IsvdHdr*>(p);
  h->view.N = reinterpret_cast<double*>(p + 256);
  h->view.sigma = h->view.N + wsz;
  h->view.ldn = c.ccap;
}

void alloc_v(strom_isvd* h, cudaStream_t s) {
  h->vmem = dev_alloc((size_t)h->caps.kcap * (h->caps.rcap + 1) * 8, s, false);
  h->view.V = h->vmem->as<double>();
  h->view.ldv = h->caps.kcap;
}

strom_isvd* new_like(const strom_isvd* src, const Caps& caps) {
  auto* h = new strom_isvd();
  h->n = src->n;
  h->n_global = src->n_global;
  h->shard = src->shard;
  h->ldu = src->ldu;
  h->k = src->k;
  h->tol_svd = src->tol_svd;
  h->tol_sv = src->tol_sv;
  h->r_max = src->r_max;
  h->cap_mode = src->cap_mode;
  h->caps = caps;
  return h;
}

// ------------------------------------------------------------------ pipeline scratch
struct PipeMem {
  DevMemPtr mem;
  Pipe pp{};
  int32_t ccap = 0, rcap = 0;
  int pstride = 0, work_stride = 0, max_grid = 0;
  // window mode: projections G (ldg x kWB), their Gram XX (kWB x kWB), the
  // window pass's per-CTA partials, and a second V_bar (parity-buffered: the
  // V update trails on its own stream)
  double* wG = nullptr;
  double* wXX = nullptr;
  double* wpart = nullptr;
  double* vbar2 = nullptr;
  int ldg = 0, wpstride = 0;
};

PipeMem make_pipe(const Caps& c, cudaStream_t s) {
  PipeMem m;
  m.ccap = c.ccap;
  m.rcap = c.rcap;
  m.max_grid = sm_count() * 8;
  m.pstride = (int)(2 * round_up(c.ccap + 1, 4) + 16);
  const int64_t rc2 = c.rcap + 2;
  m.work_stride = (int)round_up(std::max<int64_t>(c.ccap, rc2), 32);
  const size_t work_elems = 4 * (size_t)m.work_stride + 3 * rc2 * rc2 + 16 * (size_t)m.work_stride +
                            (size_t)c.ccap * rc2;  // step B's layout (global fallback)
  const size_t nv = round_up(c.ccap + 2, 4), nell = round_up(rc2, 4);
  const size_t n_part = (size_t)m.max_grid * m.pstride;
  m.ldg = (int)round_up(c.ccap + 1, 8);
  m.wpstride = (int)(round_up(c.ccap, 8) * kWB + kWB * kWB);
  const size_t n_win = (size_t)m.ldg * kWB + kWB * kWB + (size_t)m.max_grid * m.wpstride + rc2 * rc2;
  size_t total = 2 * nell + 2 * nv + 7 * nv + 2 * (2 * nv + 8 + kWB) + rc2 * rc2 + work_elems + (size_t)c.ccap * rc2 + n_part +
                 n_win;
  total = round_up(total, 32);
  const size_t bytes = total * 8 + 512;
  m.mem = dev_alloc(bytes, s, true);
  double* p = m.mem->as<double>();
  for (int i = 0; i < 2; ++i) { m.pp.ell[i] = p; p += nell; }
  for (int i = 0; i < 2; ++i) { m.pp.nj[i] = p; p += nv; }
  m.pp.tvec = p; p += nv;
  m.pp.gt = p; p += nv;
  m.pp.y = p; p += nv;
  m.pp.l1 = p; p += nv;
  m.pp.h = p; p += nv;
  m.pp.tmp = p; p += nv;
  m.pp.w = p; p += nv;
  m.pp.fo.e = p; p += nv;
  m.pp.fo.gn = p; p += nv;
  m.pp.fo.scal = p; p += 8;
  m.pp.fo.gw = p; p += kWB;
  m.pp.ro.e = p; p += nv;
  m.pp.ro.gn = p; p += nv;
  m.pp.ro.scal = p; p += 8;
  m.pp.ro.gw = p; p += kWB;
  m.pp.vbar = p; p += rc2 * rc2;
  m.pp.work = p; p += work_elems;
  m.pp.T = p; p += (size_t)c.ccap * rc2;
  m.pp.part = p; p += n_part;
  m.wG = p; p += (size_t)m.ldg * kWB;
  m.wXX = p; p += kWB * kWB;
  m.wpart = p; p += (size_t)m.max_grid * m.wpstride;
  m.vbar2 = p; p += rc2 * rc2;
  char* q = m.mem->as<char>() + total * 8;
  m.pp.ctl = reinterpret_cast<PipeCtl*>(q);
  m.pp.step[0] = reinterpret_cast<IsvdStep*>(q + 64);
  m.pp.step[1] = reinterpret_cast<IsvdStep*>(q + 192);
  m.pp.counter = reinterpret_cast<unsigned*>(q + 384);
  m.pp.vrec[0] = reinterpret_cast<VRec*>(q + 416);
  m.pp.vrec[1] = reinterpret_cast<VRec*>(q + 448);
  return m;
}

IsvdParams make_params(const strom_isvd* h, const PipeMem& m, int64_t k_new, bool init_call) {
  IsvdParams P;
  P.n = h->n_global > 0 ? h->n_global : h->n;  // decisions compare ranks with the GLOBAL row count
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
  P.parity = 0;
  P.has_next = 0;
  P.b_expect = -1;
  P.d_expect = -1;
  P.L = h->store->L();
  P.Li = h->store->Li();
  P.prof = prof_dev_bytes();
  P.tprobe = g_tprobe;
  P.trace = nullptr;
  P.wG = nullptr;
  P.wXX = nullptr;
  P.ldg = 0;
  P.wcol = 0;
  P.wn = 0;
  P.inline_next = 0;
  P.stage_doubles = 0;
  P.step_try = 0;
  P.step_smem_doubles = 0;
  return P;
}

// ------------------------------------------------------------------ launchers
// Raise a kernel's dynamic shared-memory cap whenever a launch asks for more
// than any earlier one.  ONE record per (device, kernel): two launchers of the
// same kernel with caches of their own would lower each other's setting.
std::mutex g_smem_mu;
std::map<std::pair<int, const void*>, size_t> g_smem_attr;
template <class K>
void set_smem_attr(K kernel, size_t smem, size_t* /*legacy per-call-site cache, unused*/ = nullptr) {
  if (smem <= 32 * 1024) return;
  std::lock_guard<std::mutex> g(g_smem_mu);
  size_t& cur = g_smem_attr[{current_device_id(), reinterpret_cast<const void*>(kernel)}];
  if (smem > cur) {
    STROM_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cur = smem;
  }
}

// ------------------------------------------------------------------ shard exchange kernels
// Each mirrors the reduction it follows: the same skip conditions and output
// ranges, read from the same device control block, so every rank exchanges (or
// skips) alike without a host decision.
__global__ void __launch_bounds__(kShardThreads) k_shard_pass(ShardDev sd, PassOut out, const PipeCtl* ctl, int kind,
                                                              int has_x, int has_xn, int nxw_arg, int phase) {
  pdl_enter();
  int c = ctl->c;
  bool do_e = false, do_gn = false, have_x = has_x != 0;
  if (kind == PASS_SECOND) {
    const int ro = ctl->reorth;
    if (ro == 0) return;
    have_x = true;
    if (ro == 1) do_e = true;
    else c = 0;
  } else if (kind == PASS_FUSED || kind == PASS_RESID) {
    if (kind == PASS_RESID && *(volatile const int32_t*)&ctl->resid == 0) return;
    do_e = true;
    do_gn = has_xn != 0;
  } else {
    have_x = false;
    do_gn = true;
  }
  ShardSegs sg;
  sg.n = 4;
  sg.s[0] = ShardSeg{out.e, do_e ? c : 0, 1, 0};
  sg.s[1] = ShardSeg{out.gn, do_gn ? c : 0, 1, 0};
  sg.s[2] = ShardSeg{out.scal, 3, 1, 0};
  sg.s[3] = ShardSeg{out.gw, have_x ? nxw_arg : 0, 1, 0};
  shard_exchange(sd, sg, phase);
  __syncthreads();
  if (phase != SHARD_PUBLISH && kind == PASS_FUSED && do_gn && threadIdx.x == 0)
    out.gn[c] = out.scal[2];  // r . x_next, as the pass's own reduction stores it
}

__global__ void __launch_bounds__(kShardThreads) k_shard_window(ShardDev sd, const PipeCtl* ctl, int nw, double* G,
                                                                int ldg, double* XX, int phase) {
  pdl_enter();
  ShardSegs sg;
  sg.n = 2;
  sg.s[0] = ShardSeg{G, ctl->c, nw, ldg};
  sg.s[1] = ShardSeg{XX, kWB * kWB, 1, 0};
  shard_exchange(sd, sg, phase);
}

__global__ void __launch_bounds__(kShardThreads) k_shard_gram(ShardDev sd, const int32_t* q_dev, int q_fixed,
                                                              double* G, int ld, int phase) {
  const int q = q_dev ? *q_dev : q_fixed;
  ShardSegs sg;
  sg.n = 1;
  sg.s[0] = ShardSeg{G, q, q, ld};
  shard_exchange(sd, sg, phase);
}

// Launch one exchange: a single kernel over peer memory, or -- in a
// single-process group -- publish, a host rendezvous that orders the ranks'
// streams by events, then combine.
template <class LaunchFn>
void shard_run(ShardImpl* g, cudaStream_t s, LaunchFn&& launch) {
  if (!g->lsync) {
    launch(SHARD_BOTH);
    return;
  }
  launch(SHARD_PUBLISH);
  LocalSync& ls = *g->lsync;
  const int slot = (int)(g->nsync++ % LocalSync::kRing);
  STROM_CUDA(cudaEventRecord(ls.ev[g->rank][slot], s));
  ls.barrier();  // every rank has recorded its publish
  for (int p = 0; p < g->world; ++p)
    if (p != g->rank) STROM_CUDA(cudaStreamWaitEvent(s, ls.ev[p][slot], 0));
  ls.barrier();  // every rank has queued its waits: the events may be re-recorded
  launch(SHARD_COMBINE);
}

void shard_after_pass(const strom_isvd* h, const PassArgs& a, cudaStream_t s) {
  if (!h->shard) return;
  ShardImpl* g = h->shard.get();
  shard_run(g, s, [&](int phase) {
    launch_pdl(k_shard_pass, dim3(1), dim3(kShardThreads), 0, s, g->dev, a.out, (const PipeCtl*)a.ctl, (int)a.kind,
               a.x ? 1 : 0, a.xn ? 1 : 0, (int)a.nxw, phase);
    STROM_LAUNCH_CHECK();
  });
}

void shard_after_gram(const std::shared_ptr<ShardImpl>& sh, const int32_t* q_dev, int q_fixed, double* G, int ld,
                      cudaStream_t s) {
  if (!sh) return;
  ShardImpl* g = sh.get();
  shard_run(g, s, [&](int phase) {
    k_shard_gram<<<1, kShardThreads, 0, s>>>(g->dev, q_dev, q_fixed, G, ld, phase);
    STROM_LAUNCH_CHECK();
  });
}

inline int pass_maxj(int cols) {
  const int need = (cols + kPassConsumers - 1) / kPassConsumers;
  if (need <= 1) return 1;
  if (need <= 2) return 2;
  if (need <= 4) return 4;
  if (need <= 8) return 8;
  if (need <= 12) return 12;
  if (need <= 16) return 16;
  if (need <= 18) return 18;  // c <= 144: cfg5's store (c_cap 139) without the 24-column variant's spills
  if (need <= 24) return 24;
  return 32;
}

// pipeline depth: stages of kStageRows x cols within ~140 KB (2 .. kPassMaxStages)
size_t pass_stage_budget() {
  static size_t v = [] {
    const char* e = getenv("STROM_STAGE_KB");
    const int kb = e ? atoi(e) : 140;
    return (size_t)std::max(16, std::min(212, kb)) * 1024;
  }();
  return v;
}
inline int pass_stages(int cols) {
  const size_t per = (size_t)kStageRows * (std::max(cols, 1) + 2 + (kWB - 1)) * 8;
  return (int)std::max<size_t>(2, std::min<size_t>(kPassMaxStages, pass_stage_budget() / per));
}

template <int MAXJ>
void launch_pass_t(const PassArgs& a, int cols_ub, int reserve, int kind_prof, cudaStream_t s) {
  const int cols = std::max(cols_ub, 1);
  const int nst = pass_stages(cols);
  // stages (+ x and x_next segments); the decision tail reuses them as its workspace
  const size_t smem = std::max((size_t)nst * kStageRows * (cols + 2 + (kWB - 1)) * 8,
                               (size_t)2 * (kPassThreads / 32) * round_up(a.ccap, 32) * 8);
  static PerDevice<size_t> cfg;
  set_smem_attr(k_pass<MAXJ>, smem, &cfg.get());
  const int64_t ntiles = a.ldu / kStageRows;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, std::max(1, sm_count() - reserve)));
  ProfScope ps(kind_prof, s);
  launch_pdl(k_pass<MAXJ>, dim3(grid), dim3(kPassThreads), smem, s, a, nst);
  {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, k_pass<MAXJ>);
      char buf[256];
      snprintf(buf, sizeof buf, "k_pass<%d> launch (grid %d, smem %zu + static %zu, max dyn %d, regs %d, stages %d): %s",
               MAXJ, grid, smem, (size_t)fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes, fa.numRegs, nst,
               cudaGetErrorString(e));
      throw Error(kCudaError, buf);
    }
  }
}

// kind PASS_*; cols_ub bounds the U columns the pass may read.  tail: the
// decision run by the last CTA (1 decide after FUSED, 2 decide2 after SECOND)
struct PassTail {
  int32_t tail = 0, b_expect = -1;
  const StateView* src = nullptr;
  const IsvdParams* P = nullptr;
};

void launch_pass(int kind, int cols_ub, const strom_isvd* h, const PipeMem& m, const double* x, const double* xn,
                 int reserve, cudaStream_t s, const PassTail& tl = PassTail(), const double* const* xw = nullptr,
                 int nxw = 0) {
  PassArgs a;
  a.nxw = nxw;
  for (int j = 0; j < kWB - 1; ++j) a.xw[j] = j < nxw ? xw[j] : nullptr;
  a.U = h->store->U();
  a.ldu = h->ldu;
  a.n = h->n;
  a.ccap = h->store->ccap;
  {
    static const int dbg = [] {
      const char* e = getenv("STROM_PASS_DBG");
      return e ? atoi(e) : 0;
    }();
    a.dbg = dbg;
  }
  auto bulk_ok = [&](const double* v) {
    return v && (reinterpret_cast<uintptr_t>(v) % 16 == 0) && (h->n % 2 == 0);
  };
  a.x_bulk = bulk_ok(x) ? 1 : 0;
  a.xn_bulk = bulk_ok(xn) ? 1 : 0;
  static const bool xw_stage = [] {
    const char* e = getenv("STROM_XW_STAGE");
    return !(e && atoi(e) == 0);
  }();
  a.xw_bulk = xw_stage ? 1 : 0;
  for (int j = 0; j < nxw; ++j)
    if (!bulk_ok(xw[j])) a.xw_bulk = 0;
  a.ctl = m.pp.ctl;
  a.kind = kind;
  a.pstride = m.pstride;
  a.pld = m.max_grid;
  a.x = x;
  a.coef = (kind == PASS_FUSED || kind == PASS_RESID) ? m.pp.gt : (kind == PASS_SECOND ? m.pp.h : nullptr);
  a.xn = xn;
  a.out = (kind == PASS_SECOND) ? m.pp.ro : m.pp.fo;
  a.part = m.pp.part;
  a.counter = m.pp.counter;
  a.prof = prof_dev_bytes();
  a.trace = g_cur_trace;
  a.tail = tl.tail;
  a.b_expect = tl.b_expect;
  a.dpp = m.pp;
  if (tl.src) a.dsrc = *tl.src;
  if (tl.P) a.dP = *tl.P;
  const int pk = (kind == PASS_SECOND) ? P_RESID : P_PROJ;
  const int cu = std::max(cols_ub, 1);
  switch (pass_maxj(cu)) {
    case 1: launch_pass_t<1>(a, cu, reserve, pk, s); break;
    case 2: launch_pass_t<2>(a, cu, reserve, pk, s); break;
    case 4: launch_pass_t<4>(a, cu, reserve, pk, s); break;
    case 8: launch_pass_t<8>(a, cu, reserve, pk, s); break;
    case 12: launch_pass_t<12>(a, cu, reserve, pk, s); break;
    case 16: launch_pass_t<16>(a, cu, reserve, pk, s); break;
    case 18: launch_pass_t<18>(a, cu, reserve, pk, s); break;
    case 24: launch_pass_t<24>(a, cu, reserve, pk, s); break;
    default: launch_pass_t<32>(a, cu, reserve, pk, s); break;
  }
  if (h->shard) {
    if (tl.tail) throw Error(kInternal, "sharded passes take their decisions in their own kernels");
    shard_after_pass(h, a, s);
  }
}

size_t decide_smem(const PipeMem& m) { return (size_t)2 * (kDecideThreads / 32) * round_up(m.ccap, 32) * 8; }


void launch_prep(const PipeMem& m, const IsvdParams& P, cudaStream_t s) {
  static PerDevice<size_t> cfg;
  const size_t smem = decide_smem(m);
  set_smem_attr(k_prep, smem, &cfg.get());
  ProfScope ps(P_STEP_A, s);
  k_prep<<<1, kDecideThreads, smem, s>>>(m.pp, P);
  STROM_LAUNCH_CHECK();
}

void launch_decide_kernel(bool second, const StateView& src, const PipeMem& m, const IsvdParams& P,
                          cudaStream_t s) {
  static PerDevice<size_t> cfg1, cfg2;
  const size_t smem = decide_smem(m);
  ProfScope ps(P_STEP_A, s);
  if (!second) {
    set_smem_attr(k_decide, smem, &cfg1.get());
    launch_pdl(k_decide, dim3(1), dim3(kDecideThreads), smem, s, src, m.pp, P);
  } else {
    set_smem_attr(k_decide2, smem, &cfg2.get());
    launch_pdl(k_decide2, dim3(1), dim3(kDecideThreads), smem, s, src, m.pp, P);
  }
  STROM_LAUNCH_CHECK();
}

// The decisions as their own 512-thread kernels (default; measured faster than
// running them in the pass's last CTA, STROM_DECIDE_TAIL=1, at cfg2).
bool decide_as_kernel() {
  static const bool v = [] {
    const char* e = getenv("STROM_DECIDE_TAIL");
    return !(e && atoi(e) != 0);
  }();
  return v;
}

// r_ub >= 0: a bound on the state's current rank (the kernel lays its work area out by the
// current m = r + 1, not by the capacity: an uncapped state whose rank capacity has grown past
// what shared memory holds keeps the fast path while its rank still fits).
size_t small_kernel_smem(const Caps& c, int* use_smem, int r_ub = -1) {
  // step B layout: 3 m^2 + 16 ms (secular work) + ccap m (staged N_b / QR's M)
  const size_t m = (r_ub >= 0 ? std::min<int>(c.rcap, r_ub) : c.rcap) + 1;
  const size_t ms = round_up(std::max<int64_t>(c.ccap, c.rcap + 2), 32);
  const size_t need = (3 * m * m + 16 * ms + (size_t)c.ccap * m) * 8;
  const size_t limit = max_smem_optin() - 8 * 1024;
  *use_smem = need <= limit ? 1 : 0;
  return *use_smem ? need : 0;
}

// The core step.  Its work area (3 m^2 + 16 ms + ccap m doubles, m = r + 1) lives in shared
// memory when the layout of the rank CAPACITY fits, or of the host's rank bound; otherwise
// (an uncapped state whose capacity has grown) the shared-memory kernel is still tried with
// all the shared memory there is -- it decides on the device by the CURRENT rank -- with the
// global-memory kernel queued behind it as its fallback (IsvdParams::step_try).
void launch_step_b_pp(const StateView& src, const StateView& dst, const Pipe& pp, const IsvdParams& P,
                      const Caps& caps, cudaStream_t s, int r_ub = -1, int r_max = -1) {
  int fits_cap = 0, fits_ub = 0;
  size_t smem = small_kernel_smem(caps, &fits_cap);
  if (!fits_cap && r_ub >= 0) smem = small_kernel_smem(caps, &fits_ub, r_ub);
  ProfScope ps(P_STEP_B, s);
  if (fits_cap || fits_ub) {
    set_smem_attr(k_step_b<true>, smem);
    k_step_b<true><<<1, kSmallThreads, smem, s>>>(src, dst, pp, P);
  } else {
    int fits_rmax = 1;
    if (r_max >= 0) small_kernel_smem(caps, &fits_rmax, r_max);  // a capped stream sits at its cap
    if (fits_rmax) {
      const size_t room = max_smem_optin() - 8 * 1024;
      IsvdParams Pt = P;
      Pt.step_try = 1;
      Pt.step_smem_doubles = (int32_t)(room / 8);
      set_smem_attr(k_step_b<true>, room);
      k_step_b<true><<<1, kSmallThreads, room, s>>>(src, dst, pp, Pt);
      Pt.step_try = 2;
      k_step_b<false><<<1, kSmallThreads, 0, s>>>(src, dst, pp, Pt);
    } else {
      k_step_b<false><<<1, kSmallThreads, 0, s>>>(src, dst, pp, P);
    }
  }
  STROM_LAUNCH_CHECK();
}
void launch_step_b(const StateView& src, const StateView& dst, const PipeMem& m, const IsvdParams& P,
                   const Caps& caps, cudaStream_t s, int r_ub = -1, int r_max = -1) {
  launch_step_b_pp(src, dst, m.pp, P, caps, s, r_ub, r_max);
}

void launch_vupdate(const StateView& src, const StateView& dst, const PipeMem& m, const IsvdParams& P, int rcap,
                    cudaStream_t s) {
  dim3 grid((unsigned)ceil_div(P.k_new, kVRows), (unsigned)ceil_div(rcap + 1, kVCols));
  ProfScope ps(P_VUPDATE, s);
  k_vupdate<<<grid, kVRows, (size_t)(rcap + 2) * kVCols * 8, s>>>(src, dst, m.pp, P);
  STROM_LAUNCH_CHECK();
}

void launch_compact_prep(const StateView& src, const StateView& dst, const PipeMem& m, const IsvdParams& P,
                         const Caps& caps, cudaStream_t s) {
  int use_smem = 0;
  const size_t smem = small_kernel_smem(caps, &use_smem);
  static PerDevice<size_t> cfg;
  set_smem_attr(k_compact_prep, smem, &cfg.get());
  ProfScope ps(P_COMPACT, s);
  k_compact_prep<<<1, kSmallThreads, smem, s>>>(src, dst, m.pp, P, use_smem);
  STROM_LAUNCH_CHECK();
}

void launch_tall_gemm(const Tall& A, const int32_t* col0_dev, const double* T, int64_t ldt, const int32_t* p_dev,
                      const int32_t* q_dev, const Tall& out, bool row_major, int64_t n, int64_t nrows_pad,
                      cudaStream_t s) {
  const int64_t tiles = ceil_div(nrows_pad, kGemmRows);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sm_count() * 4));
  ProfScope ps(P_TALL_GEMM, s);
  k_tall_gemm<<<grid, 256, kGemmKc * 64 * 8, s>>>(A, col0_dev, 0, T, ldt, p_dev, q_dev, 0, out, row_major ? 1 : 0, n,
                                                  nrows_pad);
  STROM_LAUNCH_CHECK();
}

// Gram from per-CTA partials (QP x QP each, summed in CTA order) -> L = chol, Li = L^{-1}
void gram_finish(const double* part, int nparts, int QP, const int32_t* q_dev, int q_fixed, double* L, double* Li,
                 int ldl, const IsvdHdr* hdr_c, int* status_dev, cudaStream_t s,
                 const std::shared_ptr<ShardImpl>& shard) {
  k_gram_reduce<<<(unsigned)ceil_div((int64_t)QP * QP, 256), 256, 0, s>>>(part, nparts, QP, q_dev, q_fixed, L, ldl);
  STROM_LAUNCH_CHECK();
  shard_after_gram(shard, q_dev, q_fixed, L, ldl, s);  // row-sharded: the Gram of all ranks' rows
  k_cholesky<<<1, 256, 0, s>>>(L, ldl, hdr_c, q_fixed, status_dev);
  STROM_LAUNCH_CHECK();
  k_lower_inverse<<<1, 1024, 0, s>>>(L, ldl, hdr_c, q_fixed, Li);
  STROM_LAUNCH_CHECK();
}

// Shared memory of the fused compaction sweep handling `tr` rows of a tile per step.
size_t compact_pass_smem(int cmax, int rmax, int tr) {
  const int c4 = (cmax + 3) & ~3, RP = (rmax + 31) & ~31;
  return ((size_t)c4 * (RP + 4) + (size_t)c4 * (tr + 4) + (size_t)RP * (tr + 4)) * 8;
}
// 64 (whole tiles), 32 (half tiles) or 0 (does not fit: the unfused GEMM + Gram)
int compact_pass_rows(int cmax, int rmax) {
  if (rmax > 128) return 0;
  for (int tr : {64, 32})
    if (compact_pass_smem(cmax, rmax, tr) <= max_smem_optin()) return tr;
  return 0;
}

template <int GB, int TR>
int launch_compact_pass_t(const Store& src, const int32_t* base_dev, const int32_t* c_dev, const int32_t* r_dev,
                          const double* T, int64_t ldt, int cmax, int rmax, const Store& dst, double* part, int QP,
                          cudaStream_t s) {
  const size_t smem = compact_pass_smem(cmax, rmax, TR);
  static PerDevice<size_t> cfg;
  set_smem_attr(k_compact_pass<GB, TR>, smem, &cfg.get());
  ProfScope ps(P_TALL_GEMM, s);
  k_compact_pass<GB, TR><<<sm_count(), kCompactThreads, smem, s>>>(src.U(), src.ccap, base_dev, c_dev, r_dev, T, ldt,
                                                                   dst.U(), dst.ccap, src.ldu / kUTile, part, QP,
                                                                   prof_dev_bytes());
  STROM_LAUNCH_CHECK();
  return sm_count();  // per-CTA Gram partials written
}
// (Half tiles with two CTAs per SM at r <= 64 -- one loads while the other multiplies -- were
// tried: under a millisecond per cfg2 step, bought with a 128-register cap that slows the
// whole-tile sweep by 9 %, and the other split of the Gram partials only re-rolled the
// noise-level decisions: dropped.)
template <int GB>
int launch_compact_pass(const Store& src, const int32_t* base_dev, const int32_t* c_dev, const int32_t* r_dev,
                        const double* T, int64_t ldt, int cmax, int rmax, const Store& dst, double* part, int QP,
                        cudaStream_t s) {
  if (compact_pass_rows(cmax, rmax) == 64)
    return launch_compact_pass_t<GB, 64>(src, base_dev, c_dev, r_dev, T, ldt, cmax, rmax, dst, part, QP, s);
  if constexpr (GB >= 3)  // half tiles are only ever needed for 96- and 128-column Gram blocks
    return launch_compact_pass_t<GB, 32>(src, base_dev, c_dev, r_dev, T, ldt, cmax, rmax, dst, part, QP, s);
  throw Error(kInternal, "compaction sweep: no shared-memory layout");
}

// L = chol(A[:, col0:col0+q]^T A[:, col0:col0+q]) with the DMMA tall Gram.
// q is read on the device (q_dev) or fixed; the Cholesky reads c from hdr_c.
void gram_cholesky(const Tall& A, const int32_t* col0_dev, const int32_t* q_dev, int q_fixed,
                   int qmax, int64_t n, double* L, double* Li, int ldl, const IsvdHdr* hdr_c, int* status_dev,
                   cudaStream_t s, const std::shared_ptr<ShardImpl>& shard) {
  const int QP = (int)round_up(std::max(qmax, 1), 8);
  const int64_t ntiles = ceil_div(n, kGramRows);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)sm_count() * 2));
  auto part = dev_alloc((size_t)grid * QP * QP * 8, s, false);
  const size_t smem = (size_t)QP * kGramLd * 8;
  ProfScope ps(P_OTHER, s);
  if (QP <= 64) {
    k_tall_gram<1, 8><<<grid, 256, smem, s>>>(A, col0_dev, q_dev, q_fixed, n, part->as<double>(), QP);
  } else if (QP <= 128) {
    static PerDevice<bool> cfgs;
    bool& cfg = cfgs.get();
    if (!cfg) {
      STROM_CUDA(cudaFuncSetAttribute(k_tall_gram<2, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
      cfg = true;
    }
    k_tall_gram<2, 16><<<grid, 256, smem, s>>>(A, col0_dev, q_dev, q_fixed, n, part->as<double>(), QP);
  } else {
    throw Error(kInvalidArgument, "Gram of more than 128 columns is not supported");
  }
  STROM_LAUNCH_CHECK();
  gram_finish(part->as<double>(), grid, QP, q_dev, q_fixed, L, Li, ldl, hdr_c, status_dev, s, shard);
}

// Compaction into a fresh store (also used to grow capacities):
// U_new = U[:, base:base+c] L^{-T} Q_c, N_new = L_new^T R_c, L_new measured.
strom_isvd* compact(strom_isvd* src, const Caps& caps, cudaStream_t s) {
  strom_isvd* t = new_like(src, caps);
  std::unique_ptr<strom_isvd> guard(t);
  alloc_small(t, s);
  t->vmem = src->vmem;  // V is immutable: share it
  t->view.V = src->view.V;
  t->view.ldv = src->view.ldv;
  t->caps.kcap = src->caps.kcap;
  set_store(t, alloc_store(src->n, src->ldu, caps.ccap, s));
  Caps kc = caps;
  kc.ccap = std::max(caps.ccap, src->caps.ccap);
  kc.rcap = std::max(caps.rcap, src->caps.rcap);
  PipeMem m = make_pipe(kc, s);
  IsvdParams P = make_params(src, m, src->k, false);
  P.ccap = kc.ccap;
  launch_compact_prep(src->view, t->view, m, P, kc, s);
  // p = source c (step->m), q = r (step->mkeep); source columns start at base
  if (compact_pass_rows(src->caps.ccap, kc.rcap) > 0) {
    // one fused DMMA sweep: U_new = U T and the measured Gram of the stored U_new
    const int RP = (int)round_up(kc.rcap, 32);
    auto part = dev_alloc((size_t)2 * sm_count() * RP * RP * 8, s, false);  // up to two CTAs per SM
    int nparts = sm_count();
    const int nbg = (RP / 16) * (RP / 32);
    const int gb = (nbg + 7) / 8;
    const int32_t* bptr = &src->view.hdr->base;
    const int32_t* cptr = &m.pp.step[0]->m;
    const int32_t* rptr = &m.pp.step[0]->mkeep;
    const int cmax = src->caps.ccap;
    switch (gb) {
      case 1: nparts = launch_compact_pass<1>(*src->store, bptr, cptr, rptr, m.pp.T, P.ccap, cmax, kc.rcap, *t->store, part->as<double>(), RP, s); break;
      case 2: nparts = launch_compact_pass<2>(*src->store, bptr, cptr, rptr, m.pp.T, P.ccap, cmax, kc.rcap, *t->store, part->as<double>(), RP, s); break;
      case 3: nparts = launch_compact_pass<3>(*src->store, bptr, cptr, rptr, m.pp.T, P.ccap, cmax, kc.rcap, *t->store, part->as<double>(), RP, s); break;
      default: nparts = launch_compact_pass<4>(*src->store, bptr, cptr, rptr, m.pp.T, P.ccap, cmax, kc.rcap, *t->store, part->as<double>(), RP, s); break;
    }
    gram_finish(part->as<double>(), nparts, RP, rptr, 0, t->view.L, t->view.Li, t->view.ldl, t->view.hdr,
                &m.pp.step[0]->pad0, s, src->shard);
  } else {
    launch_tall_gemm(tall_tiled(src->store->U(), src->store->ccap), &src->view.hdr->base, m.pp.T, P.ccap,
                     &m.pp.step[0]->m, &m.pp.step[0]->mkeep, tall_tiled(t->store->U(), t->store->ccap), false, t->n,
                     t->ldu, s);
    // measure the Gram of the stored U_new: L describes the memory, not an assumed identity
    gram_cholesky(tall_tiled(t->store->U(), t->store->ccap), nullptr, &m.pp.step[0]->mkeep, 0, caps.rcap, t->n,
                  t->view.L, t->view.Li, t->view.ldl, t->view.hdr, &m.pp.step[0]->pad0, s, src->shard);
  }
  k_compact_finish<<<1, 256, 0, s>>>(t->view, m.pp.T, P.ccap);
  STROM_LAUNCH_CHECK();
  t->r_ub = std::min(src->r_ub, caps.rcap);
  t->c_ub = t->r_ub;
  t->store->claimed = t->c_ub;
  return guard.release();
}

// Sticky exchange errors of a shard group (the caller has synchronised).
void shard_check(ShardImpl* g) {
  int32_t err = 0;
  STROM_CUDA(cudaMemcpy(&err, g->dev.err, sizeof(err), cudaMemcpyDeviceToHost));
  if (err == SHARD_ERR_TIMEOUT)
    throw Error(kCudaError, "shard exchange timed out waiting for a peer rank (results are invalid)");
  if (err) throw Error(kInternal, "shard exchange: vector larger than the mailbox");
}

void read_hdr(const strom_isvd* h, cudaStream_t s, IsvdHdr* out) {
  STROM_CUDA(cudaMemcpyAsync(out, h->view.hdr, sizeof(IsvdHdr), cudaMemcpyDeviceToHost, s));
  STROM_CUDA(cudaStreamSynchronize(s));
}

// Capacity management before an update of `cur` (host side; synchronises only
// when a bound says it might be needed).  Returns the state to update from
// (cur itself, or a compacted copy owned by *hold).
strom_isvd* ensure_capacity(strom_isvd* cur, std::unique_ptr<strom_isvd>* hold, cudaStream_t s) {
  if (cur->r_max < 0 && cur->r_ub + 1 > cur->caps.rcap && cur->caps.rcap < rank_rows(cur)) {
    IsvdHdr hh;
    read_hdr(cur, s, &hh);
    cur->r_ub = hh.r;
    cur->c_ub = std::min(cur->c_ub, hh.base + hh.c);
    if (hh.r + 1 > cur->caps.rcap) {
      Caps nc = make_caps(rank_rows(cur), -1, std::min<int64_t>(rank_rows(cur), 2 * (int64_t)cur->caps.rcap),
                          cur->k, mem_rows(cur));
      nc.kcap = cur->caps.kcap;
      hold->reset(compact(cur, nc, s));
      cur = hold->get();
    }
  }
  if (cur->c_ub + 1 > cur->caps.ccap) {
    IsvdHdr hh;
    read_hdr(cur, s, &hh);  // refine the bound: dependent updates did not append
    cur->c_ub = hh.base + hh.c;
    cur->r_ub = hh.r;
    if (cur->c_ub + 1 > cur->caps.ccap) {
      hold->reset(compact(cur, cur->caps, s));
      cur = hold->get();
    }
  }
  return cur;
}

// The store a successor of `cur` may append to (shared, or a private copy).
std::shared_ptr<Store> successor_store(const strom_isvd* cur, cudaStream_t s) {
  if (cur->store->claimed != cur->c_ub) return clone_store(*cur->store, cur->n, cur->c_ub, s);
  return cur->store;
}

// One functional update cur -> new state (all device-side decisions), on one stream.
strom_isvd* update_once(strom_isvd* src, const double* x, cudaStream_t s, bool init_call = false) {
  std::unique_ptr<strom_isvd> hold;
  strom_isvd* cur = ensure_capacity(src, &hold, s);
  Caps nc = cur->caps;
  if (cur->k + 1 > nc.kcap) nc.kcap = round_up((cur->k + 1) * 2, 64);
  strom_isvd* dst = new_like(cur, nc);
  std::unique_ptr<strom_isvd> dguard(dst);
  dst->k = cur->k + 1;
  alloc_small(dst, s);
  alloc_v(dst, s);
  set_store(dst, successor_store(cur, s));
  PipeMem m = make_pipe(cur->caps, s);
  IsvdParams P = make_params(dst, m, dst->k, init_call);
  const int cols = cur->c_ub;
  k_init_ctl<<<1, 1, 0, s>>>(m.pp.ctl, cur->view.hdr);
  STROM_LAUNCH_CHECK();
  launch_pass(PASS_PROJ, cols, dst, m, nullptr, x, 0, s);
  trace_point("proj", s);
  launch_prep(m, P, s);
  trace_point("prep", s);
  if (cur->shard) {
    // row-sharded: the partial sums cross the ranks between a pass and its decision
    launch_pass(PASS_FUSED, cols, dst, m, x, nullptr, 0, s);
    launch_decide_kernel(false, cur->view, m, P, s);
    launch_pass(PASS_SECOND, cols, dst, m, x, nullptr, 0, s);
    launch_decide_kernel(true, cur->view, m, P, s);
  } else {
    PassTail tl;
    tl.tail = 1;  // decide (basis.py:112-139) in the pass's last CTA
    tl.src = &cur->view;
    tl.P = &P;
    launch_pass(PASS_FUSED, cols, dst, m, x, nullptr, 0, s, tl);
    trace_point("fused+decide", s);
    tl.tail = 2;  // re-orthogonalisation / restart copy, only when requested
    launch_pass(PASS_SECOND, cols, dst, m, x, nullptr, 0, s, tl);
    trace_point("second+decide2", s);
  }
  launch_step_b(cur->view, dst->view, m, P, cur->caps, s, cur->r_ub, cur->r_max);
  trace_point("step_b", s);
  launch_vupdate(cur->view, dst->view, m, P, cur->caps.rcap, s);
  trace_point("vupdate", s);
  dst->c_ub = cur->c_ub + 1;
  dst->store->claimed = std::max(dst->store->claimed, dst->c_ub);
  dst->r_ub = std::min(cur->r_ub + 1, cur->caps.rcap);
  return dguard.release();
}

// ------------------------------------------------------------------ window-mode launchers

// Measured: spinning k_decide_a on the core step's counter (STROM_DECIDE_SPIN=1)
// is slower than the cross-stream event -- the spinner and the core step it
// waits for hold SMs the V update and the passes then queue behind.
// Window or per-snapshot pipeline for one ingest call.  A window pass costs
// ~(c + kWB) / kWB column reads per snapshot and saves a full pass for every
// dependent snapshot; with every update independent -- cfg5's rank-100
// stream, whose residuals sit above tol -- the fused per-snapshot pass is
// cheaper.  The choice uses the source state's own counters (one header read
// per call); STROM_WINDOW forces a width.
int choose_window(const strom_isvd* src, cudaStream_t s) {
  static const int forced = [] {
    const char* e = getenv("STROM_WINDOW");
    return e ? std::max(0, std::min(kWB, atoi(e))) : -1;
  }();
  if (forced >= 0) return forced;
  if (src->k < 16) return kWB;
  IsvdHdr hh;
  read_hdr(src, s, &hh);
  // the per-snapshot pipeline only for a stream that has sat at its rank cap
  // (>= 64 truncations) without a single dependent update: every snapshot
  // would need its residual pass anyway.  (A cumulative dependent fraction
  // misleads: the rank build-up phase is all independent.)
  return (hh.n_dependent == 0 && hh.n_truncated >= 64) ? 1 : kWB;
}

// STROM_INLINE_DECIDE=0: k_decide_a always runs the first half itself
bool inline_decide() {
  static const bool v = [] {
    const char* e = getenv("STROM_INLINE_DECIDE");
    return !(e && atoi(e) == 0);
  }();
  return v;
}

bool decide_spins() {
  static const bool v = [] {
    const char* e = getenv("STROM_DECIDE_SPIN");
    return e && atoi(e) != 0;
  }();
  return v;
}

size_t wproj_stage_bytes(int c) { return wproj_stage_elems(std::max(c, 1)) * 8; }

template <int MT>
void launch_wproj_t(const WprojArgs& a, int cols_ub, cudaStream_t s) {
  const size_t per = wproj_stage_bytes(cols_ub);
  const size_t budget = max_smem_optin() - 24 * 1024;  // the static half-sum buffer
  const int nst = (int)std::max<size_t>(1, std::min<size_t>(kWMaxStages, std::min<size_t>(3, budget / per)));
  const size_t smem = (size_t)nst * per;
  static PerDevice<size_t> cfg;
  if (smem > cfg.get()) {
    STROM_CUDA(cudaFuncSetAttribute(k_wproj<MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cfg.get() = smem;
  }
  const int64_t ntiles = a.ldu / kStageRows;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, std::max(1, sm_count() - 1)));
  ProfScope ps(P_WPROJ, s);
  launch_pdl(k_wproj<MT>, dim3(grid), dim3(kWThreads), smem, s, a, nst);
  STROM_LAUNCH_CHECK();
}

// G = U^T [x_w0 .. x_w0+nw-1], XX = their Gram; then the coefficients of the
// window's first snapshot (k_prep_w).  cols_ub bounds the live U columns.
void launch_window(const strom_isvd* h, const PipeMem& m, const double* const* xs, int nw, int cols_ub,
                   const IsvdParams& P0, cudaStream_t s) {
  WprojArgs a;
  a.U = h->store->U();
  a.ldu = h->ldu;
  a.n = h->n;
  a.ccap = h->store->ccap;
  a.ctl = m.pp.ctl;
  bool bulk = (h->n % 2 == 0);
  for (int j = 0; j < kWB; ++j) {
    a.xs[j] = j < nw ? xs[j] : nullptr;
    if (j < nw && reinterpret_cast<uintptr_t>(xs[j]) % 16 != 0) bulk = false;
  }
  a.nw = nw;
  a.xbulk = bulk ? 1 : 0;
  a.part = m.wpart;
  a.pstride = m.wpstride;
  a.prof = prof_dev_bytes();
  a.trace = g_cur_trace;
  const int cu = std::max(cols_ub, 1);
  const int mt = (int)ceil_div(ceil_div(cu, 8), kWGroups);
  switch (mt) {
    case 1: launch_wproj_t<1>(a, cu, s); break;
    case 2: launch_wproj_t<2>(a, cu, s); break;
    case 3: launch_wproj_t<3>(a, cu, s); break;
    default: launch_wproj_t<4>(a, cu, s); break;
  }
  const int64_t ntiles = h->ldu / kStageRows;
  const int nparts = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, std::max(1, sm_count() - 1)));
  const int nout = (int)(round_up(cu, 8) * kWB + kWB * kWB);
  launch_pdl(k_wreduce, dim3((unsigned)ceil_div(nout, 32)), dim3(256), 0, s, (const double*)m.wpart, nparts,
             m.wpstride, (const PipeCtl*)m.pp.ctl, nw, m.wG, m.ldg, m.wXX);
  STROM_LAUNCH_CHECK();
  if (h->shard) {
    ShardImpl* g = h->shard.get();
    shard_run(g, s, [&](int phase) {
      launch_pdl(k_shard_window, dim3(1), dim3(kShardThreads), 0, s, g->dev, (const PipeCtl*)m.pp.ctl, nw, m.wG,
                 m.ldg, m.wXX, phase);
      STROM_LAUNCH_CHECK();
    });
  }
  IsvdParams P = P0;
  P.wG = m.wG;
  P.wXX = m.wXX;
  P.ldg = m.ldg;
  P.wn = nw;
  P.wcol = -1;  // "next" = column 0
  P.has_next = 1;
  Pipe pp = m.pp;
  pp.fo.gn = m.wG;
  static PerDevice<size_t> cfg;
  const size_t smem = decide_smem(m);
  set_smem_attr(k_prep_w, smem, &cfg.get());
  ProfScope ps(P_STEP_A, s);
  launch_pdl(k_prep_w, dim3(1), dim3(kDecideThreads), smem, s, pp, P);
  STROM_LAUNCH_CHECK();
}

void launch_decide_w(int which, const StateView& src, const Pipe& pp, const PipeMem& m, const IsvdParams& P,
                     cudaStream_t s) {
  static PerDevice<size_t> cfga, cfgb, cfg2;
  const size_t smem = decide_smem(m);
  ProfScope ps(P_STEP_A, s);
  if (which == 0) {
    set_smem_attr(k_decide_a, smem, &cfga.get());
    launch_pdl(k_decide_a, dim3(1), dim3(kDecideThreads), smem, s, src, pp, P);
  } else if (which == 1) {
    // room for the live block of L^{-1} and for N (decide_b_body stages them when they fit)
    const size_t want = (size_t)m.ccap * (m.ccap + m.rcap + 1) * 8;
    const size_t lim = max_smem_optin() - 4 * 1024;
    IsvdParams Pb = P;
    Pb.stage_doubles = (smem + want <= lim) ? (int32_t)(want / 8) : 0;
    const size_t smem_b = smem + (size_t)Pb.stage_doubles * 8;
    set_smem_attr(k_decide_b, smem_b, &cfgb.get());
    launch_pdl(k_decide_b, dim3(1), dim3(kDecideThreads), smem_b, s, src, pp, Pb);
  } else {
    set_smem_attr(k_decide2, smem, &cfg2.get());
    launch_pdl(k_decide2, dim3(1), dim3(kDecideThreads), smem, s, src, pp, P);
  }
  STROM_LAUNCH_CHECK();
}

void launch_vupdate_pp(const StateView& src, const StateView& dst, const Pipe& pp, const IsvdParams& P, int rcap,
                       cudaStream_t s) {
  dim3 grid((unsigned)ceil_div(P.k_new, kVRows), (unsigned)ceil_div(rcap + 1, kVCols));
  ProfScope ps(P_VUPDATE, s);
  k_vupdate<<<grid, kVRows, (size_t)(rcap + 2) * kVCols * 8, s>>>(src, dst, pp, P);
  STROM_LAUNCH_CHECK();
}

// ------------------------------------------------------------------ ingestion
// Columns of an ingest call: device pointers, or host columns staged through a
// ring of device chunks on a copy stream.  Chunks grow 1, 2, 4, 4, ... columns,
// so the first update waits for one column's copy, not a full chunk.
//
// Pageable host columns (a plain numpy array, what the reference's callers
// pass: pipeline.py:95-111) cannot be DMA'd asynchronously.  A stager thread
// copies each chunk into a recycled pinned buffer (parallel_memcpy) and issues
// its H2D copy itself, so the host copy of chunk q+1 overlaps the DMA of chunk
// q and the updates; the compute thread only waits for a chunk it needs.
struct ColumnSource {
  const double* X = nullptr;
  int64_t ldx = 0, n = 0, ncols = 0;
  bool host = false, pageable = false;
  cudaStream_t s = nullptr, cs = nullptr;
  // largest chunk (ring slot capacity, columns) and ring depth; STROM_H2D_CHUNK /
  // STROM_H2D_RING override them for measurements
  // (cfg2 e2e, steady state: 4 x 4 columns 79.1 ms per 400 snapshots, 3 x 16
  // 80.3 ms; the device-resident path 76.5 ms)
  const int64_t kChunk = env_int("STROM_H2D_CHUNK", 4);
  // at least 2 slots: col(t + 1) is requested before release(t) issues the
  // next chunk, so one slot would hand out a column still being copied
  // (window mode reads kWB columns ahead: 6 slots keep the copies ahead of it)
  const int kRing = (int)std::max<int64_t>(2, env_int("STROM_H2D_RING", 6));
  static int64_t env_int(const char* name, int64_t dflt) {
    const char* e = getenv(name);
    return e && atoll(e) > 0 ? atoll(e) : dflt;
  }
  std::vector<DevMemPtr> ring;
  std::vector<cudaEvent_t> ready, freed, hdone;
  std::vector<void*> pinned;  // pageable mode: one staging buffer per slot
  std::vector<int64_t> start;  // chunk q holds columns [start[q], start[q+1])
  int64_t issued = 0, waited = -1;
  // pageable mode: the stager thread and its handshakes with the compute thread
  std::thread stager;
  std::mutex mu;
  std::condition_variable cv;
  int64_t staged = 0;    // chunks whose H2D copy (and ready event) the stager has enqueued
  int64_t released = 0;  // chunks whose freed event the compute thread has recorded
  bool abort = false;
  std::string stage_error;

  int64_t nchunks() const { return (int64_t)start.size() - 1; }
  int64_t chunk_of(int64_t t) const {
    return (int64_t)(std::upper_bound(start.begin(), start.end(), t) - start.begin()) - 1;
  }
  size_t slot_bytes() const { return (size_t)n * kChunk * 8; }
  void open(const double* X_, int64_t ldx_, int64_t n_, int64_t ncols_, bool host_, cudaStream_t s_) {
    X = X_; ldx = ldx_; n = n_; ncols = ncols_; host = host_; s = s_;
    if (!host) return;
    pageable = is_pageable_host(X);
    start.clear();
    for (int64_t c = 0, w = 1; c < ncols; c += w, w = std::min<int64_t>(2 * w, kChunk)) start.push_back(c);
    start.push_back(ncols);
    cs = acquire_stream();
    ring.resize(kRing);
    ready.resize(kRing);
    freed.resize(kRing);
    for (int i = 0; i < kRing; ++i) {
      ring[i] = dev_alloc(slot_bytes(), s, false);
      ready[i] = acquire_event();
      freed[i] = acquire_event();
      STROM_CUDA(cudaEventRecord(freed[i], s));
    }
    if (pageable) {
      hdone.resize(kRing);
      pinned.resize(kRing);
      for (int i = 0; i < kRing; ++i) {
        hdone[i] = acquire_event();
        pinned[i] = acquire_pinned(slot_bytes());
      }
      int dev = 0;
      STROM_CUDA(cudaGetDevice(&dev));
      stager = std::thread([this, dev] { stage_all(dev); });
      return;
    }
    while (issued < std::min<int64_t>(kRing, nchunks())) issue(issued++);
  }
  void issue(int64_t q) {
    const int slot = (int)(q % kRing);
    const int64_t c0 = start[q], cn = start[q + 1] - start[q];
    STROM_CUDA(cudaStreamWaitEvent(cs, freed[slot], 0));
    STROM_CUDA(cudaMemcpy2DAsync(ring[slot]->ptr, n * 8, X + c0 * ldx, ldx * 8, n * 8, cn, cudaMemcpyHostToDevice,
                                 cs));
    STROM_CUDA(cudaEventRecord(ready[slot], cs));
  }
  // pageable mode, stager thread: chunk q -> pinned[slot] -> ring[slot]
  void stage_all(int dev) {
    try {
      STROM_CUDA(cudaSetDevice(dev));
      for (int64_t q = 0; q < nchunks(); ++q) {
        const int slot = (int)(q % kRing);
        const int64_t c0 = start[q], cn = start[q + 1] - start[q];
        if (q >= kRing) STROM_CUDA(cudaEventSynchronize(hdone[slot]));  // DMA of chunk q - kRing is done
        {
          std::unique_lock<std::mutex> g(mu);
          if (abort) return;
        }
        double* dst = static_cast<double*>(pinned[slot]);
        if (ldx == n) {
          parallel_memcpy(dst, X + c0 * ldx, (size_t)cn * n * 8);
        } else {
          for (int64_t c = 0; c < cn; ++c) parallel_memcpy(dst + c * n, X + (c0 + c) * ldx, (size_t)n * 8);
        }
        {
          // the compute thread must have recorded freed[slot] for chunk q - kRing
          std::unique_lock<std::mutex> g(mu);
          cv.wait(g, [&] { return abort || released > q - kRing; });
          if (abort) return;
        }
        STROM_CUDA(cudaStreamWaitEvent(cs, freed[slot], 0));
        STROM_CUDA(cudaMemcpyAsync(ring[slot]->ptr, dst, (size_t)cn * n * 8, cudaMemcpyHostToDevice, cs));
        STROM_CUDA(cudaEventRecord(ready[slot], cs));
        STROM_CUDA(cudaEventRecord(hdone[slot], cs));
        {
          std::lock_guard<std::mutex> g(mu);
          staged = q + 1;
        }
        cv.notify_all();
      }
    } catch (const std::exception& e) {
      std::lock_guard<std::mutex> g(mu);
      stage_error = e.what();
      abort = true;
      cv.notify_all();
    }
  }
  // device pointer of column t; the compute stream waits for its chunk once
  const double* col(int64_t t) {
    if (t < 0 || t >= ncols) return nullptr;
    if (!host) return X + t * ldx;
    const int64_t q = chunk_of(t);
    if (q > waited) {
      if (pageable) {
        std::unique_lock<std::mutex> g(mu);
        cv.wait(g, [&] { return abort || staged > q; });
        if (!stage_error.empty()) throw Error(kCudaError, "host staging: " + stage_error);
      }
      for (int64_t w = waited + 1; w <= q; ++w) STROM_CUDA(cudaStreamWaitEvent(s, ready[w % kRing], 0));
      waited = q;
    }
    return ring[q % kRing]->as<double>() + (t - start[q]) * n;
  }
  // every kernel reading columns <= t has been queued on s
  void release(int64_t t) {
    if (!host) return;
    const int64_t q = chunk_of(t);
    if (t + 1 != start[q + 1]) return;
    STROM_CUDA(cudaEventRecord(freed[q % kRing], s));
    if (pageable) {
      {
        std::lock_guard<std::mutex> g(mu);
        released = q + 1;
      }
      cv.notify_all();
      return;
    }
    if (issued < nchunks() && issued <= q + kRing) issue(issued++);
  }
  void close() {
    if (!host) return;
    if (pageable) {
      {
        std::lock_guard<std::mutex> g(mu);
        abort = true;
      }
      cv.notify_all();
      if (stager.joinable()) stager.join();
    }
    STROM_CUDA(cudaStreamSynchronize(cs));
    for (int i = 0; i < kRing; ++i) {
      release_event(ready[i]);
      release_event(freed[i]);
    }
    if (pageable) {
      for (int i = 0; i < kRing; ++i) {
        release_event(hdone[i]);
        release_pinned(pinned[i], slot_bytes());
      }
    }
    release_stream(cs);
    cs = nullptr;
  }
};

// Pipelined ingestion of ncols snapshots (basis.py:187-194): stream s carries
// the passes and the decisions, stream s2 the core step and V update of update
// t while s already runs the pass of update t+1.
strom_isvd* ingest_pipelined(strom_isvd* src, ColumnSource& cols, cudaStream_t s) {
  const int64_t ncols = cols.ncols;
  static const int dbg = [] {
    const char* e = getenv("STROM_PIPE_DEBUG");
    return e ? atoi(e) : 0;
  }();
  cudaStream_t s2;
  s2 = acquire_stream();
  cudaStream_t s2_created = s2;
  if (dbg & 1) s2 = s;  // diagnostics: one stream
  cudaEvent_t evD, evB, evV;
  evD = acquire_event();
  evB = acquire_event();
  evV = acquire_event();
  // s2 starts after everything queued on s so far
  STROM_CUDA(cudaEventRecord(evV, s));
  STROM_CUDA(cudaStreamWaitEvent(s2, evV, 0));
  std::unique_ptr<strom_isvd> slot[2];
  std::unique_ptr<strom_isvd> hold;  // a compacted state
  strom_isvd* prev = src;
  const int64_t kfinal = src->k + ncols;
  PipeMem m;
  bool need_prep = true;
  int64_t b_launched = 0;  // core steps queued on s2 since the last k_init_ctl
  int64_t d_launched = 0;  // decision chains queued on s since then
  bool fresh_alloc = false;  // this iteration allocated on s: order s2 behind it
  auto join = [&]() {  // s waits for all of s2
    STROM_CUDA(cudaEventRecord(evV, s2));
    STROM_CUDA(cudaStreamWaitEvent(s, evV, 0));
  };
  for (int64_t t = 0; t < ncols; ++t) {
    // ---- capacity (host bounds; synchronises only when a bound is hit)
    {
      const bool rank_hit = prev->r_max < 0 && prev->r_ub + 1 > prev->caps.rcap && prev->caps.rcap < rank_rows(prev);
      const bool col_hit = prev->c_ub + 1 > prev->caps.ccap;
      if (rank_hit || col_hit) {
        join();
        std::unique_ptr<strom_isvd> h2;
        strom_isvd* nx = ensure_capacity(prev, &h2, s);
        if (nx != prev) {
          hold = std::move(h2);
          prev = nx;
          need_prep = true;
        }
        STROM_CUDA(cudaEventRecord(evB, s));  // s2 may not run ahead of the compaction
        STROM_CUDA(cudaStreamWaitEvent(s2, evB, 0));
      }
    }
    if (t == 0) {
      if (prev->store->claimed != prev->c_ub) {
        // copy-on-write once for the whole sequence: intermediate states are private
        std::shared_ptr<Store> st = successor_store(prev, s);
        auto* cp = new strom_isvd(*prev);
        set_store(cp, st);
        hold.reset(cp);
        prev = cp;
      }
    }
    // ---- destination state of update t (ping-pong blocks, V sized for the whole call)
    std::unique_ptr<strom_isvd>& dslot = slot[t & 1];
    if (!dslot || dslot->caps.rcap != prev->caps.rcap || dslot->caps.ccap != prev->caps.ccap) {
      Caps nc = prev->caps;
      nc.kcap = std::max<int64_t>(prev->caps.kcap, round_up(kfinal, 64));
      if (dslot) join();  // the old block may still be read by s2
      dslot.reset(new_like(prev, nc));
      alloc_small(dslot.get(), s);
      alloc_v(dslot.get(), s);
      fresh_alloc = true;
    }
    strom_isvd* dst = dslot.get();
    dst->k = prev->k + 1;
    set_store(dst, prev->store);
    if (!m.mem || m.ccap != prev->caps.ccap || m.rcap != prev->caps.rcap) {
      join();
      m = make_pipe(prev->caps, s);
      need_prep = true;
      fresh_alloc = true;
    }

    IsvdParams P = make_params(dst, m, dst->k, false);
    P.parity = (int)(t & 1);
    P.has_next = (t + 1 < ncols && !(dbg & 2)) ? 1 : 0;
    if (dbg & 2) need_prep = true;  // diagnostics: re-project every snapshot
    const int cols_ub = prev->c_ub;
    const double* xt = cols.col(t);
    const double* xn = cols.col(t + 1);
    if (need_prep) {
      if (t > 0) STROM_CUDA(cudaStreamWaitEvent(s, evB, 0));  // prev's header comes from s2
      k_init_ctl<<<1, 1, 0, s>>>(m.pp.ctl, prev->view.hdr);    // also resets the counters
      STROM_LAUNCH_CHECK();
      b_launched = 0;
      d_launched = 0;
      fresh_alloc = true;  // s2's next core step must see the reset counters
      launch_pass(PASS_PROJ, cols_ub, dst, m, nullptr, xt, 0, s);
      launch_prep(m, P, s);
      need_prep = false;
    }
    if (fresh_alloc) {
      // s2 is ordered behind this point of s: memory the stream-ordered pool
      // handed out on s, and the counters k_init_ctl reset (a core step spinning
      // on a stale counter would run ahead of its decisions)
      STROM_CUDA(cudaEventRecord(evV, s));
      STROM_CUDA(cudaStreamWaitEvent(s2, evV, 0));
      fresh_alloc = false;
    }
    if (decide_as_kernel() || prev->shard) {
      // s: pass -> decide -> second pass -> decide2, kernel to kernel (PDL);
      // the cross-stream dependencies are device counters, not events:
      // k_decide(t) waits for k_step_b(t-1), k_step_b(t) for k_decide2(t)
      // s: pass -> [wait for k_step_b(t-1)] -> decide -> second pass -> decide2
      // (kernel to kernel, PDL).  k_step_b(t) on s2 starts on a device counter
      // that decide2(t) bumps -- no event between decide2 and the next pass.
      // (Measured at cfg2: the decide waiting on an event beats a device spin,
      // which keeps an SM busy; the core step spinning costs nothing, it has
      // the reserved SM anyway.)
      P.b_expect = -1;
      P.d_expect = (int32_t)(d_launched + 1);
      launch_pass(PASS_FUSED, cols_ub, dst, m, xt, (dbg & 2) ? nullptr : xn, 1, s);
      if (b_launched > 0) STROM_CUDA(cudaStreamWaitEvent(s, evB, 0));
      launch_decide_kernel(false, prev->view, m, P, s);
      launch_pass(PASS_SECOND, cols_ub, dst, m, xt, xn, 1, s);
      launch_decide_kernel(true, prev->view, m, P, s);
      ++d_launched;
      cols.release(t);
      launch_step_b(prev->view, dst->view, m, P, prev->caps, s2, prev->r_ub, prev->r_max);
      ++b_launched;
      STROM_CUDA(cudaEventRecord(evB, s2));
      launch_vupdate(prev->view, dst->view, m, P, prev->caps.rcap, s2);
    } else {
      PassTail tl;
      tl.tail = 1;
      tl.b_expect = (int32_t)b_launched;  // D(t) needs B(t-1): the pass's last CTA waits for it
      tl.src = &prev->view;
      tl.P = &P;
      launch_pass(PASS_FUSED, cols_ub, dst, m, xt, (dbg & 2) ? nullptr : xn, 1, s, tl);
      tl.tail = 2;
      launch_pass(PASS_SECOND, cols_ub, dst, m, xt, xn, 1, s, tl);
      cols.release(t);
      STROM_CUDA(cudaEventRecord(evD, s));
      STROM_CUDA(cudaStreamWaitEvent(s2, evD, 0));
      launch_step_b(prev->view, dst->view, m, P, prev->caps, s2, prev->r_ub, prev->r_max);
      ++b_launched;
      STROM_CUDA(cudaEventRecord(evB, s2));
      launch_vupdate(prev->view, dst->view, m, P, prev->caps.rcap, s2);
    }
    dst->c_ub = prev->c_ub + 1;
    dst->store->claimed = std::max(dst->store->claimed, dst->c_ub);
    dst->r_ub = std::min(prev->r_ub + 1, prev->caps.rcap);
    prev = dst;
  }
  join();
  // the result owns its block; the other ping-pong block dies here (stream-ordered free)
  strom_isvd* out = slot[(ncols - 1) & 1].release();
  STROM_CUDA(cudaStreamSynchronize(s2));
  release_event(evD);
  release_event(evB);
  release_event(evV);
  release_stream(s2_created);
  return out;
}

// Window-mode ingestion: per window of up to kWB
// snapshots one projection pass G = U^T X_w (k_wproj); per snapshot t
//   s : k_decide_a(t) -> PASS_RESID(t) [no-op when dependent] -> k_decide_b(t)
//       -> PASS_SECOND(t) [rare] -> k_decide2(t)
//   s2: k_step_b(t): the core SVD as soon as k_decide_a(t) is done (overlapping
//       the residual pass), the N update after k_decide2(t)
//   s3: k_vupdate(t) (off the critical path; V_bar and its record are
//       parity-buffered, k_step_b(t+2) waits for k_vupdate(t))
// Every decision stays on the device; the host only orders the launches.
strom_isvd* ingest_windowed(strom_isvd* src, ColumnSource& cols, cudaStream_t s, int wb) {
  const int64_t ncols = cols.ncols;
  cudaStream_t s2 = acquire_stream(), s3 = acquire_stream();
  cudaEvent_t evB = acquire_event(), evJ = acquire_event(), evJ3 = acquire_event();
  cudaEvent_t evU[2] = {acquire_event(), acquire_event()};
  bool u_pending[2] = {false, false};
  STROM_CUDA(cudaEventRecord(evJ, s));
  STROM_CUDA(cudaStreamWaitEvent(s2, evJ, 0));
  STROM_CUDA(cudaStreamWaitEvent(s3, evJ, 0));
  std::unique_ptr<strom_isvd> slot[2];
  std::unique_ptr<strom_isvd> hold;
  strom_isvd* prev = src;
  const int64_t kfinal = src->k + ncols;
  PipeMem m;
  bool need_init = true;
  int64_t w0 = 0, wn = 0;
  int64_t b_launched = 0, d_launched = 0;
  bool fresh_alloc = false;
  auto join = [&]() {  // s waits for all of s2 and s3
    STROM_CUDA(cudaEventRecord(evJ, s2));
    STROM_CUDA(cudaStreamWaitEvent(s, evJ, 0));
    STROM_CUDA(cudaEventRecord(evJ3, s3));
    STROM_CUDA(cudaStreamWaitEvent(s, evJ3, 0));
  };
  static const bool host_timing = getenv("STROM_HOST_TIMING") != nullptr;  // diagnostics: enqueue time of the loop
  const auto host_t0 = std::chrono::steady_clock::now();
  for (int64_t t = 0; t < ncols; ++t) {
    {
      const bool rank_hit = prev->r_max < 0 && prev->r_ub + 1 > prev->caps.rcap && prev->caps.rcap < rank_rows(prev);
      const bool col_hit = prev->c_ub + 1 > prev->caps.ccap;
      if (rank_hit || col_hit) {
        join();
        std::unique_ptr<strom_isvd> h2;
        strom_isvd* nx = ensure_capacity(prev, &h2, s);
        if (nx != prev) {
          hold = std::move(h2);
          prev = nx;
          need_init = true;
        }
        fresh_alloc = true;  // s2 / s3 may not run ahead of the compaction
      }
    }
    if (t == 0 && prev->store->claimed != prev->c_ub) {
      std::shared_ptr<Store> st = successor_store(prev, s);
      auto* cp = new strom_isvd(*prev);
      set_store(cp, st);
      hold.reset(cp);
      prev = cp;
    }
    std::unique_ptr<strom_isvd>& dslot = slot[t & 1];
    if (!dslot || dslot->caps.rcap != prev->caps.rcap || dslot->caps.ccap != prev->caps.ccap) {
      Caps nc = prev->caps;
      nc.kcap = std::max<int64_t>(prev->caps.kcap, round_up(kfinal, 64));
      if (dslot) join();
      dslot.reset(new_like(prev, nc));
      alloc_small(dslot.get(), s);
      alloc_v(dslot.get(), s);
      fresh_alloc = true;
    }
    strom_isvd* dst = dslot.get();
    dst->k = prev->k + 1;
    set_store(dst, prev->store);
    if (!m.mem || m.ccap != prev->caps.ccap || m.rcap != prev->caps.rcap) {
      join();
      m = make_pipe(prev->caps, s);
      need_init = true;
      fresh_alloc = true;
    }
    const int cols_ub = prev->c_ub;
    IsvdParams P = make_params(dst, m, dst->k, false);
    P.parity = (int)(t & 1);
    if (need_init) {
      join();  // prev's header comes from s2; the counters restart
      k_init_ctl<<<1, 1, 0, s>>>(m.pp.ctl, prev->view.hdr);
      STROM_LAUNCH_CHECK();
      b_launched = 0;
      d_launched = 0;
      fresh_alloc = true;
      wn = 0;  // a new window (U may have changed under the old one)
      need_init = false;
    }
    g_cur_trace = (g_trace && t < g_trace_rows) ? g_trace + 16 * t : nullptr;
    P.trace = g_cur_trace;
    if (t >= w0 + wn) {
      w0 = t;
      wn = std::min<int64_t>(wb, ncols - t);
      const double* xs[kWB];
      for (int j = 0; j < wn; ++j) xs[j] = cols.col(t + j);
      launch_window(dst, m, xs, (int)wn, cols_ub, P, s);
    }
    if (fresh_alloc) {
      STROM_CUDA(cudaEventRecord(evJ, s));
      STROM_CUDA(cudaStreamWaitEvent(s2, evJ, 0));
      STROM_CUDA(cudaStreamWaitEvent(s3, evJ, 0));
      fresh_alloc = false;
    }
    P.wG = m.wG;
    P.wXX = m.wXX;
    P.ldg = m.ldg;
    P.wn = (int)wn;
    P.wcol = (int)(t - w0);
    P.has_next = (P.wcol + 1 < P.wn) ? 1 : 0;
    // k_decide_a(t) waits for k_step_b(t-1) on a cross-stream event (or spins on
    // its device counter with STROM_DECIDE_SPIN=1)
    P.b_expect = decide_spins() ? (int32_t)b_launched : -1;
    P.d_expect = (int32_t)(d_launched + 1);
    P.trace = (g_trace && t < g_trace_rows) ? g_trace + 16 * t : nullptr;
    g_cur_trace = P.trace;
    Pipe pp = m.pp;
    pp.fo.gn = m.wG + (int64_t)(P.has_next ? P.wcol + 1 : 0) * m.ldg;
    pp.vbar = (t & 1) ? m.vbar2 : m.pp.vbar;
    const double* xt = cols.col(t);
    const double* xw[kWB];
    const int nxw = (int)(wn - 1 - P.wcol);
    for (int j = 0; j < nxw; ++j) xw[j] = cols.col(t + 1 + j);
    if (b_launched > 0 && !decide_spins()) STROM_CUDA(cudaStreamWaitEvent(s, evB, 0));  // k_step_b(t-1) wrote N
    launch_decide_w(0, prev->view, pp, m, P, s);
    launch_pass(PASS_RESID, cols_ub, dst, m, xt, nullptr, 1, s, PassTail(), xw, nxw);
    launch_decide_w(1, prev->view, pp, m, P, s);
    launch_pass(PASS_SECOND, cols_ub, dst, m, xt, nullptr, 1, s, PassTail(), xw, nxw);
    launch_decide_w(2, prev->view, pp, m, P, s);
    ++d_launched;
    cols.release(t);
    // s2: the core step (V_bar[t & 1] is free once k_vupdate(t - 2) is done).  It
    // may also run snapshot t+1's first-half decision when nothing can come
    // between them: same window, and no capacity event at t+1 (host bounds)
    if (u_pending[t & 1]) STROM_CUDA(cudaStreamWaitEvent(s2, evU[t & 1], 0));
    {
      const int32_t c_ub = prev->c_ub + 1;
      const int32_t r_ub = std::min(prev->r_ub + 1, prev->caps.rcap);
      const bool rank_hit = prev->r_max < 0 && r_ub + 1 > prev->caps.rcap && prev->caps.rcap < rank_rows(prev);
      const bool col_hit = c_ub + 1 > prev->caps.ccap;
      P.inline_next = (P.has_next && !rank_hit && !col_hit && inline_decide()) ? 1 : 0;
    }
    launch_step_b_pp(prev->view, dst->view, pp, P, prev->caps, s2, prev->r_ub, prev->r_max);
    ++b_launched;
    STROM_CUDA(cudaEventRecord(evB, s2));
    // s3: the V update
    STROM_CUDA(cudaStreamWaitEvent(s3, evB, 0));
    launch_vupdate_pp(prev->view, dst->view, pp, P, prev->caps.rcap, s3);
    STROM_CUDA(cudaEventRecord(evU[t & 1], s3));
    g_cur_trace = nullptr;
    u_pending[t & 1] = true;
    dst->c_ub = prev->c_ub + 1;
    dst->store->claimed = std::max(dst->store->claimed, dst->c_ub);
    dst->r_ub = std::min(prev->r_ub + 1, prev->caps.rcap);
    prev = dst;
  }
  if (host_timing) {
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - host_t0).count();
    fprintf(stderr, "[strom] window ingest: %lld snapshots enqueued in %.0f us (%.1f us each)\n", (long long)ncols, us,
            us / (double)std::max<int64_t>(1, ncols));
  }
  join();
  strom_isvd* out = slot[(ncols - 1) & 1].release();
  STROM_CUDA(cudaStreamSynchronize(s2));
  STROM_CUDA(cudaStreamSynchronize(s3));
  release_event(evB);
  release_event(evJ);
  release_event(evJ3);
  release_event(evU[0]);
  release_event(evU[1]);
  release_stream(s2);
  release_stream(s3);
  return out;
}

// A brand-new state created while a shard group is current (strom_shard_make_current)
// is that rank's row block of the group's matrix.
void adopt_current_shard(strom_isvd* h) {
  h->n_global = h->n;
  if (!t_current_shard) return;
  STROM_REQUIRE(t_current_shard->connected, "the current shard group is not connected");
  STROM_REQUIRE(t_current_shard->n_global >= h->n, "shard group: global row count below the local one");
  h->shard = t_current_shard;
  h->n_global = t_current_shard->n_global;
}

strom_isvd* init_state(int64_t n, const double* x, int64_t k, double tol_svd, double tol_sv, int64_t r_max,
                       int32_t cap_mode, cudaStream_t s) {
  STROM_REQUIRE(n >= 1, "need n >= 1");
  STROM_REQUIRE(k >= 1, "need k >= 1");
  STROM_REQUIRE(cap_mode == 0 || cap_mode == 1, "unknown cap_mode");
  // an empty state (r = c = base = 0) at column k - 1; the update machinery's
  // restart branch then implements isvd_init (basis.py:65-102)
  strom_isvd e;
  e.n = n;
  adopt_current_shard(&e);
  e.ldu = round_up(n, kGemmRows);
  e.k = k - 1;
  e.tol_svd = tol_svd;
  e.tol_sv = tol_sv;
  e.r_max = (int32_t)r_max;
  e.cap_mode = cap_mode;
  e.caps = make_caps(rank_rows(&e), e.r_max, 1, k, mem_rows(&e));
  alloc_small(&e, s);
  alloc_v(&e, s);
  set_store(&e, alloc_store(n, e.ldu, e.caps.ccap, s));
  e.c_ub = 0;
  e.r_ub = 0;
  return update_once(&e, x, s, true);
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
    STROM_REQUIRE(src && x_dev && out, "null argument");
    *out = update_once(src, x_dev, as_stream(stream));
  });
}

int strom_isvd_ingest(strom_isvd* src, const double* X, int64_t ldx, int64_t ncols, int32_t x_on_host,
                      void* stream, strom_isvd** out) {
  return guarded([&] {
    STROM_REQUIRE(src && out, "null argument");
    STROM_REQUIRE(ncols >= 0 && ldx >= src->n, "bad ingest shape");
    cudaStream_t s = as_stream(stream);
    if (ncols == 0) {
      *out = new strom_isvd(*src);  // a copy of the state (new handle sharing immutable buffers)
      return;
    }
    ColumnSource cols;
    cols.open(X, ldx, src->n, ncols, x_on_host != 0, s);
    strom_isvd* res = nullptr;
    try {
      const int wb = choose_window(src, s);
      res = wb > 1 ? ingest_windowed(src, cols, s, wb) : ingest_pipelined(src, cols, s);
    } catch (...) {
      cols.close();
      throw;
    }
    cols.close();
    *out = res;
  });
}

int strom_isvd_query(strom_isvd* h, void* stream, strom_isvd_info* out) {
  return guarded([&] {
    STROM_REQUIRE(h && out, "null argument");
    IsvdHdr hh;
    read_hdr(h, as_stream(stream), &hh);
    if (h->shard) shard_check(h->shard.get());
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

void strom_trim_cache(void) {
  SpareStore& sp = spare_store();
  std::lock_guard<std::mutex> g(sp.mu);
  for (auto& m : sp.mem) m.reset();
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
      launch_tall_gemm(tall_tiled(h->store->U(), h->store->ccap), &h->view.hdr->base, wtmp->as<double>(), hh.c,
                       &h->view.hdr->c, &h->view.hdr->r, tall_cm(phi_dev, r), true, h->n, h->ldu, s);
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
    adopt_current_shard(h);
    h->ldu = round_up(n, kGemmRows);
    h->k = k;
    h->tol_svd = tol_svd;
    h->tol_sv = tol_sv;
    h->r_max = (int32_t)r_max;
    h->cap_mode = cap_mode;
    h->caps = make_caps(rank_rows(h), h->r_max, (int32_t)std::max<int64_t>(c, r + 1), k, mem_rows(h));
    STROM_REQUIRE(c + 1 <= h->caps.ccap, "too many factored columns for this capacity");
    alloc_small(h, s);
    alloc_v(h, s);
    set_store(h, alloc_store(n, h->ldu, h->caps.ccap, s));
    if (c > 0) {
      k_copy_tall<<<(unsigned)ceil_div(n * c, 256), 256, 0, s>>>(tall_cm(u_dev, ldu), n, c,
                                                                tall_tiled(h->store->U(), h->store->ccap));
      STROM_LAUNCH_CHECK();
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
        gram_cholesky(tall_tiled(h->store->U(), h->store->ccap), nullptr, nullptr, (int)c, (int)c, n, h->view.L,
                      h->view.Li,
                      h->view.ldl, nullptr, st->as<int>(), s, h->shard);
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
    h->store->claimed = (int32_t)c;
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
    if (u_dev && hh.c > 0) {
      Tall src = tall_tiled(h->store->U(), h->store->ccap);
      src.p += (int64_t)hh.base * kUTile;  // logical column 0 = physical column base
      k_copy_tall<<<(unsigned)ceil_div(h->n * hh.c, 256), 256, 0, s>>>(src, h->n, hh.c, tall_cm(u_dev, h->n));
      STROM_LAUNCH_CHECK();
    }
    if (w_dev && hh.c > 0 && hh.r > 0) {
      k_n_to_w<<<(unsigned)ceil_div((int64_t)hh.c * hh.r, 256), 256, 0, s>>>(h->view, w_dev);
      STROM_LAUNCH_CHECK();
    }
    if (l_dev && hh.c > 0)
      STROM_CUDA(cudaMemcpy2DAsync(l_dev, hh.c * 8, h->view.L + (int64_t)hh.base * (h->view.ldl + 1),
                                   h->view.ldl * 8, hh.c * 8, hh.c,
                                   cudaMemcpyDeviceToDevice, s));
    STROM_CUDA(cudaStreamSynchronize(s));
  });
}

// Diagnostics: time `iters` FUSED passes over a synthetic n x c store (random
// values), reserve SMs left idle; writes the mean ms per pass.
int strom_debug_pass_bw(int64_t n, int32_t c, int32_t iters, int32_t reserve, double* ms_out) {
  return guarded([&] {
    cudaStream_t s = nullptr;  // legacy stream: outlives every stream-ordered free below
    strom_isvd h;
    h.n = n;
    h.ldu = round_up(n, kGemmRows);
    h.caps = make_caps(n, -1, std::max(c, 1), 1);
    STROM_REQUIRE(c + 1 <= h.caps.ccap, "c too large for the capacity");
    set_store(&h, alloc_store(n, h.ldu, h.caps.ccap, s));
    STROM_CUDA(cudaMemsetAsync(h.store->U(), 0, (size_t)h.ldu * h.caps.ccap * 8, s));
    auto xs = dev_alloc((size_t)n * 2 * 8, s, true);
    PipeMem m = make_pipe(h.caps, s);
    std::vector<int32_t> ctl = {c, 0, 0, 0};
    STROM_CUDA(cudaMemcpyAsync(m.pp.ctl, ctl.data(), 16, cudaMemcpyHostToDevice, s));
    cudaEvent_t e0, e1;
    STROM_CUDA(cudaEventCreate(&e0));
    STROM_CUDA(cudaEventCreate(&e1));
    launch_pass(PASS_FUSED, c, &h, m, xs->as<double>(), xs->as<double>() + n, reserve, s);
    STROM_CUDA(cudaEventRecord(e0, s));
    for (int i = 0; i < iters; ++i) launch_pass(PASS_FUSED, c, &h, m, xs->as<double>(), xs->as<double>() + n, reserve, s);
    STROM_CUDA(cudaEventRecord(e1, s));
    STROM_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    STROM_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *ms_out = ms / std::max(iters, 1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    STROM_CUDA(cudaStreamSynchronize(s));
  });
}

// Diagnostics: point step B's phase timestamps (clock64, 8 slots) at a device
// buffer, or NULL to disable.
void strom_debug_tprobe(long long* dev_buf) { g_tprobe = dev_buf; }

// Diagnostics: globaltimer stamps (16 per update: decide A/B, passes, core step,
// V update, window pass) of the first `rows` updates of the next window-mode
// ingest calls into dev_buf (rows x 16 int64); NULL disables.
void strom_debug_trace(long long* dev_buf, int64_t rows) {
  g_trace = dev_buf;
  g_trace_rows = dev_buf ? rows : 0;
}

// ------------------------------------------------------------------ row-shard groups (shard.cuh)
int strom_shard_mailbox_create(int32_t world, strom_shard** out, void* handle64_out) {
  return guarded([&] {
    STROM_REQUIRE(out && handle64_out, "null argument");
    STROM_REQUIRE(world >= 1 && world <= kShardMax, "shard groups hold 1..8 ranks");
    static_assert(sizeof(cudaIpcMemHandle_t) == STROM_SHARD_HANDLE_BYTES, "IPC handle size");
    auto g = std::make_unique<strom_shard>();
    g->impl = std::make_shared<ShardImpl>();
    g->impl->alloc(world);
    cudaIpcMemHandle_t hnd;
    memset(&hnd, 0, sizeof(hnd));
    if (world > 1) STROM_CUDA(cudaIpcGetMemHandle(&hnd, g->impl->mailbox));
    memcpy(handle64_out, &hnd, sizeof(hnd));
    *out = g.release();
  });
}

int strom_shard_connect(strom_shard* g, int32_t rank, int64_t n_global, const void* handles_host) {
  return guarded([&] {
    STROM_REQUIRE(g && g->impl, "null argument");
    ShardImpl* im = g->impl.get();
    STROM_REQUIRE(!im->connected, "shard group already connected");
    STROM_REQUIRE(rank >= 0 && rank < im->world, "rank outside the group");
    STROM_REQUIRE(n_global >= 1, "need n_global >= 1");
    STROM_REQUIRE(im->world == 1 || handles_host, "need the peers' mailbox handles");
    for (int p = 0; p < im->world; ++p) {
      if (p == rank) {
        im->peer[p] = im->mailbox;
        continue;
      }
      cudaIpcMemHandle_t hnd;
      memcpy(&hnd, static_cast<const char*>(handles_host) + (size_t)p * sizeof(hnd), sizeof(hnd));
      // maps the peer GPU's mailbox here and enables peer access (NVLink / NVSwitch)
      STROM_CUDA(cudaIpcOpenMemHandle(&im->peer[p], hnd, cudaIpcMemLazyEnablePeerAccess));
      im->ipc_opened[p] = true;
    }
    im->finish(rank, n_global);
  });
}

int strom_shard_create_local(int32_t world, int64_t n_global, strom_shard** out) {
  return guarded([&] {
    STROM_REQUIRE(out, "null argument");
    STROM_REQUIRE(world >= 1 && world <= kShardMax, "shard groups hold 1..8 ranks");
    STROM_REQUIRE(n_global >= 1, "need n_global >= 1");
    std::vector<std::unique_ptr<strom_shard>> gs;
    auto ls = std::make_shared<LocalSync>();
    ls->world = world;
    for (int r = 0; r < world; ++r)
      for (int i = 0; i < LocalSync::kRing; ++i)
        STROM_CUDA(cudaEventCreateWithFlags(&ls->ev[r][i], cudaEventDisableTiming));
    for (int r = 0; r < world; ++r) {
      gs.emplace_back(new strom_shard());
      gs.back()->impl = std::make_shared<ShardImpl>();
      gs.back()->impl->alloc(world);
      gs.back()->impl->lsync = ls;
    }
    for (int r = 0; r < world; ++r) {
      for (int p = 0; p < world; ++p) {
        gs[r]->impl->peer[p] = gs[p]->impl->mailbox;
        gs[r]->impl->peers_mem.push_back(gs[p]->impl->box_mem);  // outlives every rank that stores into it
      }
      gs[r]->impl->finish(r, n_global);
    }
    for (int r = 0; r < world; ++r) out[r] = gs[r].release();
  });
}

void strom_shard_make_current(strom_shard* g) { t_current_shard = g ? g->impl : nullptr; }

int strom_shard_status(strom_shard* g, int64_t* exchanges_out, int32_t* error_out) {
  return guarded([&] {
    STROM_REQUIRE(g && g->impl && g->impl->connected, "shard group not connected");
    STROM_CUDA(cudaDeviceSynchronize());
    unsigned long long seq = 0;
    int32_t err = 0;
    STROM_CUDA(cudaMemcpy(&seq, g->impl->dev.seq, sizeof(seq), cudaMemcpyDeviceToHost));
    STROM_CUDA(cudaMemcpy(&err, g->impl->dev.err, sizeof(err), cudaMemcpyDeviceToHost));
    if (exchanges_out) *exchanges_out = (int64_t)seq;
    if (error_out) *error_out = err;
  });
}

void strom_shard_free(strom_shard* g) { delete g; }

void strom_isvd_free(strom_isvd* h) { delete h; }

}  // extern "C"
