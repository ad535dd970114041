#include <cstring>
#include <mutex>
#include <algorithm>
#include <cstdlib>
#include <thread>
#include <condition_variable>
#include <vector>

#include "runtime.cuh"
#include "../../include/strom_b200.h"

namespace strom {

static thread_local std::string g_last_error;

void set_last_error(const std::string& msg) { g_last_error = msg; }

static void configure_pool_once() {
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;  // keep freed blocks cached in the pool
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
}

DevMem::DevMem(size_t b, cudaStream_t s) : bytes(b), stream(s) {
  configure_pool_once();
  if (b == 0) return;
  cudaError_t e = cudaMallocAsync(&ptr, b, s);
  if (e != cudaSuccess) {
    ptr = nullptr;
    throw Error(kCudaError, std::string("cudaMallocAsync(") + std::to_string(b) + "): " + cudaGetErrorString(e));
  }
}

DevMem::~DevMem() {
  if (ptr) cudaFreeAsync(ptr, stream);
}

DevMemPtr dev_alloc(size_t bytes, cudaStream_t s, bool zero) {
  auto m = std::make_shared<DevMem>(bytes, s);
  if (zero && bytes) STROM_CUDA(cudaMemsetAsync(m->ptr, 0, bytes, s));
  return m;
}

int current_device_id() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
  return d;
}

int sm_count() {
  static PerDevice<int> cache;
  int& n = cache.get();
  if (n == 0) {
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, current_device_id());
    n = v;
  }
  return n;
}

size_t device_total_mem() {
  static PerDevice<size_t> cache;
  size_t& n = cache.get();
  if (n == 0) {
    size_t f = 0, t = 0;
    n = cudaMemGetInfo(&f, &t) == cudaSuccess ? t : (size_t)0;
  }
  return n;
}

namespace {
std::mutex g_res_mu;
std::vector<std::pair<int, cudaStream_t>> g_streams;
std::vector<std::pair<int, cudaEvent_t>> g_events;
int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
}  // namespace

cudaStream_t acquire_stream() {
  const int d = current_device();
  {
    std::lock_guard<std::mutex> g(g_res_mu);
    for (size_t i = 0; i < g_streams.size(); ++i)
      if (g_streams[i].first == d) {
        cudaStream_t s = g_streams[i].second;
        g_streams.erase(g_streams.begin() + (std::ptrdiff_t)i);
        return s;
      }
  }
  cudaStream_t s;
  STROM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  return s;
}

void release_stream(cudaStream_t s) {
  if (!s) return;
  std::lock_guard<std::mutex> g(g_res_mu);
  g_streams.emplace_back(current_device(), s);
}

cudaEvent_t acquire_event() {
  const int d = current_device();
  {
    std::lock_guard<std::mutex> g(g_res_mu);
    for (size_t i = 0; i < g_events.size(); ++i)
      if (g_events[i].first == d) {
        cudaEvent_t e = g_events[i].second;
        g_events.erase(g_events.begin() + (std::ptrdiff_t)i);
        return e;
      }
  }
  cudaEvent_t e;
  STROM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return e;
}

void release_event(cudaEvent_t e) {
  if (!e) return;
  std::lock_guard<std::mutex> g(g_res_mu);
  g_events.emplace_back(current_device(), e);
}

namespace {
std::vector<std::pair<size_t, void*>> g_pinned;
}  // namespace

void* acquire_pinned(size_t bytes) {
  {
    std::lock_guard<std::mutex> g(g_res_mu);
    for (size_t i = 0; i < g_pinned.size(); ++i)
      if (g_pinned[i].first == bytes) {
        void* p = g_pinned[i].second;
        g_pinned.erase(g_pinned.begin() + (std::ptrdiff_t)i);
        return p;
      }
  }
  void* p = nullptr;
  STROM_CUDA(cudaHostAlloc(&p, bytes, cudaHostAllocPortable));
  return p;
}

void release_pinned(void* p, size_t bytes) {
  if (!p) return;
  std::lock_guard<std::mutex> g(g_res_mu);
  g_pinned.emplace_back(bytes, p);
}

bool is_pageable_host(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

namespace {
// Persistent copy workers: job = [dst, src, bytes) split in equal pieces; the
// caller copies piece 0 and waits for the rest.
struct CopyPool {
  std::mutex mu;
  std::condition_variable cv_job, cv_done;
  std::vector<std::thread> workers;
  char* dst = nullptr;
  const char* src = nullptr;
  size_t bytes = 0;
  int pieces = 1;
  uint64_t gen = 0;
  int pending = 0;
  bool stop = false;

  explicit CopyPool(int nworkers) {
    for (int w = 0; w < nworkers; ++w) workers.emplace_back([this, w] { run(w + 1); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(mu);
      stop = true;
    }
    cv_job.notify_all();
    for (auto& t : workers) t.join();
  }
  void piece(int i, char* d, const char* s0, size_t b, int np) {
    const size_t per = (b / np + 63) & ~(size_t)63;
    const size_t lo = std::min(b, per * (size_t)i), hi = std::min(b, lo + per);
    if (hi > lo) std::memcpy(d + lo, s0 + lo, hi - lo);
  }
  void run(int idx) {
    uint64_t seen = 0;
    for (;;) {
      char* d;
      const char* s0;
      size_t b;
      int np;
      {
        std::unique_lock<std::mutex> g(mu);
        cv_job.wait(g, [&] { return stop || gen != seen; });
        if (stop) return;
        seen = gen;
        d = dst; s0 = src; b = bytes; np = pieces;
      }
      if (idx < np) piece(idx, d, s0, b, np);
      {
        std::lock_guard<std::mutex> g(mu);
        if (--pending == 0) cv_done.notify_one();
      }
    }
  }
  void copy(void* d, const void* s0, size_t b) {
    const int np = (int)workers.size() + 1;
    if (b < ((size_t)1 << 20) || np == 1) {
      std::memcpy(d, s0, b);
      return;
    }
    {
      std::lock_guard<std::mutex> g(mu);
      dst = static_cast<char*>(d);
      src = static_cast<const char*>(s0);
      bytes = b;
      pieces = np;
      pending = (int)workers.size();
      ++gen;
    }
    cv_job.notify_all();
    piece(0, static_cast<char*>(d), static_cast<const char*>(s0), b, np);
    std::unique_lock<std::mutex> g(mu);
    cv_done.wait(g, [&] { return pending == 0; });
  }
};
std::mutex g_copy_mu;  // one job at a time
}  // namespace

void parallel_memcpy(void* dst, const void* src, size_t bytes) {
  static CopyPool* pool = [] {
    const char* e = getenv("STROM_COPY_THREADS");
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    int nt = e ? atoi(e) : (int)std::min(8u, std::max(1u, hw / 2));
    return new CopyPool(std::max(0, nt - 1));  // leaked: lives for the process
  }();
  std::lock_guard<std::mutex> g(g_copy_mu);
  pool->copy(dst, src, bytes);
}

size_t max_smem_optin() {
  static PerDevice<size_t> cache;
  size_t& n = cache.get();
  if (n == 0) {
    int v = 48 * 1024;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, current_device_id());
    n = (size_t)v;
  }
  return n;
}

// ------------------------------------------------------------------ profiling
namespace {
struct ProfState {
  std::mutex mu;
  bool on = false;
  long long launches[P_NKINDS] = {};
  double host_bytes[P_NKINDS] = {};
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pairs;
  cudaEvent_t open[P_NKINDS] = {};
  unsigned long long* dev_bytes = nullptr;
};
ProfState& prof() {
  static ProfState p;
  return p;
}
}  // namespace

unsigned long long* prof_dev_bytes() {
  auto& p = prof();
  std::lock_guard<std::mutex> g(p.mu);
  if (!p.dev_bytes) {
    if (cudaMalloc(&p.dev_bytes, sizeof(unsigned long long) * P_NKINDS) != cudaSuccess) {
      p.dev_bytes = nullptr;
      throw Error(kCudaError, "cannot allocate the profile counters");
    }
    cudaMemset(p.dev_bytes, 0, sizeof(unsigned long long) * P_NKINDS);
  }
  return p.dev_bytes;
}

void prof_begin(int kind, cudaStream_t s) {
  auto& p = prof();
  std::lock_guard<std::mutex> g(p.mu);
  p.launches[kind] += 1;
  if (!p.on) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, s);
  p.open[kind] = e;
}

void prof_end(int kind, cudaStream_t s) {
  auto& p = prof();
  std::lock_guard<std::mutex> g(p.mu);
  if (!p.on || !p.open[kind]) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, s);
  p.pairs.push_back({kind, {p.open[kind], e}});
  p.open[kind] = nullptr;
}

void prof_add_bytes(int kind, double bytes) {
  auto& p = prof();
  std::lock_guard<std::mutex> g(p.mu);
  p.host_bytes[kind] += bytes;
}

}  // namespace strom

namespace {
// fp64 tensor-pipe probe: every warp issues `iters` x 8 independent DMMA.
__global__ void __launch_bounds__(256) k_dmma_probe(int iters, double* sink) {
  const int lane = threadIdx.x & 31;
  double c[8][2];
#pragma unroll
  for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = 0.0;
  double a = 1.0 + 1e-3 * lane, b = 1.0 - 1e-3 * lane;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
  if (s == 12345.678) sink[0] = s;
}
}  // namespace

extern "C" {

const char* strom_last_error(void) { return strom::g_last_error.c_str(); }

int strom_abi_version(void) { return STROM_B200_ABI_VERSION; }

int strom_device_synchronize(void) {
  return strom::guarded([] { STROM_CUDA(cudaDeviceSynchronize()); });
}

void strom_profile_enable(int32_t on) {
  auto& p = strom::prof();
  std::lock_guard<std::mutex> g(p.mu);
  p.on = on != 0;
}

int strom_profile_reset(void) {
  return strom::guarded([] {
    unsigned long long* d = strom::prof_dev_bytes();
    auto& p = strom::prof();
    std::lock_guard<std::mutex> g(p.mu);
    for (auto& pr : p.pairs) {
      cudaEventDestroy(pr.second.first);
      cudaEventDestroy(pr.second.second);
    }
    p.pairs.clear();
    for (int k = 0; k < strom::P_NKINDS; ++k) {
      p.launches[k] = 0;
      p.host_bytes[k] = 0.0;
      p.open[k] = nullptr;
    }
    STROM_CUDA(cudaMemset(d, 0, sizeof(unsigned long long) * strom::P_NKINDS));
  });
}

int strom_profile_read(int32_t nkinds, int64_t* launches, double* ms, double* bytes) {
  return strom::guarded([&] {
    unsigned long long* d = strom::prof_dev_bytes();
    STROM_CUDA(cudaDeviceSynchronize());
    unsigned long long db[strom::P_NKINDS];
    STROM_CUDA(cudaMemcpy(db, d, sizeof(db), cudaMemcpyDeviceToHost));
    auto& p = strom::prof();
    std::lock_guard<std::mutex> g(p.mu);
    const int nk = nkinds < strom::P_NKINDS ? nkinds : strom::P_NKINDS;
    for (int k = 0; k < nk; ++k) {
      if (launches) launches[k] = p.launches[k];
      if (bytes) bytes[k] = p.host_bytes[k] + (double)db[k];
      if (ms) ms[k] = 0.0;
    }
    if (ms)
      for (auto& pr : p.pairs) {
        float t = 0.f;
        if (pr.first < nk && cudaEventElapsedTime(&t, pr.second.first, pr.second.second) == cudaSuccess)
          ms[pr.first] += t;
      }
  });
}

int strom_profile_durations(int32_t kind, int32_t max, float* ms, int32_t* n_out) {
  return strom::guarded([&] {
    STROM_REQUIRE(kind >= 0 && kind < strom::P_NKINDS && n_out, "bad profile kind");
    STROM_CUDA(cudaDeviceSynchronize());
    auto& p = strom::prof();
    std::lock_guard<std::mutex> g(p.mu);
    int n = 0;
    for (auto& pr : p.pairs) {
      if (pr.first != kind) continue;
      float t = 0.f;
      if (cudaEventElapsedTime(&t, pr.second.first, pr.second.second) != cudaSuccess) t = -1.f;
      if (ms && n < max) ms[n] = t;
      ++n;
    }
    *n_out = n;
  });
}

int strom_fp64_probe(int32_t iters, int32_t ctas_per_sm, void* stream, double* flops_out) {
  return strom::guarded([&] {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int grid = strom::sm_count() * (ctas_per_sm > 0 ? ctas_per_sm : 4);
    auto sink = strom::dev_alloc(8, s, false);
    k_dmma_probe<<<grid, 256, 0, s>>>(iters, sink->as<double>());
    STROM_LAUNCH_CHECK();
    // 8 DMMA (8x8x4 = 256 FMA = 512 flop) per warp per iteration
    *flops_out = (double)grid * 8.0 * (double)iters * 8.0 * 512.0;
  });
}

}  // extern "C"
