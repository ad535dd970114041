// Host runtime shared by the C-ABI entry points: error state, stream-ordered
// device memory, launch checks.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <stdexcept>
#include <string>

namespace strom {

enum Status : int {
  kOk = 0,
  kInvalidArgument = 1,
  kCudaError = 2,
  kNumericalError = 3,
  kSingularMatrix = 4,
  kRankError = 5,
  kInternal = 6,
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

#define STROM_CUDA(expr)                                                                  \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess) {                                                              \
      (void)cudaGetLastError(); /* reported here: a later launch check must not see it */ \
      throw ::strom::Error(::strom::kCudaError, std::string(#expr) + ": " +               \
                                                    cudaGetErrorString(_e));              \
    }                                                                                     \
  } while (0)

#define STROM_STR2(x) #x
#define STROM_STR(x) STROM_STR2(x)
#define STROM_LAUNCH_CHECK()                                                              \
  do {                                                                                    \
    cudaError_t _e = cudaGetLastError();                                                  \
    if (_e != cudaSuccess)                                                                \
      throw ::strom::Error(::strom::kCudaError, std::string("kernel launch at " __FILE__   \
                                                            ":" STROM_STR(__LINE__) ": ") + \
                                                    cudaGetErrorString(_e));              \
  } while (0)

#define STROM_REQUIRE(cond, msg)                                                          \
  do {                                                                                    \
    if (!(cond)) throw ::strom::Error(::strom::kInvalidArgument, (msg));                  \
  } while (0)

// Stream-ordered device allocation (cudaMallocAsync pool); freed on the stream
// that allocated it, so reuse is ordered after every kernel queued there.
struct DevMem {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaStream_t stream = nullptr;
  DevMem(size_t b, cudaStream_t s);
  ~DevMem();
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
  template <class T>
  T* as() const { return static_cast<T*>(ptr); }
};
using DevMemPtr = std::shared_ptr<DevMem>;
DevMemPtr dev_alloc(size_t bytes, cudaStream_t s, bool zero = false);

// Process-wide caches are keyed by device: a function attribute set or an
// attribute queried on one GPU says nothing about another GPU of the process.
constexpr int kMaxDevices = 64;
int current_device_id();  // cudaGetDevice, clamped to [0, kMaxDevices)
template <class T>
struct PerDevice {
  T v[kMaxDevices] = {};
  T& get() { return v[current_device_id()]; }
};

int sm_count();
size_t max_smem_optin();
size_t device_total_mem();  // HBM bytes of the current device (queried once per device)

// Non-blocking streams and timing-free events recycled across calls: creating
// and destroying them per ingest call is a driver round trip each, and those
// occasionally stall for hundreds of milliseconds.  A recycled stream may
// still hold work of an earlier call; new work queues behind it.
cudaStream_t acquire_stream();
void release_stream(cudaStream_t s);
cudaEvent_t acquire_event();
void release_event(cudaEvent_t e);

// Pinned host staging buffers recycled across calls (cudaHostAlloc of tens of
// MB is a millisecond-scale driver call).  Contents are undefined.
void* acquire_pinned(size_t bytes);
void release_pinned(void* p, size_t bytes);
// Host memcpy split over a small persistent worker pool (pageable -> pinned
// staging runs at several threads' memory bandwidth, not one's).
void parallel_memcpy(void* dst, const void* src, size_t bytes);
// true when p is ordinary pageable host memory (not cudaHostAlloc'ed or registered)
bool is_pageable_host(const void* p);

// Wrap a C-ABI body: map exceptions to status codes + thread-local message.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return kOk;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return kInternal;
  }
}

}  // namespace strom

namespace strom {

// ------------------------------------------------------------------ profiling
// Launch counts are always kept; CUDA-event timing per kernel kind only when
// enabled (strom_profile_enable).  Algorithmic bytes: host-known sizes are
// added with prof_add_bytes; kernels whose size is device-side (the iSVD
// passes) add theirs into prof_dev_bytes() with one atomic per launch.
enum ProfKind : int {
  P_PROJ = 0, P_RESID, P_STEP_A, P_STEP_B, P_VUPDATE, P_COMPACT, P_TALL_GEMM, P_SPATIAL,
  P_ST_GEMM, P_ST_SMALL, P_LU, P_TEMPORAL, P_OTHER, P_WPROJ, P_NKINDS
};
void prof_begin(int kind, cudaStream_t s);
void prof_end(int kind, cudaStream_t s);
void prof_add_bytes(int kind, double bytes);
unsigned long long* prof_dev_bytes();  // device array [P_NKINDS]

struct ProfScope {
  int kind;
  cudaStream_t s;
  ProfScope(int k, cudaStream_t st) : kind(k), s(st) { prof_begin(k, st); }
  ~ProfScope() { prof_end(kind, s); }
};

}  // namespace strom
