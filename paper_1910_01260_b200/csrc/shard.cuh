// Row-sharded incremental SVD: the cross-GPU exchange.
//
// Each rank owns a block of rows of U and of every snapshot; sigma, V, N, L and
// every decision are replicated.  The only data that crosses GPUs are the
// per-rank partial sums the tall kernels already produce -- U^T x, x.x, U^T r,
// r.r (the passes, basis.py:135-139 and 150-156), the window projections
// (isvd_window.cuh) and the Gram of a compacted store -- a few hundred doubles
// per snapshot.  They are exchanged by ONE small kernel over NVLink peer
// memory instead of a library collective:
//
//   every rank has a mailbox [slot][source rank][maxcount] in its own HBM,
//   mapped into every peer (CUDA IPC);  exchange number q uses slot q % 4:
//     publish  rank r stores its partial vector into box[p][slot][r] of every
//              peer p (peer stores travel over NVLink), fences system-wide and
//              raises flag[p][slot][r] = q (st.release.sys)
//     wait     spin (ld.acquire.sys) until its own flag[slot][*] >= q
//     combine  sum box[self][slot][0..world) in RANK ORDER into the vector
//   Every rank adds the same values in the same order: the replicated small
//   state stays bit-identical on all ranks, which the decisions require.
//   Slot reuse is safe with >= 2 slots: a peer can publish q + 2 only after
//   it completed q + 1, i.e. after every rank published q + 1, i.e. after every
//   rank finished combining q.
//
// A single-process group (strom_shard_create_local, the one-GPU test harness)
// splits the kernel into its publish and combine halves and orders them with
// stream events instead of flags: no kernel ever waits for another rank's
// kernel there.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace strom {

constexpr int kShardMax = 8;    // ranks per group (one NVSwitch domain)
constexpr int kShardSlots = 4;  // mailbox ring depth
constexpr int kShardThreads = 512;
constexpr int kShardMaxCount = 128 * 128 + 64;  // the largest exchange: a 128 x 128 Gram

enum : int32_t { SHARD_BOTH = 0, SHARD_PUBLISH = 1, SHARD_COMBINE = 2 };
enum : int32_t { SHARD_ERR_TIMEOUT = 1, SHARD_ERR_COUNT = 2 };

struct ShardDev {
  int32_t rank, world, maxcount, pad;
  double* box[kShardMax];               // box[p]: rank p's mailbox as mapped in this process
  unsigned long long* flag[kShardMax];  // flag[p]: rank p's arrival flags [slot][source]
  unsigned long long* seq;              // this rank's exchange counter (device-side: skipped
                                        // exchanges are skipped by every rank alike)
  int32_t* err;                         // this rank's sticky error word
  long long timeout_ns;
};

// A strided piece of the vector being exchanged: element i at p[(i / rows) * ld + i % rows].
struct ShardSeg {
  double* p;
  int32_t rows, cols;
  int64_t ld;
};
struct ShardSegs {
  ShardSeg s[4];
  int32_t n;
  __device__ int total() const {
    int t = 0;
    for (int i = 0; i < n; ++i) t += s[i].rows * s[i].cols;
    return t;
  }
  __device__ double* at(int i) const {
    for (int k = 0; k < n; ++k) {
      const int cnt = s[k].rows * s[k].cols;
      if (i < cnt) return s[k].p + (int64_t)(i / s[k].rows) * s[k].ld + i % s[k].rows;
      i -= cnt;
    }
    return nullptr;
  }
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// One CTA.  phase: SHARD_BOTH (flags), or the two halves of the event-ordered mode.
__device__ inline void shard_exchange(const ShardDev& sd, const ShardSegs& sg, int phase) {
  __shared__ unsigned long long s_seq;
  const int total = sg.total();
  if (total > sd.maxcount) {
    if (threadIdx.x == 0) *sd.err = SHARD_ERR_COUNT;
    return;
  }
  if (threadIdx.x == 0) s_seq = *sd.seq + (phase == SHARD_COMBINE ? 0ull : 1ull);
  __syncthreads();
  const unsigned long long seq = s_seq;
  const int slot = (int)(seq % kShardSlots);
  const int64_t mine = ((int64_t)slot * sd.world + sd.rank) * sd.maxcount;
  if (phase != SHARD_COMBINE) {
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
      const double v = *sg.at(i);
      for (int p = 0; p < sd.world; ++p) sd.box[p][mine + i] = v;
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) *sd.seq = seq;
    if (phase == SHARD_BOTH && threadIdx.x < sd.world)
      st_release_sys(sd.flag[threadIdx.x] + slot * kShardMax + sd.rank, seq);
    if (phase == SHARD_PUBLISH) return;
  }
  if (phase == SHARD_BOTH) {
    if (threadIdx.x < sd.world) {
      const unsigned long long* f = sd.flag[sd.rank] + slot * kShardMax + threadIdx.x;
      unsigned long long t0, t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      while (ld_acquire_sys(f) < seq) {
        __nanosleep(200);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if ((long long)(t1 - t0) > sd.timeout_ns) {  // a peer died: fail loudly, never hang the GPU
          *sd.err = SHARD_ERR_TIMEOUT;
          break;
        }
      }
      __threadfence_system();
    }
    __syncthreads();
  }
  const double* box = sd.box[sd.rank] + (int64_t)slot * sd.world * sd.maxcount;
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    double s = 0.0;
    for (int p = 0; p < sd.world; ++p) s += __ldcg(box + (int64_t)p * sd.maxcount + i);  // rank order
    *sg.at(i) = s;
  }
}

}  // namespace strom
