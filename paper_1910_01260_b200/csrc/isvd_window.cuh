// Window projections of the streaming incremental SVD (window-mode ingestion).
//
// The per-snapshot pass of isvd_kernels.cuh reads all of U for every snapshot,
// also to project the next one.  In window mode one pass projects kWB
// snapshots at once, G = U^T [x_t .. x_{t+kWB-1}] plus their Gram XX, and the
// per-snapshot pass (PASS_RESID) runs only for snapshots that enter U
// (independent ones; basis.py:139).  Columns appended inside the window get
// their rows of G from XX (window_row, isvd_kernels.cuh).  Bytes per snapshot
// drop from 8 n (c + 3) to 8 n ((c + kWB) / kWB + [independent] (c + 2)).
//
// k_wproj: one CTA per SM (minus the core step's), a bulk-copy producer warp
// and 8 consumer warps.  The contraction G_cta += U_tile^T X_tile is DMMA
// m8n8k4 (M = U columns, N = the window, K = rows); per-CTA partials are
// summed by k_wreduce in a fixed order.
#pragma once

#include "isvd_kernels.cuh"
#include "runtime.cuh"

namespace strom {

constexpr int kWXLd = kStageRows + 8;  // 72: x slot stride (conflict-free 16-byte fragment loads)
constexpr int kWConsumers = 16;  // two warps per m-tile group, one per half of the stage's rows
constexpr int kWGroups = 8;      // m-tile groups (warp cw: group cw % 8, row half cw / 8)
constexpr int kWThreads = 32 * (kWConsumers + 1);
constexpr int kWMaxStages = 4;

struct WprojArgs {
  const double* U;
  int64_t ldu, n, ccap;
  const PipeCtl* ctl;
  const double* xs[kWB];
  int32_t nw;     // window columns (<= kWB)
  int32_t xbulk;  // every xs[j] 16-byte aligned and n even: stage x by bulk copy
  double* part;   // per-CTA partials, pstride doubles each: [i * kWB + j] G, then kWB^2 XX
  int32_t pstride;
  unsigned long long* prof;
  long long* trace;
};

// Stage layout: the tile's c live U column segments as ONE contiguous bulk copy
// (a TMA op costs tens of cycles whatever its size: one per stage, not one per
// column), then kWB x slots of kWXLd doubles.  Fragment loads are 16 bytes:
// k-steps are taken in pairs whose rows interleave (lane t of pair kp holds
// rows 8 kp + 2t and 8 kp + 2t + 1), so one LDS.128 feeds two DMMAs.
__host__ __device__ inline size_t wproj_stage_elems(int c) {
  return (size_t)c * kStageRows + (size_t)kWB * kWXLd;
}

template <int MT>  // m-tiles (8 U columns) per consumer warp: c <= 64 MT
__global__ void __launch_bounds__(kWThreads, 1) k_wproj(WprojArgs a, int nstages) {
  extern __shared__ __align__(128) double wst[];
  __shared__ __align__(8) uint64_t full[kWMaxStages];
  __shared__ __align__(8) uint64_t empty[kWMaxStages];
  pdl_enter();
  trace_stamp(a.trace, 14);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int c = a.ctl->c, base = a.ctl->base;
  const int c8 = (c + 7) & ~7;
  const size_t stage_elems = wproj_stage_elems(c);
  const size_t xoff = (size_t)c * kStageRows;
  const int64_t tstride = (int64_t)kUTile * a.ccap;
  if (a.prof && blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd(a.prof + P_WPROJ, 8ull * (unsigned long long)a.n * (unsigned long long)(c + a.nw));
  const int64_t ntiles = a.ldu / kStageRows;
  const int64_t per = ceil_div(ntiles, gridDim.x);
  const int64_t t0 = blockIdx.x * per;
  const int64_t nt = max((int64_t)0, min(ntiles, t0 + per) - t0);
  __shared__ double hsum[kWGroups][(kWB / 2 + 1) * 64];  // the upper row half's accumulators
  if (threadIdx.x == 0) {
    for (int st = 0; st < nstages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kWConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (wid == 0) {
    // ---------------- producer: lane 0 issues one U copy and the x copies per stage
    if (lane == 0) {
      const uint64_t pol_stream = l2_policy_evict_first();  // U is read once per pass (bulk.cuh)
      for (int64_t i = 0; i < nt; ++i) {
        const int st = (int)(i % nstages);
        const int64_t use = i / nstages;
        if (use > 0) mbar_wait(&empty[st], (unsigned)((use - 1) & 1));
        const int64_t row0 = (t0 + i) * kStageRows;
        const int valid = (int)max((int64_t)0, min((int64_t)kStageRows, a.n - row0));
        const unsigned ub = (unsigned)c * kStageRows * 8u;
        const unsigned xb = a.xbulk ? (unsigned)valid * 8u : 0u;
        mbar_expect_tx(&full[st], ub + xb * (unsigned)a.nw);
        double* dst = wst + (size_t)st * stage_elems;
        if (ub) bulk_g2s_stream(dst, a.U + (t0 + i) * tstride + (int64_t)base * kUTile, ub, &full[st], pol_stream);
        if (xb)
          for (int j = 0; j < a.nw; ++j) bulk_g2s(dst + xoff + (size_t)j * kWXLd, a.xs[j] + row0, xb, &full[st]);
      }
    }
  } else {
    // ---------------- consumers: warp cw owns m-tiles (cw % 8) + 8 q over the row
    // half cw / 8 of every stage (two accumulation chains per tile, halved latency)
    const int cw = wid - 1;
    const int grp = cw % kWGroups, half = cw / kWGroups;
    double acc[MT][2];
#pragma unroll
    for (int q = 0; q < MT; ++q) acc[q][0] = acc[q][1] = 0.0;
    double xa0 = 0.0, xa1 = 0.0;
    const double* xg = (g < a.nw) ? a.xs[g] : nullptr;
    for (int64_t i = 0; i < nt; ++i) {
      const int st = (int)(i % nstages);
      const int64_t use = i / nstages;
      mbar_wait(&full[st], (unsigned)(use & 1));
      const double* tile = wst + (size_t)st * stage_elems;
      const int64_t row0 = (t0 + i) * kStageRows;
      const int valid = (int)max((int64_t)0, min((int64_t)kStageRows, a.n - row0));
#pragma unroll 2
      for (int kp = half * (kStageRows / 16); kp < (half + 1) * (kStageRows / 16); ++kp) {
        const int kr = 8 * kp + 2 * t;  // this lane's two rows of the k-step pair
        double2 b = make_double2(0.0, 0.0);
        if (xg) {
          if (a.xbulk) b = *reinterpret_cast<const double2*>(tile + xoff + (size_t)g * kWXLd + kr);
          else if (kr < valid) b = make_double2(__ldg(xg + row0 + kr), kr + 1 < valid ? __ldg(xg + row0 + kr + 1) : 0.0);
          if (kr >= valid) b.x = 0.0;
          if (kr + 1 >= valid) b.y = 0.0;
        }
#pragma unroll
        for (int q = 0; q < MT; ++q) {
          const int col = 8 * (grp + kWGroups * q) + g;
          if (8 * (grp + kWGroups * q) < c) {
            const double2 u = col < c ? *reinterpret_cast<const double2*>(tile + (size_t)col * kStageRows + kr)
                                      : make_double2(0.0, 0.0);
            dmma884(acc[q][0], acc[q][1], u.x, b.x);
            dmma884(acc[q][0], acc[q][1], u.y, b.y);
          }
        }
        if (grp == 0) {  // XX = X^T X (A = X^T: a = X(kr, g) = b)
          dmma884(xa0, xa1, b.x, b.x);
          dmma884(xa0, xa1, b.y, b.y);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    // upper half -> shared, then the lower half adds it (fixed order: deterministic)
    double* hs = hsum[grp];
    if (half == 1) {
#pragma unroll
      for (int q = 0; q < MT; ++q) {
        hs[(2 * q) * 32 + lane] = acc[q][0];
        hs[(2 * q + 1) * 32 + lane] = acc[q][1];
      }
      if (grp == 0) {
        hs[(2 * MT) * 32 + lane] = xa0;
        hs[(2 * MT + 1) * 32 + lane] = xa1;
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kWConsumers) : "memory");
    if (half == 0) {
      double* mypart = a.part + (int64_t)blockIdx.x * a.pstride;
#pragma unroll
      for (int q = 0; q < MT; ++q) {
        const int i = 8 * (grp + kWGroups * q) + g;
        if (i < c) {
          mypart[i * kWB + 2 * t] = acc[q][0] + hs[(2 * q) * 32 + lane];
          mypart[i * kWB + 2 * t + 1] = acc[q][1] + hs[(2 * q + 1) * 32 + lane];
        }
      }
      if (grp == 0) {
        double* xp = mypart + (int64_t)c8 * kWB;
        xp[g * kWB + 2 * t] = xa0 + hs[(2 * MT) * 32 + lane];
        xp[g * kWB + 2 * t + 1] = xa1 + hs[(2 * MT + 1) * 32 + lane];
      }
    }
  }
}

// Sum the per-CTA partials in CTA order (fixed: deterministic) into
// G (c x nw, ld ldg) and XX (kWB x kWB).  32 outputs per CTA, 8 warps split
// the partials, lanes = outputs (coalesced).
__global__ void __launch_bounds__(256) k_wreduce(const double* part, int nparts, int pstride, const PipeCtl* ctl,
                                                 int nw, double* G, int ldg, double* XX) {
  __shared__ double red[8][33];
  pdl_enter();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int c = ctl->c, c8 = (c + 7) & ~7;
  const int nout = c8 * kWB + kWB * kWB;
  const int o = blockIdx.x * 32 + lane;
  double s = 0.0;
  if (o < nout)
    for (int b = wid; b < nparts; b += 8) s += part[(int64_t)b * pstride + o];
  red[wid][lane] = s;
  __syncthreads();
  if (wid == 0 && o < nout) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += red[w][lane];
    if (o < c8 * kWB) {
      const int i = o / kWB, j = o % kWB;
      if (i < c && j < nw) G[(int64_t)j * ldg + i] = v;
    } else {
      XX[o - c8 * kWB] = v;
    }
  }
}

// First snapshot of a window: tvec = L^{-1} G[:, 0], gt = L^{-T} tvec, xx = XX[0, 0]
// (prep_next with the window's column 0 as "next": the caller passes wcol = -1).
__global__ void __launch_bounds__(kDecideThreads) k_prep_w(Pipe pp, IsvdParams P) {
  extern __shared__ double part[];
  pdl_enter();
  prep_next(P, pp, part);
  trace_stamp(P.trace, 15);
}

}  // namespace strom
